cd $GRAFT_REPO_ROOT
for v in def a b d; do
  if [ $v = def ]; then L=""; else L="LEANOT_LIB=$PWD/expt/lib_$v.so"; fi
  for k in points3 points2; do env $L timeout 200 python tools/time_phases.py --kind $k --n 100000 --iters 5 --tag $v >> gpurun_out/variants.txt 2>&1; done
  env $L timeout 200 python tools/time_phases.py --kind points2 --n 10000 --iters 20 --tag $v >> gpurun_out/variants.txt 2>&1
done
