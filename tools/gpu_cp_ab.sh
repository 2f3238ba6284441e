# pass-B occupancy A/B: default (2 CTAs/SM, 128 registers) vs variants/lib_cp3.so (3 CTAs/SM, 80 registers)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
  for v in base cp3; do
    case $v in base) E="";; cp3) E="LEANOT_LIB=$PWD/variants/lib_cp3.so";; esac
    env $E timeout 300 python tools/time_phases.py --kind hash --n 100000 --iters 6 --tag $v >> gpurun_out/cp_ab.log 2>&1
  done
done
