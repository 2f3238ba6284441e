cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in base new; do
  if [ $v = base ]; then export LEANOT_LIB=$PWD/expt/lib_base.so; else unset LEANOT_LIB; fi
  for kind in points3 points2; do
    python tools/time_phases.py --kind $kind --n 100000 --iters 6 --tag $v
  done
  python tools/time_phases.py --kind points2 --n 10000 --iters 20 --tag $v
done
done
unset LEANOT_LIB
python -m pytest tests -m gpu -x -q -k "gram or points or parity" 2>&1 | tail -2
