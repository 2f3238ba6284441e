# SR sweep: parity tests (g, t) of the default build; timing fold-in (default) vs no fold-in, and two-pass
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in g t; do
  LEANOT_SR_VAR=$v timeout 600 python -m pytest tests/test_gpu_single_read.py -x -q > gpurun_out/sr_tests_$v.log 2>&1
done
for rep in 1 2; do
  for v in fold nofold; do
    case $v in fold) E="";; nofold) E="LEANOT_LIB=$PWD/variants/lib_nofold.so";; esac
    env $E timeout 300 python tools/sr_bench.py --iters 10 --modes sr >> gpurun_out/sr_bench_$v.log 2>&1
    env $E LEANOT_SR_DBG_NOWAIT=2 timeout 300 python tools/sr_bench.py --iters 10 --modes sr >> gpurun_out/sr_bench_${v}_dbg2.log 2>&1
  done
  timeout 300 python tools/sr_bench.py --iters 10 --modes two >> gpurun_out/sr_bench_two.log 2>&1
done
