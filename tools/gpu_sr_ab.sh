# SR sweep: parity tests (variants g, t, r) + timing of g (real / no exchange wait / compute only) vs two-pass
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in g t r; do
  LEANOT_SR_VAR=$v timeout 600 python -m pytest tests/test_gpu_single_read.py -x -q > gpurun_out/sr_tests_$v.log 2>&1
done
for w in 0 1 2; do
  LEANOT_SR_VAR=g LEANOT_SR_DBG_NOWAIT=$w timeout 300 python tools/sr_bench.py --iters 10 --modes sr > gpurun_out/sr_bench_g_dbg$w.log 2>&1
done
timeout 300 python tools/sr_bench.py --iters 10 --modes two,sr > gpurun_out/sr_bench_two.log 2>&1
