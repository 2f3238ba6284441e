# SR sweep: consumer-only timing (LEANOT_SR_DBG_NOWAIT=1: no exchange wait) vs the real sweep
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in g r; do
  for w in 1 0; do
    LEANOT_SR_VAR=$v LEANOT_SR_DBG_NOWAIT=$w timeout 300 python tools/sr_bench.py --iters 10 --modes sr > gpurun_out/sr_bench_${v}_nowait$w.log 2>&1
  done
done
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv > gpurun_out/smi.log
