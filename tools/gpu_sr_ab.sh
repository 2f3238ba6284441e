# SR variant w (16 warps) vs g: real / no exchange wait / compute only
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in w g; do
  for w in 0 1 2; do
    LEANOT_SR_VAR=$v LEANOT_SR_DBG_NOWAIT=$w timeout 300 python tools/sr_bench.py --iters 10 --modes sr > gpurun_out/sr_bench_${v}_dbg$w.log 2>&1
  done
done
