cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in g r; do LEANOT_SR_VAR=$v timeout 300 python tools/sr_trace.py > gpurun_out/sr_trace_$v.log 2>&1; done
