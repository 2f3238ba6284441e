# ncu source/raw pages of the single-read sweep (variant $V, debug mode $DBG) on a row shard
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in g:2 g:0; do
  V=${cfg%%:*}; DBG=${cfg##*:}
  LEANOT_SR_VAR=$V LEANOT_SR_DBG_NOWAIT=$DBG timeout 600 ncu --set full --import-source on --clock-control none -k regex:sr_sweep -c 1 \
     -o /tmp/sr_$V$DBG python tools/profile_sr.py --reps 2 > gpurun_out/ncu_sr_$V$DBG.log 2>&1
  ncu -i /tmp/sr_$V$DBG.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sr_${V}${DBG}_sass.csv 2>&1
  ncu -i /tmp/sr_$V$DBG.ncu-rep --page details --csv > gpurun_out/ncu_sr_${V}${DBG}_details.csv 2>&1
done
