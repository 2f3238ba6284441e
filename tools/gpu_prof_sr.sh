# SR sweep A/B (register vs TMEM parking) + ncu source/raw pages of each; reports land in
# gpurun_out/ as CSV (the .ncu-rep files stay on the box: they exceed the copy-back limit)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tm in 1 0; do
  LEANOT_SR_TM=$tm timeout 300 python tools/profile_sr.py > gpurun_out/prof_sr_tm$tm.log 2>&1
done
for tm in 1 0; do
  LEANOT_SR_TM=$tm timeout 300 python tools/sr_bench.py --iters 10 --modes sr > gpurun_out/sr_bench_tm$tm.log 2>&1
done
timeout 300 python tools/sr_bench.py --iters 10 --modes two > gpurun_out/sr_bench_two.log 2>&1
for tm in 1 0; do
  LEANOT_SR_TM=$tm timeout 600 ncu --set full --import-source on --clock-control none -k regex:sr_sweep -c 1 \
     -o /tmp/sr_tm$tm python tools/profile_sr.py --reps 2 > gpurun_out/ncu_sr_tm$tm.log 2>&1
  ncu -i /tmp/sr_tm$tm.ncu-rep --page raw --csv > gpurun_out/ncu_sr_tm${tm}_raw.csv 2>&1
  ncu -i /tmp/sr_tm$tm.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sr_tm${tm}_sass.csv 2>&1
  ncu -i /tmp/sr_tm$tm.ncu-rep --page details --csv > gpurun_out/ncu_sr_tm${tm}_details.csv 2>&1
done
ls -la gpurun_out
