# ncu capture of one fused_sweep_kernel launch (application replay: the 80 GB cost at n = 1e5
# is regenerated per pass instead of being saved/restored by kernel replay)
set -e
cd $GRAFT_REPO_ROOT
N=${1:-100000}
python tools/profile_fused.py $N > gpurun_out/fused_plain.txt 2>&1
ncu --replay-mode application --section SpeedOfLight --section WarpStateStats --section SourceCounters \
    --section MemoryWorkloadAnalysis --section LaunchStats --section Occupancy --import-source on \
    --clock-control none -k regex:"fused_sweep" -s 1 -c 1 -o gpurun_out/fused -f \
    python tools/profile_fused.py $N > gpurun_out/ncu_fused.log 2>&1
ncu -i gpurun_out/fused.ncu-rep --page raw --csv > gpurun_out/fused_raw.csv 2>&1
ncu -i gpurun_out/fused.ncu-rep --page details --csv > gpurun_out/fused_details.csv 2>&1
ncu -i gpurun_out/fused.ncu-rep --page source --csv --print-source sass > gpurun_out/fused_source.csv 2>&1 || true
rm -f gpurun_out/fused.ncu-rep
