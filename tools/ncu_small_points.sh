# ncu of the expanded-form pass A / pass B at n = 1e4 (BASELINE config 2 shape)
set -e
cd $GRAFT_REPO_ROOT
python tools/profile_sweep.py --kind points2 --n 10000 --iters 3 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"rowpass|colpass" -s 2 -c 2 -o gpurun_out/small_pts -f \
    python tools/profile_sweep.py --kind points2 --n 10000 --iters 3 > gpurun_out/ncu_small_pts.log 2>&1
ncu -i gpurun_out/small_pts.ncu-rep --page raw --csv > gpurun_out/small_pts_raw.csv 2>&1
ncu -i gpurun_out/small_pts.ncu-rep --page source --csv --print-source sass > gpurun_out/small_pts_source.csv 2>&1 || true
rm -f gpurun_out/small_pts.ncu-rep
