# round-end evidence at HEAD: GPU tests, smoke, bench line, launch list of the bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/final_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.log 2> gpurun_out/final_bench.err; echo "rc=$?" >> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/final_bench_ref.log 2> gpurun_out/final_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-tte --no-e2e > gpurun_out/final_ncu.log 2>&1
