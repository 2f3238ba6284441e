cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_single_read.py -x -q > gpurun_out/sr_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sr_tests.log
