cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pdxg.py tests/test_gpu_spec_acceptance.py -x -q > gpurun_out/pdxg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdxg_tests.log
