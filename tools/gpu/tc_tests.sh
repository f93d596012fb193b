timeout 600 python -m pytest tests/test_gpu_tc.py -x -q > gpurun_out/tc_tests.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/tc_tests.log
