for i in 1 2; do
echo "deferred:"; python tools/probe_exact.py
echo "eager:"; B200_GEMM_EXACT_EAGER=1 python tools/probe_exact.py
done
echo "deferred 8192:"; N=8192 python tools/probe_exact.py
echo "eager 8192:"; N=8192 B200_GEMM_EXACT_EAGER=1 python tools/probe_exact.py
timeout 900 python -m pytest tests/test_gpu_exact_tma.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/ed_tests.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/ed_tests.log
