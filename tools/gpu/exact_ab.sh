set -x
for v in "B200_GEMM_EXACT_OLD=1" "B200_GEMM_EXACT_AK=4" "B200_GEMM_EXACT_AK=2"; do
  env $v python tools/probe_exact.py
  env $v N=8192 python tools/probe_exact.py
done
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "exact or fullsize or races or tiled or parity or known" > gpurun_out/exact_tests.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/exact_tests.log
