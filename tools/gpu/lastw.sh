# Measured a last-warp-refill variant (B200_GEMM_EXACT_EAGER=2) that was not kept.
for i in 1 2 3; do
echo "deferred:"; python tools/probe_exact.py
echo "last-warp:"; B200_GEMM_EXACT_EAGER=2 python tools/probe_exact.py
done
echo "deferred 8192:"; N=8192 python tools/probe_exact.py
echo "last-warp 8192:"; N=8192 B200_GEMM_EXACT_EAGER=2 python tools/probe_exact.py
