for v in "B200_GEMM_EXACT_TMA=1 B200_GEMM_EXACT_TMAV=0" "B200_GEMM_EXACT_TMA=1 B200_GEMM_EXACT_TMAV=1" "B200_GEMM_EXACT_TMA=1 B200_GEMM_EXACT_TMAV=2"; do
  echo "== $v"; for i in 1 2; do env $v python tools/probe_exact.py; done
done
