for o in 0 1 2; do for i in 1 2; do B200_GEMM_EXACT_ORD=$o python tools/probe_exact.py; done; done
