for gsz in 8 16 32; do
B200_GEMM_EXACT_GROUP=$gsz python tools/probe_exact.py
B200_GEMM_EXACT_GROUP=$gsz ncu --metrics dram__bytes_read.sum -k regex:gemm_exact_tma -s 2 -c 1 python tools/probe_exact.py 2>&1 | grep -E "dram__"
done
