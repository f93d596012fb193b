python tools/probe_exact.py; N=8192 python tools/probe_exact.py
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "exact or fullsize or tiled or stream or known" > gpurun_out/er_tests.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/er_tests.log
python tools/probe_exact.py > gpurun_out/plain.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemm_exact_tma -s 2 -c 1 python tools/probe_exact.py 2>&1 | grep -E "dram__|gpu__time" 
