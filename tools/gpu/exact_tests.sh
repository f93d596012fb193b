python tools/probe_exact.py; N=8192 python tools/probe_exact.py
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "exact or fullsize or tiled or parity or known or random or stream or shard or irgen or calls or sweep" > gpurun_out/exact_tests2.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/exact_tests2.log
python tools/probe_exact.py > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:gemm_exact_tma -s 2 -c 1 -o gpurun_out/exact_tma python tools/probe_exact.py > gpurun_out/ncu_exact_tma.log 2>&1; echo "ncu exit $?"
