python tools/probe_exact.py > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:gemm_exact_full -s 2 -c 1 \
    -o gpurun_out/exact_full python tools/probe_exact.py > gpurun_out/ncu_exact.log 2>&1
echo "exit $?"; tail -3 gpurun_out/ncu_exact.log
