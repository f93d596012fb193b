python tools/probe_gemm.py --kind 0 --variant 3 --init 0 > gpurun_out/plain_solo4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 3 -c 1 -o gpurun_out/solo4 python tools/probe_gemm.py --kind 0 --variant 3 --init 0 > gpurun_out/ncu_solo4.log 2>&1; echo "solo4 $?"
cat gpurun_out/plain_solo4.log
