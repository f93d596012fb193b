bash tools/ncu_traffic.sh mm_gemm_bf16 gemm_tc2 1 --workload mm --precision bf16
bash tools/ncu_traffic.sh mm_gemm_tf32 gemm_tc2 1 --workload mm --precision tf32
bash tools/ncu_traffic.sh conv_conv_bf16 conv_tc_kernel 1 --workload conv --precision bf16
bash tools/ncu_traffic.sh ls_gemm_bf16 gemm_tc2 2 --workload ls --precision bf16
ls -la gpurun_out/*.ncu-rep | tail -6
