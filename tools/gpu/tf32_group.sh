for gm in 4 8 16 32; do
B200_TC2_GROUP=$gm python tools/probe_gemm.py --kind 1 --variant 2 --init 0 --iters 50 | tail -1
B200_TC2_GROUP=$gm ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gemm_tc2 -s 5 -c 1 python tools/probe_gemm.py --kind 1 --variant 2 --init 0 --iters 5 2>&1 | grep -E "dram__|gpu__time" | tr -s ' ' | tr '\n' ' '; echo " <- group $gm"
done
for gm in 4 8 16; do
B200_TC2_GROUP=$gm python tools/probe_gemm.py --kind 0 --variant 2 --init 0 --iters 50 | tail -1
done
