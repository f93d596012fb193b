python tools/probe_gemm.py --kind 0 --variant 3 --init 0 > gpurun_out/plain1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 3 -c 1 -o gpurun_out/solo python tools/probe_gemm.py --kind 0 --variant 3 --init 0 > gpurun_out/ncu_solo.log 2>&1; echo "solo $?"
ONLY=fused python tools/probe_conv_fused.py 8 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -c 1 -o gpurun_out/conv_fused python -c "
import os; os.environ['ONLY']='fused'
import sys; sys.argv=['x','8']; sys.path.insert(0,'tools'); import probe_conv_fused as p; p.main()" > gpurun_out/ncu_cf.log 2>&1; echo "fused $?"
