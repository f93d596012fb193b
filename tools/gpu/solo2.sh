python tools/probe_gemm.py --kind 0 1 --variant 1 2 3 --init 0
B200_TC_SOLO_OFF=1 python tools/probe_gemm.py --kind 0 --variant 3 --init 0
python tools/probe_gemm.py --kind 0 --variant 1 3 --init 0 --mnk 8192 8192 8192
