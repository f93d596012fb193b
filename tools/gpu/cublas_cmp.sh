python tools/probe_gemm.py --cublas --kind 0 --variant 2 --init 1 0 --iters 50
python tools/probe_gemm.py --cublas --kind 0 --variant 2 --init 1 --iters 20 --mnk 8192 8192 8192
python - <<'PY'
import torch
X=torch.randn(4096,4096,device='cuda').bfloat16(); Y=torch.randn(4096,4096,device='cuda').bfloat16()
try:
    for _ in range(3): Z=torch.mm(X,Y,out_dtype=torch.float32)
    torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): Z=torch.mm(X,Y,out_dtype=torch.float32)
    e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/50
    print('cublas bf16->f32 out 4096 ms', ms, 2*4096**3/ms/1e9)
except Exception as e: print('no out_dtype', e)
PY
