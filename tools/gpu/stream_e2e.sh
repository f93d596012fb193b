NOGEMM=1 python tools/probe_stream_e2e.py 4 2 1 3 1 1 1 1
python - <<'PY'
import torch
n=4096
h=torch.rand(n,n).pin_memory(); d=torch.empty(n,n,device='cuda')
for name,f in (("h2d 64MiB",lambda: d.copy_(h,non_blocking=True)),("d2h 64MiB",lambda: h.copy_(d,non_blocking=True))):
    f(); torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/5
    print(name, ms, 'ms', 64*2**20/ms/1e6, 'GB/s')
s1,s2=torch.cuda.Stream(),torch.cuda.Stream()
h2=torch.rand(n,n).pin_memory(); d2=torch.empty(n,n,device='cuda')
torch.cuda.synchronize()
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h,non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2,non_blocking=True)
torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/5
print('bidirectional 64+64 MiB', ms, 'ms')
PY
