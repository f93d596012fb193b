"""Dev probe: the device timeline of one end-to-end run (runtime.STREAM_TRACE:
timed events around each streamed panel's upload, kernels and write-back),
printed relative to the run's first event.

    python tools/probe_stream_trace.py [workload] [precision]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import bench
    import torch

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import runtime
    from staircase.interp import machine

    name = sys.argv[1] if len(sys.argv) > 1 else "ls"
    wl = bench.Workload(name)
    b2.configure(precision=sys.argv[2] if len(sys.argv) > 2 else "bf16")
    host = bench.host_inputs(wl.fn)
    for _ in range(2):
        machine.run(wl.fn.module, wl.fn.__name__, host, engine=b2.engine)
    torch.cuda.synchronize()
    runtime.STREAM_TRACE = []
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record()
    w0 = time.perf_counter()
    # host-side: when each streamed op was entered (ms after the run started)
    orig = runtime.Staging.stream_rows

    def traced(self, *a, **k):
        print(f"host: stream_rows entered at {1e3 * (time.perf_counter() - w0):.2f} ms")
        return orig(self, *a, **k)

    runtime.Staging.stream_rows = traced
    machine.run(wl.fn.module, wl.fn.__name__, host, engine=b2.engine)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record()
    torch.cuda.synchronize()
    print(f"run: wall {1e3 * (time.perf_counter() - w0):.2f} ms, device {t0.elapsed_time(t1):.2f} ms")
    for what, e in runtime.STREAM_TRACE:
        print(f"{t0.elapsed_time(e):8.2f} ms  {what}")
    runtime.STREAM_TRACE = None


if __name__ == "__main__":
    main()
