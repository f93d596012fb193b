"""Benchmark: GFLOP/s of the B200 backend on BASELINE.json's matmul config.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--precision bf16|tf32|exact]

Workload (BASELINE.json configs[1]): ``linalg.matmul`` 4096x4096x4096, the
reference's matmul nest (reference tests/kernels.py:24-38) at full size:
C[i,k] += A[i,j] * B[j,k] on f32 Buffers.  A step is one pass of the hot
path over one batch: one C += A.B contraction, including the operand
packing the tensor-core path needs (f32 -> bf16/tf32, B transposed to
K-major).  Data: U(-1,1) f32 from torch.Generator().manual_seed(arg index)
(SURVEY.md §8d).

* ``value``  — device-resident: the C-ABI sequence (pack, pack, tcgen05
  GEMM) on HBM tensors, timed with CUDA events on the launch stream; inputs
  (3 x 64 MiB f32) are larger than the 126 MB L2.
* ``roofline`` — the dominant kernel (b200_gemm_tc) alone: algorithmic
  2*M*N*K flops per launch / its average CUDA-event duration inside the
  timed region, against MEASURED_PEAKS.json bf16 (tf32: half of it).
* ``e2e``    — through the reference-facing plugin: staircase's own
  ``machine.run(module, "mm", [A, B, C], engine=b200)`` with host Buffers;
  the H2D of A, B, C and the D2H of C are inside the timed region.
* ``cpu_baseline`` — the reference executor itself (baseline/_ref, compiled
  _evalcy engine) on a 1x4096x256 slice of the same nest (same loop
  structure and reduction length), 1 core; its rate extrapolates.
* ``--impl reference`` — rank 0 times that reference CPU path per step.

Multi-GPU (torchrun): every rank runs its own 4096^3 matmul (weak scaling,
no data-path collective); time is the max over ranks.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()

from staircase import F32, MemRef, staged  # noqa: E402

M = N = K = 4096
FLOP = 2.0 * M * N * K


@staged(range_ctor="affine_for")
def mm(A: MemRef[(4096, 4096), F32], B: MemRef[(4096, 4096), F32],
       C: MemRef[(4096, 4096), F32]):
    for i in range(4096):
        for j in range(4096):
            for k in range(4096):
                a = A[i, j]
                b = B[j, k]
                c = C[i, k]
                d = a * b
                e = c + d
                C[i, k] = e


@staged(range_ctor="affine_for")
def mm_slice(A: MemRef[(1, 4096), F32], B: MemRef[(4096, 256), F32],
             C: MemRef[(1, 256), F32]):
    for i in range(1):
        for j in range(4096):
            for k in range(256):
                a = A[i, j]
                b = B[j, k]
                c = C[i, k]
                d = a * b
                e = c + d
                C[i, k] = e


def host_inputs(shapes, dtype="f32"):
    import torch
    from staircase.interp import Buffer

    out = []
    for seed, shape in enumerate(shapes):
        g = torch.Generator().manual_seed(seed)
        t = torch.rand(shape, generator=g, dtype=torch.float32) * 2 - 1
        out.append(Buffer(shape, dtype, t.numpy().tobytes()))
    return out


def reference_slice_rate():
    """GFLOP/s of the reference's compiled executor on the 1x4096x256 slice."""
    from staircase.interp import _evalcy, machine

    times = []
    for _ in range(3):
        args = host_inputs([(1, 4096), (4096, 256), (1, 256)])
        _, stats = machine.run(mm_slice.module, "mm_slice", args, engine=_evalcy)
        times.append(stats.wall_time)
    t = statistics.median(times)
    flops = 2.0 * 1 * 4096 * 256
    return flops / t / 1e9, t


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md recipe)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.proc = None
        self.path = f"/tmp/b200_clocks_{os.getpid()}.csv"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        t0 = time.time()
        while time.time() - t0 < 5.0:
            if os.path.exists(self.path) and os.path.getsize(self.path) > 0:
                break
            time.sleep(0.02)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return json.load(open(path)), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def load_traffic(precision):
    """dram bytes per GEMM launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        return json.load(open(path)).get(f"gemm_{precision}")
    return None


def run_reference(args, rank, world):
    if rank != 0:
        return
    rates = []
    for _ in range(args.warmup):
        reference_slice_rate()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        rate, _ = reference_slice_rate()
        rates.append(rate)
    wall = time.perf_counter() - t0
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": "GFLOP/s (matmul 4096^3)", "value": value,
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "linalg.matmul 4096x4096x4096 (reference CPU executor on a "
                               "1x4096x256 slice of the nest, rate extrapolates)"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": 1, "kind": "reference",
                         "sample": "1x4096x256 slice of the 4096^3 matmul nest, "
                                   "staircase _evalcy, median of 3 runs per step"},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import runtime
    from staircase.interp import machine

    lib = runtime.load_library()
    dev = torch.device("cuda", local)
    tens = []
    for seed, shape in enumerate([(M, K), (K, N), (M, N)]):
        g = torch.Generator().manual_seed(seed)
        tens.append((torch.rand(shape, generator=g) * 2 - 1).to(dev))
    A, B, C = tens
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    prec = args.precision
    tc = runtime.tc_supported(prec, K)
    kind = 0 if prec == "bf16" else 1
    elt = torch.bfloat16 if prec == "bf16" else torch.float32
    Ap = torch.empty(M, K, dtype=elt, device=dev)
    Bp = torch.empty(N, K, dtype=elt, device=dev)
    P = ctypes.c_void_p
    gemm_ms = []

    def step(timed):
        if tc:
            assert lib.b200_pack_operand(kind, P(A.data_ptr()), K, 1, P(Ap.data_ptr()),
                                         M, K, sp) == 0
            assert lib.b200_pack_operand(kind, P(B.data_ptr()), 1, N, P(Bp.data_ptr()),
                                         N, K, sp) == 0
        if timed:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        if tc:
            rc = lib.b200_gemm_tc(kind, P(Ap.data_ptr()), P(Bp.data_ptr()), P(C.data_ptr()),
                                  N, 1, M, N, K, 0, 0.0, None, 0, 0, args.variant, sp)
        else:
            rc = lib.b200_gemm_f32_exact(P(A.data_ptr()), K, 1, P(B.data_ptr()), N, 1,
                                         P(C.data_ptr()), N, 1, M, N, K, 0, 0.0, None, 0, sp)
        assert rc == 0
        if timed:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record(stream)
            gemm_ms.append((e0, e1))

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    barrier(world)
    clocks = Clocks(local)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(True)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    kernel_ms = statistics.mean(a.elapsed_time(b) for a, b in gemm_ms)
    clk = clocks.stop()
    barrier(world)
    ms = max_over_ranks(ms, world)
    kernel_ms = max_over_ranks(kernel_ms, world)
    value = world * FLOP / (ms * 1e-3) / 1e9
    launches_per_step = 3 if tc else 1

    # e2e through the plugin: host Buffers, H2D + D2H inside the timed region
    b2.configure(precision=prec)
    e2e_steps = max(1, min(args.steps, 3))
    host = host_inputs([(M, K), (K, N), (M, N)])
    machine.run(mm.module, "mm", host, engine=b2.engine)   # warm
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        machine.run(mm.module, "mm", host, engine=b2.engine)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    e2e_ms = max_over_ranks(e2e_ms, world)
    plan = list(b2.engine.last_plan)

    if rank != 0:
        return
    peaks, src = load_peaks()
    if tc:
        peak = peaks["bf16_tflops"] * (1.0 if prec == "bf16" else 0.5)
        bound = "tensor"
        peak_source = (f"{src} bf16 dense (MEASURED_PEAKS.json)" if prec == "bf16" else
                       f"{src} bf16 x 0.5 (tf32 = half rate, derived)")
    else:
        peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        bound = "fp32-simt"
        peak_source = "derived: 148 SM x 128 FP32 lanes x 2 x sm_max_mhz"
    achieved = FLOP / (kernel_ms * 1e-3) / 1e12
    cpu_rate, cpu_t = reference_slice_rate()
    dtype = {"bf16": "bf16 (fp32 accumulate)", "tf32": "tf32 (fp32 accumulate)",
             "exact": "f32"}[prec]
    line = {
        "metric": "GFLOP/s (matmul 4096^3)", "value": value, "unit": "GFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic",
        "config": {"workload": "linalg.matmul 4096x4096x4096, C += A.B on f32 buffers "
                               "(step = operand pack + contraction)",
                   "precision": prec, "l2": "inputs 192 MiB f32 > 126 MB L2 (no flush)",
                   "parallelism": f"replica x{world}"},
        "roofline": {"bound": bound, "kernel": "b200_gemm_tc" if tc else "b200_gemm_f32_exact",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "peak_source": peak_source,
                     "kernel_ms": kernel_ms, "traffic": load_traffic(prec)},
        "e2e": {"value": FLOP / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                "ms_per_step": e2e_ms, "h2d_bytes_per_step": 3 * M * N * 4,
                "d2h_bytes_per_step": M * N * 4, "plan": [list(p) for p in plan]},
        "cpu_baseline": {"value": cpu_rate, "unit": "GFLOP/s", "cores": 1,
                         "kind": "reference",
                         "sample": f"1x4096x256 slice of the matmul nest via staircase _evalcy "
                                   f"({cpu_t:.2f} s); host cores {len(os.sched_getaffinity(0))}"},
        "clocks": clk, "gpu_launches": launches_per_step * args.steps,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "tf32", "exact"])
    ap.add_argument("--variant", type=int, default=0,
                    help="tcgen05 schedule: 0 auto, 1 single-CTA, 2 CTA pair")
    args = ap.parse_args()
    rank, world, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
