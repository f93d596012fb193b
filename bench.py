"""Benchmark: GFLOP/s of the B200 backend on BASELINE.json's configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload auto|mm|mm_tiled|conv|ls|linear32|ewise|sweep]
                    [--precision exact|tf32|bf16] [--min-seconds S]

Default (``--workload auto``) prints ONE JSON line:

* N = 1: the headline is BASELINE configs[1], ``linalg.matmul`` 4096^3 —
  the reference's matmul nest (reference tests/kernels.py:24-38) at full
  size on f32 Buffers, at the reference's own arithmetic (``exact``: every
  product and sum rounded to f32 in nest order, bit-identical to the
  reference executor).  ``variants`` carries the same config on the tensor
  cores (bf16, tf32) and with the reference tile sizes (8, 8) / (4, 16)
   through the reference's tiling pass; ``configs`` carries
  every other BASELINE config: Linear(32,32) (configs[0]), the ResNet conv
  exact and bf16 (configs[2]), the Linear stack (configs[3]), the
  elementwise nest, and the 512-config sweep (configs[4]).
* N > 1 (torchrun, one rank per GPU): the headline is configs[2], the
  ResNet conv batch-sharded over the ranks (paper_2307_16080_b200.shard:
  contiguous image ranges, the worksharing rule of interp/_evalpy.py:279);
  ``configs`` adds the bf16 conv, the Linear stack and the sweep, sharded the
  same way (N=1's line carries the same records for the scaling baseline).

Per record:

* ``value`` — device-resident: the engine's own launch sequence (recorded
  once by paper_2307_16080_b200.Session, replayed as a CUDA graph), K steps
  timed with CUDA events on the launch stream, max over ranks; inputs are
  larger than the 126 MB L2 except linear32 (stated in ``config.l2``).
* ``sustained`` — the same replay back to back for >= --min-seconds, with
  the nvidia-smi clock sampler running (``clocks`` covers both regions).
* ``roofline`` — the dominant kernel family, timed per launch with CUDA
  events: algorithmic flops (or bytes) / time against MEASURED_PEAKS.json
  (burst), plus the step's fraction of the sustained peak.
* ``e2e`` — through the reference-facing plugin: staircase's own
  ``machine.run`` (or shard.run) on host Buffers, host<->device copies in
  the timed region, >= --min-seconds of runs.
* ``cpu_baseline`` — the reference executor (baseline/_ref, compiled
  _evalcy engine) on a slice of the same nest, one process per host core
  running concurrently; the rate extrapolates to the full size.
* ``--impl reference`` — rank 0 times that same reference CPU path per step.
"""
import argparse
import ctypes
import json
import math
import multiprocessing as mproc
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()

import bench_kernels as bk  # noqa: E402

TILE = "builtin.module(func.func(scf-parallel-loop-tiling{{sizes=[{}, {}]}}))"


# -- workloads -------------------------------------------------------------------

class Workload:
    """One BASELINE config: the nest, its flops, its CPU slice."""

    def __init__(self, name, tiles=None):
        self.name = name
        self.tiles = tiles
        self.sharded = False
        self.module = None
        self.bytes = None
        self.tc_bytes = None
        if name == "mm":
            self.fn = bk.mm_par4096 if tiles else bk.mm4096
            self.flops = 2.0 * 4096 ** 3
            self.desc = ("linalg.matmul 4096x4096x4096, C += A.B on f32 buffers" +
                         (f", parallel form tiled ({tiles[0]}, {tiles[1]}) by the reference's "
                          f"scf-parallel-loop-tiling" if tiles else ""))
            self.slice = (bk.mm_slice, 2.0 * 4096 * 256, "1x4096x256 slice of the matmul nest")
            self.config = "configs[1]"
        elif name == "conv":
            self.fn = bk.make_conv(256)
            self.flops = 2.0 * 256 * 64 * 56 * 56 * 64 * 9
            self.sharded = True
            self.desc = ("conv_2d_nchw_fchw N=256 C=F=64 58x58 pre-padded -> 56x56, 3x3, f32 "
                         "buffers, out += conv")
            self.slice = (bk.conv_slice, 2.0 * 2 * 8 * 56 * 64 * 9,
                          "1x2x8x56 outputs of the conv nest (C=64, 3x3)")
            # algorithmic DRAM bytes of b200_conv2d_tc: the NHWC bf16 input
            # once, the f32 output read and written (out += conv)
            self.tc_bytes = 256 * 58 * 58 * 64 * 2 + 2 * 256 * 64 * 56 * 56 * 4
            # the fused kernel reads the f32 NCHW input itself
            self.tc_fused_bytes = 256 * 58 * 58 * 64 * 4 + 2 * 256 * 64 * 56 * 56 * 4
            self.config = "configs[2]"
        elif name == "ls":
            self.fn = bk.make_linear_stack(65536)
            self.flops = 2.0 * 65536 * (1024 * 4096 * 2) + 2.0 * 65536 * (4096 + 1024)
            self.sharded = True
            self.desc = ("Linear stack 65536 x 1024 -> 4096 -> 1024, fill + contraction + bias "
                         "nests per layer")
            self.slice = (bk.make_linear_stack(1), 2.0 * (1024 * 4096 * 2),
                          "1 row through both Linear lowerings")
            self.config = "configs[3]"
        elif name == "linear32":
            self.fn = bk.linear32
            self.flops = 2.0 * 32 ** 3 + 32 * 32
            self.desc = "torch.nn.Linear(32,32) lowering: fill + copy + 32^3 contraction + bias"
            self.slice = (bk.linear32, self.flops, "the full Linear(32,32) lowering")
            self.config = "configs[0]"
        elif name == "ewise":
            self.fn = bk.saxpy8k
            self.flops = 2.0 * 8192 * 8192
            self.bytes = 3 * 8192 * 8192 * 4
            self.desc = "elementwise y = y + 2x over 8192x8192 f32 (512 MB working set)"
            self.slice = (bk.saxpy_slice, 2.0 * 16 * 4096, "16x4096 rows of the same nest")
            self.config = "fill / copy / ewise nests (SURVEY a14)"
        else:
            raise SystemExit(f"unknown workload {name!r}")
        self.module = self.fn.module
        if tiles:
            from staircase.passes import run_pipeline

            self.module, _ = run_pipeline(self.fn.module, TILE.format(*tiles))
        self.func = self.fn.__name__

    @property
    def key(self):
        return self.name + (f"_tile{self.tiles[0]}x{self.tiles[1]}" if self.tiles else "")


def host_inputs(fn):
    """U(-1,1) f32 Buffers, arg i from torch.Generator().manual_seed(i)
    (SURVEY §8d): the same global batch on every rank."""
    import torch
    from staircase.interp import Buffer

    out = []
    for i, a in enumerate(fn.func_op.body().args):
        shape = tuple(a.type.shape)
        g = torch.Generator().manual_seed(i)
        t = torch.rand(shape, generator=g, dtype=torch.float32) * 2 - 1
        out.append(Buffer(shape, "f32", t.numpy().tobytes()))
    return out


# -- the reference CPU path: one process per host core ----------------------------

def _ref_worker(conn, name):
    """A process that times the reference executor on a workload's slice."""
    sys.path.insert(0, ROOT)
    from paper_2307_16080_b200.host import ensure_staircase

    ensure_staircase()
    from staircase.interp import _evalcy, machine

    fn = _slice_fn(name)
    args = host_inputs(fn)
    while True:
        msg = conn.recv()
        if msg is None:
            return
        # the nest accumulates into its output: fresh inputs each time keep
        # the values (and the timing) the same as a first run
        args = host_inputs(fn)
        _, stats = machine.run(fn.module, fn.__name__, args, engine=_evalcy)
        conn.send(stats.wall_time)


def _slice_fn(name):
    return {"mm": bk.mm_slice, "conv": bk.conv_slice, "ls": None, "linear32": bk.linear32,
            "ewise": bk.saxpy_slice}.get(name) or bk.make_linear_stack(1)


class ReferencePool:
    """C concurrent processes of the reference executor (staircase _evalcy,
    from baseline/_ref), one per host core: the reference's interpreter is
    single-threaded (its worksharing mode does not scale under the GIL), so
    this is how it uses all the cores.  Each sample = one slice run in every
    process at once; rate = sum of the per-process rates."""

    def __init__(self, wl, cores=None):
        self.wl = wl
        self.cores = cores or len(os.sched_getaffinity(0))
        ctx = mproc.get_context("spawn")
        self.conns, self.procs = [], []
        for _ in range(self.cores):
            a, b = ctx.Pipe()
            p = ctx.Process(target=_ref_worker, args=(b, wl.name), daemon=True)
            p.start()
            self.conns.append(a)
            self.procs.append(p)

    def sample(self):
        """(aggregate GFLOP/s, median seconds per slice run)."""
        for c in self.conns:
            c.send(1)
        times = [c.recv() for c in self.conns]
        flops = self.wl.slice[1]
        return sum(flops / t for t in times) / 1e9, statistics.median(times)

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except (BrokenPipeError, OSError):
                pass
        for p in self.procs:
            p.join(timeout=10)

    def describe(self, t):
        return (f"{self.wl.slice[2]} via staircase _evalcy, {self.cores} concurrent processes "
                f"(one per host core; {t:.2f} s per slice run); rate extrapolates to the full "
                f"nest")


def cpu_baseline(wl, repeats=2):
    pool = ReferencePool(wl)
    try:
        pool.sample()   # warm: imports done, caches warm
        res = [pool.sample() for _ in range(repeats)]
    finally:
        pool.close()
    rate = statistics.median(r[0] for r in res)
    return {"value": rate, "unit": "GFLOP/s", "cores": pool.cores, "kind": "reference",
            "sample": pool.describe(statistics.median(r[1] for r in res))}


# -- measurement helpers ----------------------------------------------------------

class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md recipe)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,utilization.gpu")

    def __init__(self, index):
        self.proc = None
        self.path = f"/tmp/b200_clocks_{os.getpid()}_{time.time_ns()}.csv"
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
        sm, mx, reasons, power, loaded = [], [], set(), [], 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                util = float(parts[7])
            except ValueError:
                util = 0.0
            if util < 50:
                continue   # idle samples around the timed region
            loaded += 1
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                power.append(float(parts[6]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower() == "active":
                    reasons.add(name)
        try:
            os.unlink(self.path)
        except OSError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples_under_load": loaded,
                "power_w_median": statistics.median(power) if power else None}


def dist_setup():
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        # B200_BENCH_BACKEND=gloo lets the multi-rank path be exercised with
        # several ranks on one GPU (host-side collectives only); default NCCL
        backend = os.environ.get("B200_BENCH_BACKEND", "nccl")
        ngpu = torch.cuda.device_count()
        torch.cuda.set_device(local % max(1, ngpu))
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def _coll_device():
    import torch.distributed as dist

    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def capture_graph(fn):
    """Capture fn's launches (on the current stream) into a CUDA graph."""
    import torch

    try:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()   # warm-up on a side stream, as torch requires before capture
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
        return g
    except Exception as exc:  # graph capture is an optimisation of the timing only
        print(f"# graph capture failed ({exc}); timing eager replays", file=sys.stderr)
        torch.cuda.synchronize()
        return None


def gather_checksums(value, world):
    """One all_gather of per-rank result checksums (harness only)."""
    if world == 1:
        return [value]
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=_coll_device())
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return json.load(open(path)), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1590.0,
            "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


_TF32_PEAK = {}


def tf32_peak():
    """Dense tf32 tensor-core peak measured here (MEASURED_PEAKS.json has
    bf16 only): cuBLAS fp32 GEMM with tf32 allowed, 8192^3, best of 10 after
    warm-up, CUDA events (burst, like the bf16 figure it sits beside).
    Cached for the process; None without a GPU."""
    if "v" in _TF32_PEAK:
        return _TF32_PEAK["v"]
    import torch

    v = None
    if torch.cuda.is_available():
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        try:
            n = 8192
            a = torch.randn(n, n, device="cuda")
            b = torch.randn(n, n, device="cuda")
            for _ in range(3):
                torch.matmul(a, b)
            best = None
            for _ in range(10):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                torch.matmul(a, b)
                e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1)
                best = ms if best is None else min(best, ms)
            v = 2.0 * n ** 3 / (best * 1e-3) / 1e12
            del a, b
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
    _TF32_PEAK["v"] = v
    return v


def load_traffic(key):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        return json.load(open(path)).get(key)
    return None


KERNEL_OF = {"b200_gemm_tc": "gemm", "b200_gemm_f32_exact": "gemm",
             "b200_contract_exact": "contract", "b200_map_f32": "map", "b200_vm_run": "vm",
             "b200_pack_operand": "pack", "b200_conv2d_tc": "conv",
             "b200_pack_conv_input": "pack", "b200_pack_conv": "pack",
             "b200_conv2d_exact": "conv", "b200_jit_launch": "map",
             "b200_conv2d_tc_fused": "conv", "b200_pack_conv_weight": "pack"}
TENSOR_KERNELS = ("b200_gemm_tc", "b200_conv2d_tc", "b200_conv2d_tc_fused")
# entry points that run the same kernel family (timed together)
ALIASES = {"b200_gemm_tc_shadow": "b200_gemm_tc", "b200_gemm_tc_kn": "b200_gemm_tc",
           "b200_gemm_f32_exact_tiled": "b200_gemm_f32_exact"}
DTYPE = {"bf16": "bf16 (fp32 accumulate)", "tf32": "tf32 (fp32 accumulate)", "exact": "f32",
         "f32x3": "f32 (3xTF32 split, fp32 accumulate; within fp32 rel 1e-5)"}


def _timed(fn, stream, min_steps, min_seconds):
    """Run fn back to back (>= min_steps, >= min_seconds): (ms per call, calls)."""
    import torch

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # estimate the call time first so the region is sized without host syncs inside
    torch.cuda.synchronize()
    e0.record(stream)
    fn()
    e1.record(stream)
    torch.cuda.synchronize()
    one = max(e0.elapsed_time(e1), 1e-3)
    n = max(min_steps, int(math.ceil(min_seconds * 1e3 / one)))
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(n):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, n


# -- our arm ---------------------------------------------------------------------

def measure(wl, prec, rank, world, local, steps, warmup, min_seconds, with_cpu=True,
            with_e2e=True):
    """One record for workload ``wl`` at precision ``prec`` on this rank."""
    import torch

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import runtime, shard
    from staircase.interp import machine

    lib = runtime.load_library()
    b2.configure(precision=prec)
    sharded = wl.sharded and world > 1
    sess = b2.Session(shard=(rank, world) if sharded else None)
    dev_args = host_inputs(wl.fn)
    rec = sess.record(wl.module, wl.func, dev_args)
    plan = list(sess.plan)
    rows = sess.last_shard.rows if sharded else None
    torch.cuda.synchronize()
    # the recorded run applied the nest once: check sampled outputs against
    # the host recomputation before the replays accumulate further
    acc_rec = (accuracy(wl, prec, dev_args, sess.tensor(dev_args[-1]))
               if rank == 0 and not sharded else None)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        rec.replay(lib)
    torch.cuda.synchronize()
    step_graph = capture_graph(lambda: rec.replay(lib))
    run_step = step_graph.replay if step_graph is not None else (lambda: rec.replay(lib))
    for _ in range(warmup):
        run_step()
    torch.cuda.synchronize()
    barrier(world)
    clocks = Clocks(local)
    # the contract's timed region: exactly `steps` steps
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(steps):
        run_step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    # sustained: the same steps back to back for >= min_seconds
    sus_ms, sus_n = _timed(run_step, stream, steps, min_seconds)
    clk = clocks.stop()
    # per-launch device time of each recorded call: a graph of R back-to-back
    # repeats of that one launch, timed with events, / R
    fam = {}
    reps = 20 if ms < 1.0 else 3
    for cname, cargs in rec.calls:
        def one(cname=cname, cargs=cargs):
            s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            for _ in range(reps):
                runtime.check(getattr(lib, cname)(*cargs[:-1], s), cname)
        gph = capture_graph(one)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gph.replay() if gph is not None else one()
        e1.record(stream)
        torch.cuda.synchronize()
        key = ALIASES.get(cname, cname)
        fam[key] = fam.get(key, 0.0) + e0.elapsed_time(e1) / reps
    barrier(world)
    ms = max_over_ranks(ms, world)
    sus_ms = max_over_ranks(sus_ms, world)
    # whole-job work: the global batch when sharded, one nest per rank otherwise
    job_flops = wl.flops if sharded else world * wl.flops
    out = sess.tensor(dev_args[-1])
    if rows is not None:
        out = out.view(dev_args[-1].shape[0], -1)[rows[0]:rows[1]]
    sums = gather_checksums(float(out.double().sum().item()), world)
    n_launch = rec.launches
    del sess, rec, step_graph, dev_args
    torch.cuda.synchronize()

    e2e = gather = None
    if with_e2e:
        e2e, gather = _e2e(wl, rank, world, sharded, min_seconds)
    b2.configure(precision="exact")
    rate_flops = wl.flops if not sharded else wl.flops * (rows[1] - rows[0]) / \
        wl.fn.func_op.body().args[0].type.shape[0]
    rec_out = {
        "metric": f"GFLOP/s ({wl.key}, {prec})", "value": job_flops / (ms * 1e-3) / 1e9,
        "unit": "GFLOP/s", "ms_per_step": ms, "steps": steps,
        "dtype": DTYPE[prec], "precision": prec,
        "config": {"workload": wl.desc, "baseline_config": wl.config,
                   "parallelism": (f"batch shard x{world} (rows {rows[0]}..{rows[1] - 1} on "
                                   f"rank {rank})" if sharded else
                                   f"replica x{world}" if world > 1 else "1 GPU"),
                   "l2": ("L2-resident, latency-bound config" if wl.name == "linear32" else
                          "inputs larger than the 126 MB L2 (no flush needed)"),
                   "plan": [list(map(str, p)) for p in plan]},
        "sustained": {"value": job_flops / (sus_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                      "ms_per_step": sus_ms, "steps": sus_n,
                      "seconds": sus_ms * sus_n / 1e3},
        "clocks": clk, "gpu_launches": n_launch * steps,
        "checksums": sums,
    }
    if rank == 0:
        rec_out["roofline"] = roofline(wl, prec, fam, ms, sus_ms, rate_flops)
        rec_out["step_kernels_ms"] = {k: round(v, 4) for k, v in sorted(fam.items())}
        if acc_rec is not None:
            rec_out["accuracy"] = acc_rec
        if e2e is not None:
            rec_out["e2e"] = e2e
        if gather is not None:
            rec_out["gather"] = gather
        if with_cpu:
            rec_out["cpu_baseline"] = cpu_baseline(wl) if world == 1 else {
                "value": None, "unit": "GFLOP/s", "cores": None, "kind": "reference",
                "sample": "timed in the N=1 run only"}
    return rec_out


def _round_bf16(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(
        torch.bfloat16).float().numpy()


def _round_tf32(x):
    """Round to nearest even at 10 mantissa bits (b200_pack_operand kind 1)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.int32).astype(np.int64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & ~0x1FFF
    return u.astype(np.uint32).view(np.float32).reshape(np.shape(x))


def accuracy(wl, prec, host, out_dev, samples=64):
    """Sampled accuracy of one application of the nest (mm and conv).

    ``host``: the untouched host inputs; ``out_dev``: the device output after
    one run.  exact: the reference's chain (one f32 multiply and one f32 add
    per MAC, reduction in nest order) recomputed with numpy float32 ops —
    counts bit-identical samples.  bf16 / tf32: float64 sums of the rounded
    operands; max_norm_err = max |got - want| / (2^-24 sqrt(K) sum|ab|), the
    tests' bound is 8 (tests/tcbound.py).  f32x3: the same normalised error
    against unrounded operands."""
    if wl.name not in ("mm", "conv"):
        return None
    f32 = np.float32
    arr = [np.frombuffer(b.data, dtype=f32).reshape(b.shape) for b in host]
    rng = np.random.default_rng(12345)
    out = out_dev.view(-1)
    if wl.name == "mm":
        A, B, C0 = arr
        M, K = A.shape
        N = B.shape[1]
        ii, jj = rng.integers(0, M, samples), rng.integers(0, N, samples)
        a, b, c0 = A[ii, :], B[:, jj].T, C0[ii, jj]
        flat = ii * N + jj
    else:
        X, W, O0 = arr
        nb, fo, ho, wo = O0.shape
        _, C, KH, KW = W.shape
        n_, f_, h_, w_ = (rng.integers(0, e, samples) for e in (nb, fo, ho, wo))
        # operands in the reference's reduction order (ci, ki, kj)
        a = np.stack([X[n_[s], :, h_[s]:h_[s] + KH, w_[s]:w_[s] + KW].reshape(-1)
                      for s in range(samples)])
        b = np.stack([W[f_[s]].reshape(-1) for s in range(samples)])
        c0 = O0[n_, f_, h_, w_]
        flat = ((n_ * fo + f_) * ho + h_) * wo + w_
        K = C * KH * KW
    import torch

    got = out[torch.from_numpy(flat).to(out.device)].cpu().numpy().astype(np.float64)
    if prec == "exact":
        acc = c0.astype(f32).copy()
        for k in range(a.shape[1]):
            acc = (acc + (a[:, k] * b[:, k]).astype(f32)).astype(f32)
        same = int((acc.astype(np.float64) == got).sum())
        return {"samples": samples, "bit_identical": same,
                "check": "reference f32 chain (mul, add per MAC in nest order) on sampled "
                         "outputs of one run"}
    rnd = {"bf16": _round_bf16, "tf32": _round_tf32}.get(prec, lambda x: x)
    ra, rb = rnd(a).astype(np.float64), rnd(b).astype(np.float64)
    prod = ra * rb
    want = c0.astype(np.float64) + prod.sum(axis=1)
    mag = np.abs(prod).sum(axis=1)
    norm = np.abs(got - want) / (2.0 ** -24 * math.sqrt(K) * mag + 1e-300)
    return {"samples": samples, "K": K, "max_norm_err": float(norm.max()),
            "bound": 8.0,
            "check": ("|got - want| / (2^-24 sqrt(K) sum|ab|) on sampled outputs of one run; "
                      "want = float64 sum of the " +
                      ("unrounded" if prec == "f32x3" else prec + "-rounded") + " operands")}


def _e2e(wl, rank, world, sharded, min_seconds):
    """The same metric through the plugin: host Buffers in, results back."""
    import torch

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import shard
    from staircase.interp import machine

    host = host_inputs(wl.fn)

    def once():
        if sharded:
            return shard.run(wl.module, wl.func, host, rank=rank, world=world)
        machine.run(wl.module, wl.func, host, engine=b2.engine)
        return None

    # warm: plans / JIT kernels, and the host buffers get page-locked on
    # their second staging (runtime.pin_host: reused buffers are pinned)
    for _ in range(2):
        once()
    torch.cuda.synchronize()
    barrier(world)
    n = 0
    t0 = time.perf_counter()
    while n < 3 or time.perf_counter() - t0 < min_seconds:
        res = once()
        n += 1
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / n
    st = b2.engine.last_staging
    h2d, d2h = st.h2d_bytes, st.d2h_bytes
    e2e_ms = max_over_ranks(e2e_ms, world)
    gather = None
    if sharded:
        barrier(world)
        t0 = time.perf_counter()
        got = shard.gather(res)
        torch.cuda.synchronize()
        g_ms = max_over_ranks((time.perf_counter() - t0) * 1e3, world)
        gather = {"ms": g_ms, "bytes_received_per_rank": got,
                  "how": "shard.gather: one NCCL all_gather per output buffer of the batch "
                         "rows, device to device, then D2H of the whole output (timed "
                         "separately, not in value / e2e)"}
    flops = wl.flops if sharded else world * wl.flops
    return {"value": flops / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_ms,
            "runs": n, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "how": ("shard.run" if sharded else "staircase machine.run") +
                   " on host Buffers, B200 engine; H2D of the inputs and D2H of the written "
                   "buffers inside the timed region (per rank)"}, gather


def roofline(wl, prec, fam, ms, sus_ms, rank_flops):
    """The dominant kernel family against its roofline (per-rank work)."""
    peaks, src = load_peaks()
    dom = max(fam, key=fam.get)
    dom_ms = fam[dom]
    family = KERNEL_OF.get(dom, dom)
    share = dom_ms / sum(fam.values()) if sum(fam.values()) else None
    scale = rank_flops / wl.flops
    if wl.bytes is not None:
        achieved = wl.bytes * scale / (dom_ms * 1e-3) / 1e9
        peak, unit, bound = peaks["hbm_gbs"], "GB/s", "hbm"
        peak_source = f"{src} HBM copy bandwidth (MEASURED_PEAKS.json)"
        sus_peak = peak
    elif dom in TENSOR_KERNELS:
        achieved = rank_flops / (dom_ms * 1e-3) / 1e12
        tf = tf32_peak() if prec in ("tf32", "f32x3") else None
        if tf is not None:
            # tf32 ceiling: NVIDIA's nominal dense tf32 rate (1125 TFLOP/s,
            # half the nominal bf16).  MEASURED_PEAKS.json has no tf32
            # figure, cuBLAS tf32 (measured in this run) and half the
            # measured bf16 peak both sit BELOW what our tf32 / f32x3
            # kernels reach (the bf16 figure is power-capped; tf32 draws
            # less power per flop), so neither bounds them; both are shown
            half = peaks["bf16_tflops"] * 0.5
            base = 1125.0
            f = {"tf32": 1.0, "f32x3": 1.0 / 3}[prec]
            peak = base * f
            sus_peak = peak
            per3 = (" / 3 (each fp32-accurate product is 3 tf32 products)"
                    if prec == "f32x3" else "")
            peak_source = (f"nominal dense tf32 1125 TFLOP/s (NVIDIA){per3}; measured in this "
                           f"run: cuBLAS tf32 8192^3 {tf:.1f}, {src} bf16 x 0.5 {half:.1f}")
        else:
            f = {"bf16": 1.0, "tf32": 0.5, "f32x3": 0.5 / 3}[prec]
            peak = peaks["bf16_tflops"] * f
            sus_peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]) * f
            peak_source = {"bf16": f"{src} bf16 dense (MEASURED_PEAKS.json)",
                           "tf32": f"{src} bf16 x 0.5 (tf32 = half rate, derived)",
                           "f32x3": f"{src} bf16 x 0.5 / 3 (derived: each fp32-accurate product "
                                    f"is 3 tf32 products at half the bf16 rate)"}[prec]
        unit, bound = "TFLOP/s", "tensor"
        tcb = getattr(wl, "tc_fused_bytes", None) if dom == "b200_conv2d_tc_fused" else \
            wl.tc_bytes
        if tcb and tcb * scale / (dom_ms * 1e-3) / 1e9 / peaks["hbm_gbs"] > \
                achieved / peak:
            # the conv's f32 output read-modify-write makes it HBM-bound
            achieved = tcb * scale / (dom_ms * 1e-3) / 1e9
            peak, unit, bound = peaks["hbm_gbs"], "GB/s", "hbm"
            sus_peak = peak
            peak_source = (f"{src} HBM copy bandwidth (MEASURED_PEAKS.json); algorithmic bytes "
                           + ("= f32 NCHW input + 2 x f32 output" if dom == "b200_conv2d_tc_fused"
                              else "= NHWC bf16 input + 2 x f32 output"))
    else:
        # the bit-exact kernels issue a separate, individually rounded
        # multiply and add per MAC (no FMA: the reference rounds each op), so
        # their ceiling is one FP32 op per lane per cycle, half the FMA peak
        achieved = rank_flops / (dom_ms * 1e-3) / 1e12
        peak = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        sus_peak = peak
        unit, bound = "TFLOP/s", "fp32-simt (no FMA)"
        peak_source = ("derived: 148 SM x 128 FP32 lanes x sm_max_mhz x 1 flop (mul and add "
                       "issued separately: the reference rounds each op; the FMA peak is 2x)")
    # the whole step under sustained load against the sustained peak
    step_sus = (achieved * (dom_ms / (sus_ms * (share or 1.0))) if share else None)
    return {"bound": bound, "kernel": dom, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "peak_source": peak_source, "kernel_ms": dom_ms,
            "share_of_step": share,
            "frac_sustained": (step_sus / sus_peak) if step_sus else None,
            "sustained_peak": sus_peak,
            "traffic": load_traffic(f"{wl.name}_{family}_{prec}")}


# -- the sweep (configs[4]) -------------------------------------------------------

SWEEP_T = [1, 2, 4, 8, 16, 32, 64, 128]
SWEEP_U = [1, 2, 4, 8]
SWEEP_WEIGHTS = (1, 1)


def measure_sweep(rank, world, prec="exact", with_cpu=True):
    """The paper's tile-size / unroll design-space sweep (BASELINE configs[4]).

    512 configurations = tiles T x T (T in 1..128) x unroll U (1, 2, 4, 8) on
    two targets — the matmul nest (parallel form, 1024^3) and the paper's
    conv (1,1,1280,1280)*(1,3,3) — each enumerated exhaustively after the
    identity trial (strategy "grid").  sweep.search_many splits the ranks
    into one group per target (equal: the targets' trials take the same host
    time);
    inside a group trials are sharded idx % group size; all_gather_object of
    the trial records per group, then of the per-target results.  value =
    trials / wall time, max over ranks — every rank's setup (inputs, identity
    baseline) and the gathers included, so the scaling it reports is end to
    end.  A 2-trial warm-up search runs first (engine paths, CUDA context).
    """
    import torch

    import paper_2307_16080_b200 as b2
    from paper_2307_16080_b200 import runtime as b2rt
    from paper_2307_16080_b200 import sweep
    from staircase.tuner import ParamSpace

    space = ParamSpace(tile_sizes=(SWEEP_T, SWEEP_T), unroll_factors=SWEEP_U)
    targets = [(bk.mm_par1024, 2.0 * 1024 ** 3), (bk.conv_paper, 2.0 * 1280 * 1280 * 9)]
    b2.configure(precision=prec)
    t0_totals = dict(b2rt.TOTALS)
    budget = 1 + len(SWEEP_T) ** 2 * len(SWEEP_U)
    for fn, _ in targets:   # warm-up (not timed)
        sweep.search(fn.module, None, space, budget=2, seed=1, strategy="grid", rank=0,
                     world=1)
    torch.cuda.synchronize()
    timing = {}
    barrier(world)
    t0 = time.perf_counter()
    # one rank group per target (sweep.search_many): a rank builds one
    # target's inputs and baseline; equal groups — the two targets' trials
    # took the same host time at N=1 (0.69 / 0.70 s, profiles/r02_sweep_*)
    res = sweep.search_many([fn.module for fn, _ in targets], None, space, budget=budget,
                            seed=0, strategy="grid", weights=SWEEP_WEIGHTS, timing=timing)
    torch.cuda.synchronize()
    wall = max_over_ranks(time.perf_counter() - t0, world)
    trial_s = max_over_ranks(timing.get("trials_s", 0.0), world)
    setup_s = max_over_ranks(timing.get("setup_s", 0.0), world)
    total_trials = sum(len(log) for _, log in res)
    flops = sum(f * len(log) for (_, f), (_, log) in zip(targets, res))
    logs = [(fn.__name__, best, log) for (fn, _), (best, log) in zip(targets, res)]
    groups = sweep.rank_groups(SWEEP_WEIGHTS, world)
    b2.configure(precision="exact")
    moved = {k: b2rt.TOTALS[k] - t0_totals[k] for k in t0_totals}
    if rank != 0:
        return None
    rec = {
        "metric": "configs/s (tile/unroll design-space sweep)",
        "value": total_trials / wall, "unit": "configs/s", "ms_per_step": 1e3 * wall,
        "dtype": DTYPE[prec], "precision": prec,
        "data": "synthetic (tuner make_inputs, seed 0)",
        "config": {"workload": "512-config sweep: tiles T x T (T=1..128) x unroll (1,2,4,8) on "
                               "matmul 1024^3 (parallel form) and conv (1,1,1280,1280)*(1,3,3)",
                   "baseline_config": "configs[4]",
                   "strategy": "grid (identity first)", "trials": total_trials,
                   "parallelism": (f"target groups {groups} (ranks per target), trials "
                                   f"idx % group size inside a group"),
                   "best": {n: {"idx": b.idx, "params": b.params, "cost": b.cost}
                            for n, b, _ in logs}},
        "phases_s_max_rank": {"setup": setup_s, "trials": trial_s, "wall": wall},
        "rank0_per_target_s": {targets[k][0].__name__: {key: round(v, 4) for key, v in t.items()
                                                        if isinstance(v, float)}
                               for k, t in timing.get("per_kernel", {}).items()},
        "trials_only_configs_per_s": total_trials / trial_s,
        "gflops_evaluated_per_s": flops / wall / 1e9,
        "e2e": {"value": total_trials / wall, "unit": "configs/s",
                "h2d_bytes_per_step": moved["h2d_bytes"],
                "d2h_bytes_per_step": moved["d2h_bytes"],
                "how": "each rank draws the seeded inputs on the host (make_inputs), runs the "
                       "baseline through machine.run on host Buffers and uploads the inputs "
                       "once; every trial then runs on device clones of them and is checked on "
                       "the device; setup (inputs + baseline + upload) and the final all-gather "
                       "are inside value, so value already is end to end"},
        "gpu_launches": moved["launches"],
    }
    if with_cpu:
        rec["cpu_baseline"] = reference_sweep_rate() if world == 1 else {
            "value": None, "unit": "configs/s", "cores": None, "kind": "reference",
            "sample": "timed in the N=1 run only"}
    return rec


def reference_sweep_rate(budget=4):
    """Configs/s of the reference tuner on the sweep's own kernels, extrapolated:
    each trial runs the transformed nest once, and the reference executor's
    rate on that nest is measured on a slice with the same loop structure and
    reduction length (matmul: 1x1024x1024; conv: 8 output rows), so
    trial time = kernel flops / slice rate.  Full-size trials would take
    ~25 min (matmul) / ~40 s (conv) each on the CPU executor.  The
    reference's tuner machinery itself (tuner.search on the desk conv,
    budget trials) is run too, to keep the measurement honest about
    overhead.  One core: the tuner is sequential (search.py:180-279)."""
    import importlib

    from staircase.interp import _evalcy, machine
    from staircase.tuner import ParamSpace

    rates = []
    for fn, flops in ((bk.mm_slice1024, 2.0 * 1024 * 1024), (bk.conv_paper_slice,
                                                            2.0 * 8 * 1280 * 9)):
        args = host_inputs(fn)
        _, stats = machine.run(fn.module, fn.__name__, args, engine=_evalcy)
        rates.append(flops / stats.wall_time)
    trial_s = [2.0 * 1024 ** 3 / rates[0], 2.0 * 1280 * 1280 * 9 / rates[1]]
    ref = importlib.import_module("staircase.tuner.search")
    space = ParamSpace(tile_sizes=([1, 2, 4, 8, 16], [1, 2, 4, 8, 16]), unroll_factors=(1, 2, 4))
    saved = machine._engine
    machine._engine = _evalcy
    try:
        t0 = time.perf_counter()
        ref.search(bk.conv_desk_small.module, None, space, budget=budget, seed=0)
        desk = (time.perf_counter() - t0) / budget
    finally:
        machine._engine = saved
    per_config = statistics.mean(trial_s) + desk
    return {"value": 1.0 / per_config, "unit": "configs/s", "cores": 1, "kind": "reference",
            "sample": (f"reference executor (_evalcy) slice rates {rates[0] / 1e6:.2f} / "
                       f"{rates[1] / 1e6:.2f} MFLOP/s on the matmul / conv nests -> "
                       f"extrapolated {trial_s[0]:.0f} s / {trial_s[1]:.1f} s per trial, + "
                       f"tuner overhead {desk * 1e3:.0f} ms/trial (tuner.search on the desk "
                       f"conv; the tuner is sequential)")}


# -- the line ---------------------------------------------------------------------

def headline(rec, world, steps, warmup):
    line = dict(rec)
    line.update({"n_gpus": world, "steps": steps, "warmup": warmup, "higher_is_better": True,
                 "vs_baseline": None, "data": rec.get("data", "synthetic")})
    return line


def run_ours(args, rank, world, local):
    auto = args.workload == "auto"
    name = ("mm" if world == 1 else "conv") if auto else args.workload
    k = dict(steps=args.steps, warmup=args.warmup, min_seconds=args.min_seconds)
    if name == "sweep":
        main_rec = measure_sweep(rank, world, args.precision or "exact")
        main_wl = None
    else:
        tiles = tuple(int(x) for x in args.tiles.split("x")) if args.tiles else None
        main_wl = Workload(name, tiles)
        main_rec = measure(main_wl, args.precision or "exact", rank, world, local, **k)
    variants, configs = {}, {}
    if auto:
        if world == 1:
            for prec, tiles in (("f32x3", None), ("bf16", None), ("tf32", None),
                                ("bf16", (8, 8)), ("bf16", (4, 16)), ("exact", (8, 8)),
                                ("exact", (4, 16))):
                wl = Workload("mm", tiles)
                r = measure(wl, prec, rank, world, local, with_cpu=False, **k)
                if r is not None:
                    variants[f"{wl.key}_{prec}"] = r
            todo = [("linear32", "exact"), ("conv", "exact"), ("conv", "bf16"), ("ls", "bf16"),
                    ("ls", "f32x3"), ("ls", "exact"), ("ewise", "exact")]
        else:
            todo = [("conv", "bf16"), ("ls", "bf16")]
        cpu = {}
        for wname, prec in todo:
            wl = Workload(wname)
            r = measure(wl, prec, rank, world, local, with_cpu=wname not in cpu, **k)
            if r is not None and rank == 0:
                if "cpu_baseline" in r:
                    cpu[wname] = r["cpu_baseline"]
                else:
                    r["cpu_baseline"] = cpu[wname]
                configs[f"{wname}_{prec}"] = r
        sw = measure_sweep(rank, world)
        if sw is not None:
            configs["sweep"] = sw
    if rank != 0:
        return
    line = headline(main_rec, world, args.steps, args.warmup)
    line["scaling"] = "strong" if (main_wl is None or (main_wl.sharded and world > 1)) \
        else "weak"
    if main_wl is not None and main_wl.name == "mm" and world == 1:
        main_rec_cpu = line.get("cpu_baseline")
        for v in variants.values():
            v["cpu_baseline"] = main_rec_cpu
    if variants:
        line["variants"] = variants
    if configs:
        line["configs"] = configs
    print(json.dumps(line), flush=True)


# -- the reference arm -------------------------------------------------------------

def run_reference(args, rank, world):
    """The reference's own CPU implementation (baseline/_ref, _evalcy) on the
    arm's config: a bounded slice per step in one process per host core."""
    if rank != 0:
        return
    auto = args.workload == "auto"
    name = ("mm" if world == 1 else "conv") if auto else args.workload
    if name == "sweep":
        vals = [reference_sweep_rate() for _ in range(max(1, min(args.steps, 3)))]
        rec = vals[0]
        value = statistics.median(v["value"] for v in vals)
        print(json.dumps({
            "impl": "reference", "metric": "configs/s (tile/unroll design-space sweep)",
            "value": value, "unit": "configs/s", "n_gpus": world, "steps": len(vals),
            "warmup": args.warmup, "ms_per_step": 1e3 / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "reference tuner trials (extrapolated from slices)"},
            "cpu_baseline": dict(rec, value=value),
            "e2e": {"value": value, "unit": "configs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return
    wl = Workload(name)
    prec = args.precision or "exact"
    pool = ReferencePool(wl)
    try:
        for _ in range(args.warmup):
            pool.sample()
        rates, per = [], []
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r, t = pool.sample()
            rates.append(r)
            per.append(t)
        wall = time.perf_counter() - t0
    finally:
        pool.close()
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": f"GFLOP/s ({wl.key}, {prec})", "value": value,
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "strong" if wl.sharded and world > 1 else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl.desc + " (reference CPU executor on a slice per core; rate "
                                         "extrapolates)", "baseline_config": wl.config},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": pool.cores,
                         "kind": "reference", "sample": pool.describe(statistics.median(per))},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="auto",
                    choices=["auto", "mm", "conv", "ls", "linear32", "ewise", "sweep"])
    ap.add_argument("--tiles", default=None, help="e.g. 8x8: the mm nest tiled by the "
                                                  "reference pass (parallel form)")
    ap.add_argument("--precision", default=None, choices=["bf16", "tf32", "f32x3", "exact"])
    ap.add_argument("--min-seconds", type=float, default=1.0,
                    help="length of the sustained and e2e timed regions")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3   # the contract's minimum warm-up
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
