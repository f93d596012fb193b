"""Device runtime: the libb200k.so binding, buffer staging, launch recording.

PyTorch is used only as the device allocator / stream provider.  All
compute goes through the C ABI in include/b200k.h, loaded with ctypes from
the in-tree shared object built by paper_2307_16080_b200/build.py.  There is
no CPU fallback: if the library or a GPU is missing, every entry point
raises.

Every C-ABI launch goes through ``DeviceBackend.call`` so a run can be
*recorded* (the exact launch sequence the engine chose for a module, with
its device pointers) and replayed — directly or as a CUDA graph — without
re-planning; bench.py uses this for device-resident timing.
"""
from __future__ import annotations

import ctypes
import math
import os
import weakref

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("B200_LIB") or os.path.join(_PKG, "libb200k.so")   # dev: A/B builds

_lib = None


class BackendUnavailable(RuntimeError):
    """The CUDA backend cannot run here (no library or no B200)."""


class B200Buffer(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("shape", ctypes.c_int64 * 8),
                ("strides", ctypes.c_int64 * 8)]


class B200VmError(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("slot", ctypes.c_int32),
                ("index", ctypes.c_int64), ("extent", ctypes.c_int64),
                ("loc", ctypes.c_int64)]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F32 = ctypes.c_float

SIGNATURES = {
    "b200_mt_uniform": [_P, _P, _I64, ctypes.c_double, ctypes.c_double, _P, _I32],
    "b200_copy2d": [_P, _I64, _P, _I64, _I64, _I64, _I32, _P],
    "b200_guard_close": [_I32, _P, _P, _I64, ctypes.c_double, ctypes.c_double, _P, _P],
    "b200_vm_run": [_P, _I32, _P, _P, _I32, _I32, _P, _I32, _I32, _P, _P, _P, _P,
                    _I32, _P, _P, _P],
    "b200_gemm_f32_exact": [_P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _I64,
                            _I64, _I64, _I32, _F32, _P, _I64, _P],
    "b200_gemm_f32_exact_tiled": [_P, _I64, _I64, _P, _I64, _I64, _P, _I64, _I64, _I64,
                                  _I64, _I64, _I32, _F32, _P, _I64, _I32, _I32, _P],
    "b200_contract_exact": [_I32, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64,
                            _I32, _I32, _I32, ctypes.c_double, _P, _I64, _P],
    "b200_pack_operand": [_I32, _P, _I64, _I64, _P, _I64, _I64, _P],
    "b200_map_f32": [_P, _I32, _P, _I32, _P, _P, _I32, _P, _I32, _I32, _I32, _P],
    "b200_gemm_tc": [_I32, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I32, _F32, _P,
                     _I64, _I32, _I32, _P],
    "b200_gemm_tc_shadow": [_I32, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I32, _F32, _P,
                            _I64, _P, _I64, _P],
    "b200_gemm_tc_kn": [_I32, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I32, _F32, _P,
                        _I64, _P, _I64, _P],
    "b200_pack_conv_input": [_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _P],
    "b200_pack_conv": [_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _I64, _I64, _I64,
                       _P],
    "b200_pack_conv_weight": [_P, _P, _P, _I64, _I64, _I64, _I64, _I64, _P],
    "b200_conv2d_tc_fused": [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64,
                             _I64, _I32, _F32, _P],
    "b200_conv2d_tc": [_P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _I64,
                       _I32, _F32, _P],
    "b200_conv2d_exact": [_I32, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _I64, _I64,
                          _I64, _I64, _I64, _I32, ctypes.c_double, _P],
    "b200_jit_compile": [ctypes.c_char_p, ctypes.c_char_p, _P],
    "b200_jit_cubin": [ctypes.c_char_p, _P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)],
    "b200_jit_load": [ctypes.c_char_p, ctypes.c_char_p, _P],
    "b200_jit_launch": [_P, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                        ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32,
                        _P, _P],
}


def load_library(path=LIB_PATH):
    """Load libb200k.so and declare every exported C-ABI symbol."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise BackendUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a)")
    lib = ctypes.CDLL(path)
    for name, argtypes in SIGNATURES.items():
        fn = getattr(lib, name, None)
        if fn is None and os.environ.get("B200_LIB"):
            continue   # dev A/B against an older build: entry point absent there
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = ctypes.c_int
    lib.b200_jit_log.argtypes = []
    lib.b200_jit_log.restype = ctypes.c_char_p
    _lib = lib
    return lib


def torch_mod():
    import torch

    if not torch.cuda.is_available():
        raise BackendUnavailable("no CUDA device: the B200 engine has no CPU fallback")
    return torch


def check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed with status {rc}")


_TORCH_DT = {"f32": "float32", "f64": "float64", "i32": "int32", "i64": "int64"}
DT_CODE = {"f32": 0, "f64": 1, "i32": 2, "i64": 3}


_PINNED = {}              # id(array) -> (address, nbytes) of page-locked Buffer storage
_STAGED_ONCE = {}         # id(array) -> address: staged before, not (yet) pinned
PIN_MIN_BYTES = 1 << 20


def _unpin(key, addr):
    _PINNED.pop(key, None)
    try:
        torch_mod().cuda.cudart().cudaHostUnregister(addr)
    except Exception:   # interpreter shutdown / context already gone
        pass


def pin_host(arr, host):
    """Page-lock a Buffer's storage (``array.array``) in place, once.

    The reference mutates memref Buffers in place, so their storage is the
    staging source and destination of every run; registering it with the
    driver (cudaHostRegister) turns each copy into a direct DMA instead of a
    bounce through a pageable staging buffer.  The registration lives as long
    as the array (weakref finalizer).  Registration costs milliseconds, so
    an array is pinned the second time it is staged (it is being reused
    across runs); one-shot buffers — e.g. a tuner trial's fresh inputs —
    are copied unpinned.  B200_PIN=0 disables it.
    """
    nbytes = host.numel() * host.element_size()
    if nbytes < PIN_MIN_BYTES or os.environ.get("B200_PIN", "1") == "0":
        return
    key, addr = id(arr), host.data_ptr()
    if _PINNED.get(key) == (addr, nbytes):
        return
    if _STAGED_ONCE.get(key) != addr:
        if key not in _STAGED_ONCE:
            weakref.finalize(arr, _STAGED_ONCE.pop, key, None)
        _STAGED_ONCE[key] = addr
        return
    if key in _PINNED:   # storage moved (resized array): drop the stale range
        _unpin(key, _PINNED[key][0])
    torch = torch_mod()
    if int(torch.cuda.cudart().cudaHostRegister(addr, nbytes, 0)) != 0:
        return
    _PINNED[key] = (addr, nbytes)
    weakref.finalize(arr, _unpin, key, addr)


class Staging:
    """Device copies of the host Buffers touched by a run (or a Session).

    Memref arguments are mutated in place in the reference (SPEC: memref
    reference semantics), so every buffer a region writes is copied back
    into the caller's ``array.array`` when the run ends (or faults).
    """

    def __init__(self):
        self.torch = torch_mod()
        self.lib = load_library()
        self.dev = {}        # id(Buffer) -> (Buffer, tensor)
        self.dirty = set()
        self.stream = self.torch.cuda.current_stream()
        self.h2d_bytes = 0   # host <-> device traffic of this staging (bench e2e)
        self.d2h_bytes = 0
        self.panels = 0      # row panels run with pipelined copies (stream_rows)
        self._wb_event = None   # last streamed write-back (see stream_rows)
        # batch shards (shard.py): id(Buffer) -> (r0, r1), the leading-dim rows
        # this rank owns; only those rows are copied in and out
        self.rows = {}

    @property
    def stream_ptr(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def host(self, buf):
        return self.torch.frombuffer(buf.data, dtype=getattr(self.torch, _TORCH_DT[buf.dtype]))

    def adopt(self, buf, tensor):
        """Use ``tensor`` (same dtype and element count) as the device copy of
        ``buf``: nothing is uploaded (sweep trials start from device clones
        of resident inputs)."""
        self.dev[id(buf)] = (buf, tensor)

    def staged(self, buf):
        ent = self.dev.get(id(buf))
        return ent is not None and ent[0] is buf

    def tensor(self, buf, overwrite=False):
        """The device copy of ``buf`` (uploaded on first use).  ``overwrite``:
        the caller's kernel writes every element before reading any, so a
        first use allocates without copying the host contents."""
        ent = self.dev.get(id(buf))
        if ent is None or ent[0] is not buf:
            host = self.host(buf)
            rows = self.rows.get(id(buf))
            if overwrite:
                t = self.torch.empty_like(host, device="cuda")
            elif rows is not None:
                # a batch shard: this rank's rows only (the rest is never read)
                pin_host(buf.data, host)
                t = self.torch.empty_like(host, device="cuda")
                h, d = self._row_views(buf, host, t, rows)
                d.copy_(h)
                self._count(h2d=h.numel() * h.element_size())
            else:
                pin_host(buf.data, host)
                # asynchronous on the current stream: the Buffer's storage
                # outlives the run and is only written by the final flush
                # (pageable storage is staged by the driver before it returns)
                t = host.to("cuda", non_blocking=True)
                self._count(h2d=host.numel() * host.element_size())
            ent = (buf, t)
            self.dev[id(buf)] = ent
        return ent[1]

    @staticmethod
    def _row_views(buf, host, dev, rows):
        """The (host, device) views of leading-dim rows [r0, r1) of buf."""
        r = buf.shape[0]
        r0, r1 = rows
        return host.view(r, -1)[r0:r1], dev.view(r, -1)[r0:r1]

    def mark_dirty(self, buf):
        self.dirty.add(id(buf))

    def _count(self, h2d=0, d2h=0):
        self.h2d_bytes += h2d
        self.d2h_bytes += d2h
        TOTALS["h2d_bytes"] += h2d
        TOTALS["d2h_bytes"] += d2h

    def flush(self):
        torch = self.torch
        if self._wb_event is not None:
            # streamed write-backs first: a buffer written again after its
            # streamed write-back is copied below, and must land last
            torch.cuda.current_stream().wait_event(self._wb_event)
        for key in list(self.dirty):
            if key not in self.dev:
                continue   # marked but never staged: the device never touched it
            buf, t = self.dev[key]
            host = self.host(buf)
            rows = self.rows.get(key)
            if rows is not None:
                host, t = self._row_views(buf, host, t, rows)
            host.copy_(t)
            self._count(d2h=host.numel() * host.element_size())
        self.dirty.clear()
        torch.cuda.current_stream().synchronize()
        if self._wb_event is not None:
            self._wb_event.synchronize()
            self._wb_event = None

    def stream_rows(self, panels, ins, out, launch, written_back=True, rows=None,
                    concurrent=1):
        """Run ``launch(r0, r1)`` over row panels with the host copies overlapped.

        The row-major buffers in ``ins`` (uploaded, panel by panel, on a copy
        stream) and ``out`` (``(buf, upload)``: the output, uploaded first
        unless the kernel overwrites it, and written back panel by panel on a
        second copy stream) are split along their leading dimension; panel
        p's kernels wait only for panel p's uploads, and panel p's write-back
        overlaps the uploads and kernels of the panels after it (PCIe is full
        duplex: both directions run at once).  Every buffer ends staged
        (registered in ``dev``); later regions do not wait for the
        write-backs (a chained layer's write-back of its output overlaps the
        next layer), flush() does.  ``panels``: [(r0, r1)] covering the leading dimension
        (or ``rows`` equal slices of every buffer's flat storage); they may
        cover a sub-range of the rows (a batch shard's).  ``concurrent`` > 1:
        panel kernels go round-robin to that many side streams, so the small
        grids of consecutive panels share the GPU (compute-bound kernels
        whose panel grids are under a wave); rows of different panels are
        disjoint, so they may run in any order.
        """
        torch = self.torch
        cur = torch.cuda.current_stream()
        if STREAM_TRACE is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(cur)
            STREAM_TRACE.append(("stream_rows entry (current stream)", e))
        up, down = _copy_streams(torch)
        up.wait_stream(cur)     # device storage may be recycled from earlier kernels
        comp = _compute_streams(torch, concurrent) if concurrent > 1 else [cur]
        for cs in comp:
            if cs is not cur:
                cs.wait_stream(cur)
        obuf, oup = out
        lead = rows
        rows = rows or obuf.shape[0]
        views = []
        for buf in ins + [obuf]:
            host = self.host(buf)
            pin_host(buf.data, host)
            t = torch.empty_like(host, device="cuda")
            self.dev[id(buf)] = (buf, t)
            r = lead or buf.shape[0]
            views.append((host.view(r, -1), t.view(r, -1)))
        hin, (ho, to) = views[:-1], views[-1]
        esz = to.element_size()
        tr = STREAM_TRACE

        def mark(stream, what):
            if tr is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                tr.append((what, e))

        for p, (r0, r1) in enumerate(panels):
            mark(up, f"h2d{p}<")
            with torch.cuda.stream(up):
                for (h, t) in hin + ([(ho, to)] if oup else []):
                    t[r0:r1].copy_(h[r0:r1], non_blocking=True)
                    self._count(h2d=(r1 - r0) * t.shape[1] * esz)
            mark(up, f"h2d{p}>")
            ev = torch.cuda.Event()
            ev.record(up)
            cs = comp[p % len(comp)]
            cs.wait_event(ev)
            mark(cs, f"k{p}<")
            with torch.cuda.stream(cs):
                launch(r0, r1)
            mark(cs, f"k{p}>")
            self.panels += 1
            if written_back:
                done = torch.cuda.Event()
                done.record(cs)
                down.wait_event(done)
                mark(down, f"d2h{p}<")
                with torch.cuda.stream(down):
                    ho[r0:r1].copy_(to[r0:r1], non_blocking=True)
                mark(down, f"d2h{p}>")
                self._count(d2h=(r1 - r0) * to.shape[1] * esz)
        assert panels[-1][1] <= rows
        for cs in comp:
            if cs is not cur:
                cur.wait_stream(cs)
        if written_back:
            # later kernels do not wait for the write-backs: they only read
            # these rows, or write rows whose buffer is written back again
            # after them (a later writer keeps it dirty, or streams its own
            # write-back behind these on the same stream); flush() orders its
            # copies after this event
            self._wb_event = torch.cuda.Event()
            self._wb_event.record(down)

    def buffer_table(self, buffers):
        """A device array of b200_buffer for the given host Buffers."""
        table = (B200Buffer * len(buffers))()
        for k, b in enumerate(buffers):
            t = self.tensor(b)
            table[k].ptr = t.data_ptr()
            table[k].dtype = DT_CODE[b.dtype]
            table[k].rank = len(b.shape)
            for d, (s, st) in enumerate(zip(b.shape, b.strides)):
                table[k].shape[d] = s
                table[k].strides[d] = st
        return self.upload_bytes(bytes(table))

    def upload_bytes(self, blob):
        torch = self.torch
        host = torch.frombuffer(bytearray(blob), dtype=torch.uint8) if blob else \
            torch.zeros(1, dtype=torch.uint8)
        return host.to("cuda", non_blocking=False)

    def upload_i32(self, values):
        return self.upload_bytes(np.asarray(values, dtype=np.int32).tobytes())

    def upload_i64(self, values):
        return self.upload_bytes(np.asarray(values, dtype=np.int64).tobytes())


# process-wide counters (bench.py's sweep line): entry-point calls made by
# DeviceBackend (one kernel launch each, or a fixed few for the packing
# entry points) and host <-> device bytes staged
TOTALS = {"launches": 0, "h2d_bytes": 0, "d2h_bytes": 0}

_COPY_STREAMS = {}


_COMPUTE_STREAMS = {}


def _compute_streams(torch, k):
    """k side streams of the current device for concurrent panel kernels."""
    key = (torch.cuda.current_device(), k)
    if key not in _COMPUTE_STREAMS:
        _COMPUTE_STREAMS[key] = [torch.cuda.Stream() for _ in range(k)]
    return _COMPUTE_STREAMS[key]


def _copy_streams(torch):
    """(upload, write-back) side streams of the current device."""
    dev = torch.cuda.current_device()
    if dev not in _COPY_STREAMS:
        _COPY_STREAMS[dev] = (torch.cuda.Stream(), torch.cuda.Stream())
    return _COPY_STREAMS[dev]


# exact: per-op f32 rounding on the FP32 pipes (bit-identical to the
# reference); f32x3: fp32-accurate on the tensor cores (3xTF32 split, within
# the fp32 tolerance, not bit-identical); tf32 / bf16: rounded operands.
PRECISIONS = ("exact", "f32x3", "tf32", "bf16")
TC_PRECISIONS = ("bf16", "tf32", "f32x3")
_WORKSPACE = {}
_RETIRED = []


def workspace(slot, dtype, rows, cols):
    """Device scratch for packed tensor-core operands: one growable buffer
    per (slot, dtype, device), returned as a rows x cols view of its front.

    A buffer too small for a request is replaced by one of max(need, 2 x old)
    elements, so a process that sees many shapes (streamed panels, conv
    packs per image count, tuner trials) holds at most ~2x the largest
    request per slot instead of one buffer per shape.  Replaced buffers are
    retired, not freed: a Recording may still point into them (their total
    is bounded by the geometric growth)."""
    torch = torch_mod()
    key = (slot, dtype, torch.cuda.current_device())
    need = max(1, rows * cols)
    t = _WORKSPACE.get(key)
    if t is None or t.numel() < need:
        if t is not None:
            _RETIRED.append(t)
        size = need if t is None else max(need, 2 * t.numel())
        t = torch.empty(size, dtype=getattr(torch, dtype), device="cuda")
        _WORKSPACE[key] = t
    return t[:rows * cols].view(rows, cols)


def tc_supported(precision, K):
    """tcgen05 path needs 16-byte TMA rows of packed K (bf16: K%8, tf32 and
    f32x3 — 3K tf32 values per row — K%4)."""
    return precision in TC_PRECISIONS and K > 0 and \
        (K * (2 if precision == "bf16" else 4)) % 16 == 0


def conv_tc_supported(cv):
    """The tcgen05 conv kernel (csrc/conv_tc.cu): F in {32, 64, 128}, weights
    resident in shared memory next to >= 2 halo-patch stages; any output strides."""
    cp = -(-cv.c // 64) * 64
    if cv.f not in (32, 64, 128) or cv.wo + cv.kw - 1 > 256:   # pack kernel: W <= 256
        return False
    merged = (cv.kw == 3 and cv.f in (32, 64)) or (cv.kw == 5 and cv.f == 32)   # conv_merge
    if merged:   # tile 4 x 28, patch rows of 32 pixels
        ph, prow = 4 + cv.kh - 1, 32
    else:        # tile 16 x 8, patch rows of 8 + kw - 1 pixels
        ph, prow = 16 + cv.kh - 1, 8 + cv.kw - 1
    patch = -(-(ph * prow * 128) // 1024) * 1024
    smem = 1024 + cv.kh * cv.kw * (cp // 64) * cv.f * 128 + 2 * patch + 256
    return smem <= 232448 and ph <= 256 and prow <= 256


# The fused conv reads and converts the f32 input inside the conv kernel;
# its shared memory (resident weights + staged output blocks + bf16 patches +
# raw f32 chunks) leaves two patch stages, so a row band's conversion cannot
# overlap the previous band's MMAs: at ResNet's N = 256 it is 160 us against
# 152 for pack + conv (tools/probe_conv_fused.py), while small batches, where
# the separate pack launch's fixed cost dominates, gain 15-30 % (nb 4: 13 vs
# 17 us, nb 8: 14.5 vs 17.3; nb 16: 21.2 vs 19.8, the crossover).  It
# therefore takes batches up to this size.
FUSED_CONV_MAX_IMAGES = int(os.environ.get("B200_CONV_FUSED_MAX", "8"))


def conv_tc_fused_ok(cv):
    """b200_conv2d_tc_fused applies (mirrors csrc/conv_tc.cu's checks): the
    merged 3x3 tiling (F 32 / 64), C <= 64, at most two 28-column tiles per
    row band (W - 2 <= 56, the band's rows are one TMA box), dense NCHW planes
    (unit w stride, rows back to back, 16-byte channel / image strides),
    even H and W, and shared memory for the
    weights, two patch stages and four raw chunks (one per converter warp;
    one TMA box over row pairs per 8 channels: H and W even).  B200_CONV_UNFUSED=1 forces the repack
    path (A/B)."""
    if os.environ.get("B200_CONV_UNFUSED") == "1":
        return False
    if not (cv.kw == 3 and cv.f in (32, 64)) or cv.nb > FUSED_CONV_MAX_IMAGES:
        return False
    st = cv.inp.strides
    if st[3] != 1 or st[2] != cv.wp or st[1] % 4 or st[0] % 4 or cv.hp * cv.wp >= 2 ** 31:
        return False
    ph, prow = 4 + cv.kh - 1, 32
    blen = 2 * cv.wp                           # whole row pairs per 8-channel chunk
    if cv.hp % 2 or cv.wp % 2 or blen > 256 or cv.c > 64 or -(-cv.wo // 28) > 2:
        return False
    raw = 8 * ((ph + 1) // 2) * blen * 4
    cp = -(-cv.c // 64) * 64
    patch = -(-(ph * prow * 128) // 1024) * 1024
    smem = 1024 + cv.kh * cv.kw * (cp // 64) * cv.f * 128 + 2 * patch + 4 * raw + 512
    return smem <= 232448


def conv_exact_supported(cv, esz):
    """The bit-exact direct conv kernel (csrc/conv_exact.cu): reduction in the
    nest order ci -> ki -> kj (its rounding order) and the double-buffered
    staging (8 channels of a 4 x (32 + kw - 1) patch + 8 x kh x kw x 64
    weights) within shared memory."""
    order = [r for r in ("ci", "ki", "kj") if r in cv.k_order]
    if list(cv.k_order) != order:
        return False
    pw = 32 + cv.kw - 1
    pitch = pw + (8 - pw) % 32
    smem = 2 * 8 * ((4 + cv.kh - 1) * pitch + cv.kh * cv.kw * 64) * esz
    return smem <= 227 * 1024


def _direct_call(lib):
    def call(name, *args):
        check(getattr(lib, name)(*args), name)
    return call


def cta_tile(precision, tiles):
    """The CTA tile a tiled matmul nest runs with, from its tile sizes.

    The reference's tiling pass (passes/tiling.py:56-80) splits each output
    loop into a parallel origin loop over tiles and a parallel offset loop
    within one, and its GPU mapping sends the origin loop to blocks and the
    offset loop to threads (passes/gpumap.py:22-34): a tile is the unit of
    work one block owns.  Here a tile (tm, tn) of the M and N loops selects
    the CTA tile shape of the kernel that runs the contraction — by aspect
    ratio tn / tm, and for the SIMT kernel also by area:

      exact:  tm * tn <= 16 -> 64 x 64;  tn / tm >= 2 -> 64 x 256;
              tn / tm <= 1/2 -> 256 x 64;  otherwise 128 x 128
      tcgen05: tn / tm >= 2 -> one CTA, 128 x 256 (cta_group::1);
               otherwise a CTA pair, 256 x 256 (cta_group::2)

    e.g. the reference tile sizes (8, 8) and (4, 16) map to
    128 x 128 / 64 x 256 on the exact kernel and 256 x 256 / 128 x 256 on the
    tensor cores.  Untiled nests (tiles (None, None)) return None: the
    kernel's own size-based choice.  Results never depend on the choice
    (exact: identical k-chains; tensor cores: the same MMA k order per tile).
    """
    tm, tn = tiles if tiles else (None, None)
    if tm is None and tn is None:
        return None
    tm, tn = tm or 1, tn or 1
    if precision in TC_PRECISIONS:
        return (128, 256) if tn >= 2 * tm else (256, 256)
    if tm * tn <= 16:
        return (64, 64)
    if tn >= 2 * tm:
        return (64, 256)
    if tm >= 2 * tn:
        return (256, 64)
    return (128, 128)


class PrecisionFallback(UserWarning):
    """A contraction ran at exact f32 although bf16 / tf32 was requested."""


class PrecisionUnavailable(RuntimeError):
    """configure(strict=True): a requested precision cannot be honoured."""


def launch_gemm(lib, precision, a_ptr, sA, b_ptr, sB, c_ptr, sC, M, N, K, stream,
                init=0, init_value=0.0, bias_ptr=None, bias_stride=0, max_ctas=0,
                variant=0, call=None, a_packed=None, c16=None, b_packed=None, cta=None):
    """Enqueue C (+)= A.B with the kernel chosen by ``precision``.

    Returns the list of kernel names launched (for the launch count).
    exact -> b200_gemm_f32_exact (bit-identical to the reference);
    bf16/tf32 -> b200_pack_operand x2 + b200_gemm_tc (tcgen05).
    a_packed: A already packed (a bf16 shadow, M x K) — its pack is skipped;
    c16: also write C rounded to bf16 (M x N) with b200_gemm_tc_shadow.
    b_packed: B already packed ((tensor, kn) from pack_b) — its pack is skipped.
    cta: (BM, BN) from cta_tile() — the tiled nest's CTA tile, or None.
    """
    call = call or _direct_call(lib)
    P = ctypes.c_void_p
    if not tc_supported(precision, K):
        if cta is not None:
            call("b200_gemm_f32_exact_tiled", P(a_ptr), sA[0], sA[1], P(b_ptr), sB[0], sB[1],
                 P(c_ptr), sC[0], sC[1], M, N, K, init, init_value,
                 P(bias_ptr) if bias_ptr else None, bias_stride, cta[0], cta[1], stream)
            return ["gemm_f32_exact"]
        call("b200_gemm_f32_exact", P(a_ptr), sA[0], sA[1], P(b_ptr), sB[0], sB[1],
             P(c_ptr), sC[0], sC[1], M, N, K, init, init_value,
             P(bias_ptr) if bias_ptr else None, bias_stride, stream)
        return ["gemm_f32_exact"]
    if cta is not None:
        variant = 3 if cta == (128, 256) else 2
    kind = 0 if precision == "bf16" else 1
    dt = "bfloat16" if kind == 0 else "float32"
    split = precision == "f32x3"      # packed rows hold 3 K-segments (gemm_tc.cu)
    KP = 3 * K if split else K
    names = []
    if a_packed is not None:
        Ap = a_packed
    else:
        Ap = workspace(0, dt, M, KP)
        call("b200_pack_operand", 2 if split else kind, P(a_ptr), sA[0], sA[1],
             P(Ap.data_ptr()), M, K, stream)
        names.append("pack_operand")
    if b_packed is not None:
        Bp, kn = b_packed if isinstance(b_packed, tuple) else (b_packed, False)
    else:
        # the MN-major B (b200_gemm_tc_kn) is a CTA-pair-only read: not for
        # the 128 x 256 CTA tile (variants 1 and 3)
        Bp, kn = pack_b(lib, precision, b_ptr, sB, N, K, stream, call,
                        allow_kn=variant not in (1, 3))
        names.append("pack_operand")
    if kn:
        call("b200_gemm_tc_kn", kind, P(Ap.data_ptr()), P(Bp.data_ptr()), P(c_ptr), sC[0], sC[1],
             M, N, K, init, init_value, P(bias_ptr) if bias_ptr else None, bias_stride,
             P(c16.data_ptr()) if c16 is not None else None, N if c16 is not None else 0,
             stream)
        return names + [f"gemm_tc_{precision}"]
    K = KP
    if c16 is not None:
        call("b200_gemm_tc_shadow", kind, P(Ap.data_ptr()), P(Bp.data_ptr()), P(c_ptr), sC[0],
             sC[1], M, N, K, init, init_value, P(bias_ptr) if bias_ptr else None, bias_stride,
             P(c16.data_ptr()), N, stream)
    else:
        call("b200_gemm_tc", kind, P(Ap.data_ptr()), P(Bp.data_ptr()), P(c_ptr), sC[0], sC[1],
             M, N, K, init, init_value, P(bias_ptr) if bias_ptr else None, bias_stride,
             max_ctas, variant, stream)
    return names + [f"gemm_tc_{precision}"]


GEMM_KN = os.environ.get("B200_GEMM_KN", "1") != "0"


def pack_b(lib, precision, b_ptr, sB, N, K, stream, call=None, allow_kn=True):
    """Pack B (K x N, strides sB) for the tensor cores (workspace slot 1).

    Returns (tensor, kn).  bf16 with N-contiguous rows, N a multiple of 64:
    converted in place order (K x N, a plain row conversion) and read MN-major by
    b200_gemm_tc_kn (kn True); otherwise transposed to the K-major N x K
    operand of b200_gemm_tc."""
    call = call or _direct_call(lib)
    kind = 0 if precision == "bf16" else 1
    if precision == "f32x3":
        # B^T as N rows of [hi | lo | hi] (3K tf32 values)
        Bp = workspace(1, "float32", N, 3 * K)
        call("b200_pack_operand", 3, ctypes.c_void_p(b_ptr), sB[1], sB[0],
             ctypes.c_void_p(Bp.data_ptr()), N, K, stream)
        return Bp, False
    if GEMM_KN and allow_kn and kind == 0 and sB[1] == 1 and N % 64 == 0:
        Bp = workspace(1, "bfloat16", K, N)
        call("b200_pack_operand", kind, ctypes.c_void_p(b_ptr), sB[0], sB[1],
             ctypes.c_void_p(Bp.data_ptr()), K, N, stream)
        return Bp, True
    Bp = workspace(1, "bfloat16" if kind == 0 else "float32", N, K)
    call("b200_pack_operand", kind, ctypes.c_void_p(b_ptr), sB[1], sB[0],
         ctypes.c_void_p(Bp.data_ptr()), N, K, stream)
    return Bp, False


# Host-copy pipelining (Staging.stream_rows): only when the streamed bytes
# are worth several panels; each panel ~32 MB of traffic, 2..8 panels.
STREAM_MIN_BYTES = 48 << 20
STREAM_TRACE = None   # dev: a list to collect (label, timed event) of stream_rows
# exact GEMMs stream B by column panels too (B200_STREAM_2D=0: row panels only)
STREAM_2D = os.environ.get("B200_STREAM_2D", "1") != "0"
STREAM_PANEL_BYTES = 32 << 20


def _row_major(buf):
    st, acc = [], 1
    for d in reversed(buf.shape):
        st.append(acc)
        acc *= d
    return tuple(buf.strides) == tuple(reversed(st))


def _gemm_rows(buf, off, s, rows, cols):
    """(r0, r1): the operand is rows r0 .. r1-1 of a row-major buffer whose
    leading-dim rows are ``cols`` elements wide (stride (cols, 1)), else None."""
    if tuple(s) != (cols, 1) or not buf.shape or not _row_major(buf) or cols <= 0:
        return None
    if math.prod(buf.shape[1:]) != cols or off % cols:
        return None
    r0 = off // cols
    if r0 + rows > buf.shape[0]:
        return None
    return r0, r0 + rows


def row_panels(rows, row_bytes, align, count=None):
    total = rows * row_bytes
    if total < STREAM_MIN_BYTES or rows < 2 * align:
        return None
    p = count or max(2, min(8, total // STREAM_PANEL_BYTES))
    p = max(2, min(p, rows // align))
    step = -(-rows // p)
    step = -(-step // align) * align
    return [(r, min(rows, r + step)) for r in range(0, rows, step)]


class Recording:
    """A recorded launch sequence: replayable on the current stream."""

    def __init__(self):
        self.calls = []      # (name, args)
        self.keep = []       # device uploads the recorded args point into

    def replay(self, lib=None):
        lib = lib or load_library()
        torch = torch_mod()
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for name, args in self.calls:
            # the stream is always the last argument of a C-ABI entry point
            check(getattr(lib, name)(*args[:-1], stream), name)

    @property
    def launches(self):
        return len(self.calls)

    def names(self):
        return [n for n, _ in self.calls]


class DeviceBackend:
    """Executes region plans on the B200 through libb200k.so."""

    def __init__(self, staging=None, stream_io=False):
        self.stage = staging or Staging()
        # pipeline the host copies of large first-use plans (engine runs;
        # a Session keeps its buffers resident and writes back on sync())
        self.stream_io = stream_io
        self._keep = None
        self.recording = None    # Recording while recording
        # bf16 shadow of the last tensor-core contraction's C: ((C address, M,
        # N), tensor); valid only for the immediately following contraction
        # (fusion.plan_shadows proves nothing writes C in between).  Two
        # workspace slots alternate so a consumer can also be a producer.
        self._shadow = None
        self._shadow_slot = 0
        self.last_shadow = (False, False)   # (A from a shadow, C shadow written)
        self.last_note = None    # why the last contraction ignored the precision
        self.last_cta = None     # CTA tile the last contraction's tiles selected

    def call(self, name, *args):
        check(getattr(self.stage.lib, name)(*args), name)
        TOTALS["launches"] += 1
        if self.recording is not None:
            self.recording.calls.append((name, args))

    def keep(self, *objs):
        self._keep = objs
        if self.recording is not None:
            self.recording.keep.append(objs)

    def read(self, buf, off):
        v = self.stage.tensor(buf)[off].item()
        return float(v) if buf.dtype[0] == "f" else int(v)

    def write(self, buf, off, v):
        self.stage.tensor(buf)[off] = v
        self.stage.mark_dirty(buf)

    def mark_dirty(self, buf):
        self.stage.mark_dirty(buf)

    def flush(self):
        self.stage.flush()

    def _streaming(self, out, *others):
        """Host-copy pipelining applies: an engine run (not recording), the
        output not yet on the device and not aliasing an operand."""
        return (self.stream_io and self.recording is None and not self.stage.staged(out) and
                all(o is not out for o in others))

    def contract(self, g, precision="exact", init=0, init_value=0.0, bias=None, bias_base=0,
                 bias_stride=0, shadow_out=False, shadow_in=False, last_writer=False):
        """Run a templates.ContractMatch (+ fused init / bias); returns kernel names.

        shadow_out / shadow_in (fusion.plan_shadows): on the bf16 tensor-core
        path, also write C as a bf16 K-major operand / take A from the
        previous contraction's shadow instead of packing it.  last_writer
        (engine.flush_pending): nothing queued after this plan writes C, so
        a write-back streamed here is final and C needs no flush copy.
        """
        s = self.stage
        esz = 4 if g.dtype == "f32" else 8
        self.last_note = self.last_cta = None
        if g.M == 0 or g.N == 0:
            # no outputs: an empty batch shard (shard.py gives ranks past the
            # batch no rows, as the reference's worksharing chunks do)
            return ["empty"]
        if bias is None:
            from .templates import conv_view

            cv = conv_view(None, g, dtypes=("f32", "f64"))
            if cv is not None:
                if precision == "bf16" and g.dtype == "f32" and conv_tc_supported(cv):
                    return self.conv_tc(cv, init, init_value, last_writer)
                if g.dtype == "f32" and precision != "exact":
                    self._fallback(precision, "conv shape outside the tcgen05 conv kernel"
                                   if precision == "bf16" else "no tf32 conv kernel")
                if conv_exact_supported(cv, esz):
                    return self.conv_exact(cv, g.dtype, init, init_value, last_writer)
        if g.dtype == "f32" and precision != "exact":
            if not g.strided:
                self._fallback(precision, "index maps are not one strided GEMM")
            elif not tc_supported(precision, g.K):
                self._fallback(precision, f"K={g.K} rows not 16-byte aligned")
        cta = cta_tile(precision if tc_supported(precision, g.K) else "exact",
                       getattr(g, "tiles", None)) if g.strided and g.dtype == "f32" else None
        self.last_cta = cta
        bias_ptr = s.tensor(bias).data_ptr() + esz * bias_base if bias is not None else None
        # C rows [c0, c1) of a row-major buffer of N-wide rows, all staged rows
        # (the whole buffer, or a batch shard's rows)
        crows = _gemm_rows(g.C, g.offC, g.sC, g.M, g.N) if g.strided else None
        dense_c = crows is not None and self._owned(g.C, *crows)
        if (g.strided and g.dtype == "f32" and dense_c and
                self._streaming(g.C, g.A, g.B, bias)):
            stream_a = (not s.staged(g.A) and g.A is not g.B and
                        _gemm_rows(g.A, g.offA, g.sA, g.M, g.K) == crows and
                        self._owned(g.A, *crows))
            # the exact kernels are compute-bound (4096^3: 4.5 ms against
            # 4.7 ms of copies): eight panels, whose sub-wave grids run
            # three at a time on side streams, so the copies hide behind
            # the GEMM; the tensor-core path is copy-bound (default panels)
            exact = not tc_supported(precision, g.K)
            panels = row_panels(g.M, 4 * (g.N * (1 if init else 2) + (g.K if stream_a else 0)),
                                256, count=8 if exact else None)
            if panels is not None:
                panels = [(crows[0] + a, crows[0] + b) for a, b in panels]
                if (exact and stream_a and STREAM_2D and not s.rows and not s.staged(g.B) and
                        g.B is not bias and g.B is not g.A and crows[0] == 0 and
                        _gemm_rows(g.B, g.offB, g.sB, g.K, g.N) == (0, g.K) and
                        self._owned(g.B, 0, g.K) and g.N % 256 == 0):
                    return self._gemm_streamed_2d(g, init, init_value, bias, bias_base,
                                                  bias_stride, last_writer, cta=cta)
                return self._gemm_streamed(g, precision, panels, stream_a, init, init_value,
                                           bias_ptr, bias_stride, shadow_out, shadow_in,
                                           last_writer, cta, crows[0],
                                           concurrent=3 if exact else 1)
        tA, tB = s.tensor(g.A), s.tensor(g.B)
        # a fused fill over all of a dense C: its old contents are never read
        tC = s.tensor(g.C, overwrite=bool(init) and dense_c and g.C is not g.A and
                      g.C is not g.B and g.C is not bias)
        if g.strided and g.dtype == "f32":
            a_packed = c16 = None
            if precision == "bf16" and tc_supported(precision, g.K):
                sh = self._shadow
                if shadow_in and sh is not None and \
                        sh[0] == (tA.data_ptr() + 4 * g.offA, g.M, g.K):
                    a_packed = sh[1]
                if shadow_out and tc_supported(precision, g.N):
                    c16 = workspace(4 + (self._shadow_slot ^ 1), "bfloat16", g.M, g.N)
            names = launch_gemm(s.lib, precision, tA.data_ptr() + 4 * g.offA, g.sA,
                                tB.data_ptr() + 4 * g.offB, g.sB, tC.data_ptr() + 4 * g.offC,
                                g.sC, g.M, g.N, g.K, s.stream_ptr, init=init,
                                init_value=init_value, bias_ptr=bias_ptr,
                                bias_stride=bias_stride, call=self.call, a_packed=a_packed,
                                c16=c16, cta=cta)
            self._shadow = None
            if c16 is not None:
                self._shadow_slot ^= 1
                self._shadow = ((tC.data_ptr() + 4 * g.offC, g.M, g.N), c16)
            self.last_shadow = (a_packed is not None, c16 is not None)
            return names
        return self._contract_tables(g, tA, tB, tC, init, init_value, bias_ptr, bias_stride)

    def _fallback(self, precision, why):
        """A bf16 / tf32 request this contraction cannot honour: it runs the
        exact f32 kernels (more precise, slower).  Warned and noted in the
        plan; configure(strict=True) makes it an error instead."""
        import warnings

        from . import engine

        msg = f"{precision} requested, ran exact f32: {why}"
        self.last_note = msg
        if engine.STRICT:
            raise PrecisionUnavailable(msg)
        warnings.warn(msg, PrecisionFallback, stacklevel=3)

    def _gemm_streamed_2d(self, g, init, init_value, bias, bias_base, bias_stride,
                          last_writer, mpanels=4, npanels=2, concurrent=3, kslices=4,
                          cta=None):
        """Exact C (+)= A.B with A, B and C streamed in blocks: B in column
        panels, A in row panels, C in (row, column) blocks, and each block's
        contraction in `kslices` K slices, so a block's first slice computes
        while the rest of its A rows / B columns upload.  The first launch
        waits for 20 of 192 MiB at 4096^3 (C's first block, a quarter of A's
        first rows and of B's first columns) instead of 56; blocks run three at a
        time on side streams (whole-tile 128 x 128 kernel) while later blocks
        upload and finished ones write back.  A block's slices run in K order
        on one stream, the first with the nest's init (fill value or C), the
        rest continuing from C in memory, the bias on the last: every output
        keeps its full ascending k-chain, bit-identical to the unblocked
        kernel.  Through run() at 4096^3: 6.55 ms per run with whole-K
        blocks, 6.39 with 2 slices, 6.20 with 4 (the copies alone take 4.89;
        tools/gpu/kslice.sh)."""
        s = self.stage
        torch = s.torch
        env = os.environ.get("B200_STREAM_2D_SHAPE")   # dev A/B: "m,n,concurrent[,kslices]"
        if env:
            v = [int(x) for x in env.split(",")]
            mpanels, npanels, concurrent = v[:3]
            kslices = v[3] if len(v) > 3 else kslices
        cur = torch.cuda.current_stream()
        up, down = _copy_streams(torch)
        up.wait_stream(cur)
        comp = _compute_streams(torch, concurrent)
        for cs in comp:
            cs.wait_stream(cur)
        views = {}
        for name, buf in (("A", g.A), ("B", g.B), ("C", g.C)):
            host = s.host(buf)
            pin_host(buf.data, host)
            t = torch.empty_like(host, device="cuda")
            s.dev[id(buf)] = (buf, t)
            views[name] = (host.view(buf.shape[0], -1), t.view(buf.shape[0], -1))
        (hA, tA), (hB, tB), (hC, tC) = views["A"], views["B"], views["C"]
        M, N, K = g.M, g.N, g.K
        ms = -(-M // mpanels)
        ms = -(-ms // 128) * 128
        rows = [(r, min(M, r + ms)) for r in range(0, M, ms)]
        ns = N // npanels // 128 * 128 or N
        cols = [(c, min(N, c + ns) if c + ns < N else N) for c in range(0, N, ns)]
        cols = [(c0, c1) for c0, c1 in cols if c0 < c1]
        if cols[-1][1] < N:
            cols[-1] = (cols[-1][0], N)
        bias_t = s.tensor(bias) if bias is not None else None
        P = ctypes.c_void_p
        esz = 4
        k = 0
        lib = s.lib
        upp = ctypes.c_void_p(up.cuda_stream)
        downp = ctypes.c_void_p(down.cuda_stream)

        def block(dst, src, c0, c1, r0, r1, kind, stream):
            # rows r0..r1-1, columns c0..c1-1 of two N-wide row-major views
            check(lib.b200_copy2d(P(dst.data_ptr() + esz * (r0 * N + c0)), N * esz,
                                  P(src.data_ptr() + esz * (r0 * N + c0)), N * esz,
                                  (c1 - c0) * esz, r1 - r0, kind, stream), "b200_copy2d")

        # the nest's CTA tile (its tile sizes, cta_tile) when the blocks are
        # whole tiles of it, else the 128 x 128 whole-tile kernel
        tm, tn = cta if cta is not None else (128, 128)
        if any((r1 - r0) % tm for r0, r1 in rows) or any((c1 - c0) % tn for c0, c1 in cols):
            tm, tn = 128, 128
        # K slices: multiples of 32 (the whole-tile kernel's stage depth)
        kl = -(-K // kslices)
        kl = -(-kl // 32) * 32
        ks = [(k0, min(K, k0 + kl)) for k0 in range(0, K, kl)]
        a_rows = {}   # A row panel -> K slices uploaded

        def block_a(r0, r1, k0, k1):
            # rows r0..r1-1, columns k0..k1-1 of A (K-wide rows)
            check(lib.b200_copy2d(P(tA.data_ptr() + esz * (r0 * K + k0)), K * esz,
                                  P(hA.data_ptr() + esz * (r0 * K + k0)), K * esz,
                                  (k1 - k0) * esz, r1 - r0, 1, upp), "b200_copy2d")

        tr = STREAM_TRACE

        def mark(stream, what):
            if tr is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                tr.append((what, e))

        for j, (c0, c1) in enumerate(cols):
            for r0, r1 in rows:
                mark(up, f"h2d C{r0 // ms},{j}<")
                if not init:
                    block(tC, hC, c0, c1, r0, r1, 1, upp)
                    s._count(h2d=(r1 - r0) * (c1 - c0) * esz)
                cs = comp[k % len(comp)]
                k += 1
                for si, (k0, k1) in enumerate(ks):
                    if j == 0 and a_rows.get(r0, 0) <= si:
                        block_a(r0, r1, k0, k1)
                        s._count(h2d=(r1 - r0) * (k1 - k0) * esz)
                        a_rows[r0] = si + 1
                    if r0 == rows[0][0]:   # B's column panel j, slice by slice
                        block(tB, hB, c0, c1, k0, k1, 1, upp)
                        s._count(h2d=(k1 - k0) * (c1 - c0) * esz)
                    mark(up, f"h2d {r0 // ms},{j},k{si}>")
                    ev = torch.cuda.Event()
                    ev.record(up)
                    cs.wait_event(ev)
                    mark(cs, f"gemm {r0 // ms},{j},k{si}<")
                    first, last = si == 0, si == len(ks) - 1
                    with torch.cuda.stream(cs):
                        bp = (bias_t.data_ptr() + esz * (bias_base + c0 * bias_stride)
                              if bias_t is not None and last else None)
                        self.call("b200_gemm_f32_exact_tiled", P(tA[r0, k0:].data_ptr()), K, 1,
                                  P(tB[k0, c0:].data_ptr()), N, 1, P(tC[r0, c0:].data_ptr()), N,
                                  1, r1 - r0, c1 - c0, k1 - k0, init if first else 0,
                                  init_value, P(bp) if bp else None, bias_stride, tm, tn,
                                  ctypes.c_void_p(cs.cuda_stream))
                mark(cs, f"gemm {r0 // ms},{j}>")
                with torch.cuda.stream(cs):
                    done = torch.cuda.Event()
                    done.record(cs)
                down.wait_event(done)
                mark(down, f"d2h {r0 // ms},{j}<")
                block(hC, tC, c0, c1, r0, r1, 2, downp)
                mark(down, f"d2h {r0 // ms},{j}>")
                s._count(d2h=(r1 - r0) * (c1 - c0) * esz)
                s.panels += 1
        for cs in comp:
            cur.wait_stream(cs)
        s._wb_event = torch.cuda.Event()   # see stream_rows: no wait on it here
        s._wb_event.record(down)
        if last_writer:
            s.dirty.discard(id(g.C))
        self._shadow = None
        return ["gemm_f32_exact"]

    def _gemm_streamed(self, g, precision, panels, stream_a, init, init_value, bias_ptr,
                       bias_stride, shadow_out, shadow_in, last_writer, cta=None, row0=0,
                       concurrent=1):
        """C (+)= A.B over row panels of M with the host copies pipelined
        (Staging.stream_rows): panel p's GEMM overlaps the upload of panel
        p+1 and the write-back of panel p-1.  B is uploaded (and, on the
        tensor-core path, packed) once.  ``panels``: absolute rows of C (and
        of A when streamed), starting at C's first row ``row0``."""
        s = self.stage
        tB = s.tensor(g.B)
        a_packed = c16 = Bp = None
        tc = tc_supported(precision, g.K)
        if concurrent > 1 and not tc and cta is None:
            # concurrent panels share the GPU: keep the whole-tile 128 x 128
            # kernel (by its own size rule a panel's sub-wave grid would
            # pick small tiles)
            cta = (128, 128)
        if not stream_a:
            tA = s.tensor(g.A)
            sh = self._shadow
            if (tc and precision == "bf16" and shadow_in and sh is not None and
                    sh[0] == (tA.data_ptr() + 4 * g.offA, g.M, g.K)):
                a_packed = sh[1]
        if tc:
            Bp = pack_b(s.lib, precision, tB.data_ptr() + 4 * g.offB, g.sB, g.N, g.K,
                        s.stream_ptr, self.call, allow_kn=cta != (128, 256))
            if precision == "bf16" and shadow_out and tc_supported(precision, g.N):
                c16 = workspace(4 + (self._shadow_slot ^ 1), "bfloat16", g.M, g.N)
        names = []

        def launch(r0, r1):
            tA, tC = s.dev[id(g.A)][1], s.dev[id(g.C)][1]
            q0, q1 = r0 - row0, r1 - row0      # rows of the GEMM
            names[:] = launch_gemm(
                s.lib, precision, tA.data_ptr() + 4 * (g.offA + q0 * g.sA[0]), g.sA,
                tB.data_ptr() + 4 * g.offB, g.sB, tC.data_ptr() + 4 * (r0 * g.N), g.sC,
                q1 - q0, g.N, g.K, s.stream_ptr, init=init, init_value=init_value,
                bias_ptr=bias_ptr, bias_stride=bias_stride, call=self.call,
                c16=c16[q0:q1] if c16 is not None else None, b_packed=Bp,
                a_packed=a_packed[q0:q1] if a_packed is not None else None, cta=cta)

        s.stream_rows(panels, [g.A] if stream_a else [], (g.C, not init), launch,
                      concurrent=concurrent)
        if last_writer:
            s.dirty.discard(id(g.C))
        self._shadow = None
        if c16 is not None:
            self._shadow_slot ^= 1
            self._shadow = ((s.dev[id(g.C)][1].data_ptr() + 4 * g.offC, g.M, g.N), c16)
        self.last_shadow = (a_packed is not None, c16 is not None)
        return (["pack_operand"] if tc else []) + names

    def _contract_tables(self, g, tA, tB, tC, init, init_value, bias_ptr, bias_stride):
        s = self.stage
        torch = s.torch
        tabs = [torch.from_numpy(t).to("cuda") for t in g.tables]
        a_m, a_k, b_k, b_n, c_m, c_n = g.tables
        a_k_fast = int(len(a_k) > 1 and a_k[1] - a_k[0] == 1)
        b_n_fast = int(len(b_n) > 1 and b_n[1] - b_n[0] == 1)
        P = ctypes.c_void_p
        self.keep(*tabs)   # tables must outlive the asynchronous kernel
        self.call("b200_contract_exact",
                  DT_CODE[g.dtype], P(tA.data_ptr()), P(tabs[0].data_ptr()),
                  P(tabs[1].data_ptr()), P(tB.data_ptr()), P(tabs[2].data_ptr()),
                  P(tabs[3].data_ptr()), P(tC.data_ptr()), P(tabs[4].data_ptr()),
                  P(tabs[5].data_ptr()), g.M, g.N, g.K, a_k_fast, b_n_fast, init, init_value,
                  P(bias_ptr) if bias_ptr else None, bias_stride, s.stream_ptr)
        return ["contract_exact"]

    def _owned(self, buf, r0, r1):
        """Rows [r0, r1) of buf are all the rows this run stages (the whole
        buffer, or exactly a batch shard's rows)."""
        rows = self.stage.rows.get(id(buf))
        return (r0, r1) == (rows if rows is not None else (0, buf.shape[0]))

    def _conv_panels(self, cv, esz, init):
        """Image panels for a streamed conv, or (None, False)."""
        s = self.stage
        n0, n1 = cv.n0, cv.n0 + cv.nb
        if not (self._streaming(cv.out, cv.inp, cv.ker) and _row_major(cv.out) and
                self._owned(cv.out, n0, n1)):
            return None, False
        stream_in = (not s.staged(cv.inp) and cv.inp is not cv.ker and _row_major(cv.inp) and
                     self._owned(cv.inp, n0, n1))
        row = esz * (cv.out.strides[0] * (1 if init else 2) +
                     (cv.inp.strides[0] if stream_in else 0))
        panels = row_panels(cv.nb, row, 1)
        if panels is not None:
            panels = [(n0 + a, n0 + b) for a, b in panels]
        return panels, stream_in

    def _conv_run(self, cv, esz, init, last_writer, launch):
        """launch(inp_ptr, out_ptr, nb) over the conv's images [n0, n0 + nb),
        or over image panels with the host copies pipelined
        (Staging.stream_rows)."""
        s = self.stage
        panels, stream_in = self._conv_panels(cv, esz, init)
        if panels is None:
            inp = s.tensor(cv.inp)
            out = s.tensor(cv.out, overwrite=bool(init) and _row_major(cv.out) and
                           self._owned(cv.out, cv.n0, cv.n0 + cv.nb) and
                           cv.out is not cv.inp and cv.out is not cv.ker)
            launch(inp.data_ptr() + esz * cv.n0 * cv.inp.strides[0],
                   out.data_ptr() + esz * cv.n0 * cv.out.strides[0], cv.nb)
            return
        if not stream_in:
            s.tensor(cv.inp)

        def panel(n0, n1):
            inp, out = s.dev[id(cv.inp)][1], s.dev[id(cv.out)][1]
            launch(inp.data_ptr() + esz * n0 * cv.inp.strides[0],
                   out.data_ptr() + esz * n0 * cv.out.strides[0], n1 - n0)

        s.stream_rows(panels, [cv.inp] if stream_in else [], (cv.out, not init), panel)
        if last_writer:
            s.dirty.discard(id(cv.out))

    def conv_exact(self, cv, dtype, init=0, init_value=0.0, last_writer=False):
        """conv_2d_nchw_fchw, bit-exact, operands staged in shared memory."""
        s = self.stage
        esz = 4 if dtype == "f32" else 8
        ker = s.tensor(cv.ker)
        wt = workspace(5, _TORCH_DT[dtype], cv.c * cv.kh * cv.kw, cv.f)
        P = ctypes.c_void_p
        I4 = ctypes.c_int64 * 4
        sin, sw, sout = I4(*cv.inp.strides), I4(*cv.ker.strides), I4(*cv.out.strides)
        if self.recording is not None:
            self.recording.keep.append((sin, sw, sout))
        self.keep(sin, sw, sout)

        def launch(inp_ptr, out_ptr, nb):
            self.call("b200_conv2d_exact", DT_CODE[dtype], P(inp_ptr), sin, P(ker.data_ptr()),
                      sw, P(wt.data_ptr()), P(out_ptr), sout, nb, cv.c, cv.hp, cv.wp, cv.f,
                      cv.ho, cv.wo, cv.kh, cv.kw, init, float(init_value), s.stream_ptr)

        self._conv_run(cv, esz, init, last_writer, launch)
        return ["conv2d_exact"]

    def conv_tc(self, cv, init=0, init_value=0.0, last_writer=False):
        """conv_2d_nchw_fchw on the tensor cores (bf16 operands, fp32 accumulate)."""
        s = self.stage
        cp = -(-cv.c // 64) * 64
        ker = s.tensor(cv.ker)
        xw = workspace(3, "bfloat16", cv.f, cv.kh * cv.kw * cp)
        P = ctypes.c_void_p
        I4 = ctypes.c_int64 * 4
        sin, sw, sout = I4(*cv.inp.strides), I4(*cv.ker.strides), I4(*cv.out.strides)
        if self.recording is not None:
            self.recording.keep.append((sin, sw, sout))
        self.keep(sin, sw, sout)
        first = [True]   # the first input pack also packs the weights (one launch)
        if conv_tc_fused_ok(cv):
            # the input is read as f32 and converted inside the conv kernel
            def launch_fused(inp_ptr, out_ptr, nb):
                if first[0]:
                    first[0] = False
                    self.call("b200_pack_conv_weight", P(ker.data_ptr()), sw,
                              P(xw.data_ptr()), cv.f, cv.c, cv.kh, cv.kw, cp, s.stream_ptr)
                self.call("b200_conv2d_tc_fused", P(inp_ptr), sin, P(xw.data_ptr()),
                          P(out_ptr), sout, nb, cv.c, cv.hp, cv.wp, cv.f, cv.ho, cv.wo, cv.kh,
                          cv.kw, init, init_value, s.stream_ptr)

            self._conv_run(cv, 4, init, last_writer, launch_fused)
            return ["pack_conv_weight", "conv2d_tc_bf16"]

        def launch(inp_ptr, out_ptr, nb):
            xin = workspace(2, "bfloat16", nb * cv.hp * cv.wp, cp)
            if first[0]:
                first[0] = False
                self.call("b200_pack_conv", P(inp_ptr), sin, P(xin.data_ptr()), nb, cv.c,
                          cv.hp, cv.wp, cp, P(ker.data_ptr()), sw, P(xw.data_ptr()), cv.f,
                          cv.kh, cv.kw, s.stream_ptr)
            else:
                self.call("b200_pack_conv_input", P(inp_ptr), sin, P(xin.data_ptr()), nb, cv.c,
                          cv.hp, cv.wp, cp, s.stream_ptr)
            self.call("b200_conv2d_tc", P(xin.data_ptr()), P(xw.data_ptr()), P(out_ptr), sout,
                      nb, cp, cv.hp, cv.wp, cv.f, cv.ho, cv.wo, cv.kh, cv.kw, init, init_value,
                      s.stream_ptr)

        self._conv_run(cv, 4, init, last_writer, launch)
        return ["pack_conv", "conv2d_tc_bf16"]

    def _map_stream_plan(self, m):
        """Row panels for a pointwise plan over whole dense buffers (one
        output), or None: (panels, rows, streamed inputs, output, output read)."""
        if not (self.stream_io and self.recording is None) or len(m.trips) != 1:
            return None
        s = self.stage
        T = m.trips[0]
        loads, stores = set(), set()
        pc = 0
        while pc < len(m.prog):
            w = m.prog[pc]
            op, k = w & 0xFF, (w >> 16) & 0xFF
            (loads if op == 0 else stores if op == 3 else set()).add(k)
            pc += 2 if op == 2 else 1
        outs = {id(m.buffers[k]): m.buffers[k] for k in stores}
        if len(outs) != 1:
            return None
        (out,) = outs.values()
        if s.staged(out):
            return None
        for b, base, c in zip(m.buffers, m.bases, m.coefs):
            if base != 0 or list(c) != [1] or math.prod(b.shape) != T or not _row_major(b):
                return None
        rows = 1024
        if T % rows or (T // rows) % 4:
            return None
        ins = list({id(m.buffers[k]): m.buffers[k] for k in loads
                    if m.buffers[k] is not out and not s.staged(m.buffers[k])}.values())
        out_read = any(m.buffers[k] is out for k in loads)
        per_row = 4 * (T // rows) * (len(ins) + (2 if out_read else 1))
        panels = row_panels(rows, per_row, 1)
        return None if panels is None else (panels, rows, ins, out, out_read)

    def map(self, m, last_writer=False):
        """Run a templates.MapMatch: an NVRTC-specialised kernel when the JIT
        is available (straight-line native code), else b200_map_f32.  Large
        first-use maps over whole buffers run as row panels with their host
        copies pipelined (Staging.stream_rows)."""
        s = self.stage
        from . import jit

        plan = self._map_stream_plan(m) if jit.available() else None
        if plan is not None:
            from .templates import MapMatch

            panels, rows, ins, out, out_read = plan
            for b in m.buffers:
                if b is not out and all(b is not x for x in ins):
                    s.tensor(b)
            per = m.trips[0] // rows

            def launch(r0, r1):
                mp = MapMatch()
                for k in MapMatch.__slots__:
                    setattr(mp, k, getattr(m, k))
                mp.trips = [(r1 - r0) * per]
                ptrs = [s.dev[id(b)][1].data_ptr() + 4 * r0 * per for b in m.buffers]
                ln = jit.map_launch(mp, ptrs)
                self.keep(ln)
                self.call("b200_jit_launch", ctypes.c_void_p(ln.fn), ln.grid, 1, 1, 256, 1, 1,
                          0, ln.argv, s.stream_ptr)

            s.stream_rows(panels, ins, (out, out_read), launch, rows=rows)
            if last_writer:
                s.dirty.discard(id(out))
            return ["map_jit"]
        if jit.available():
            ptrs = [s.tensor(b).data_ptr() + 4 * base for b, base in zip(m.buffers, m.bases)]
            ln = jit.map_launch(m, ptrs)
            self.keep(ln)
            if self.recording is not None:
                self.recording.keep.append(ln)
            self.call("b200_jit_launch", ctypes.c_void_p(ln.fn), ln.grid, 1, 1, 256, 1, 1, 0,
                      ln.argv, s.stream_ptr)
            return ["map_jit"]
        nd, nops = len(m.trips), len(m.buffers)
        ptrs = (ctypes.c_void_p * nops)(*[s.tensor(b).data_ptr() + 4 * base
                                          for b, base in zip(m.buffers, m.bases)])
        coefs = (ctypes.c_int64 * (nops * nd))(*[c for row in m.coefs for c in row])
        trips = (ctypes.c_int64 * nd)(*m.trips)
        prog = (ctypes.c_int32 * len(m.prog))(*m.prog)
        consts = (ctypes.c_float * max(1, len(m.consts)))(*m.consts)
        self.call("b200_map_f32", prog, len(m.prog), consts, len(m.consts), ptrs, coefs, nops,
                  trips, nd, int(m.vector), m.nload, s.stream_ptr)
        return ["map_f32"]

    def vm(self, r, prog, checked):
        """Run a VM program; returns (device tally | None, fault | None)."""
        s = self.stage
        torch = s.torch
        table = s.buffer_table(r.buffers)
        words = s.upload_i32(prog.words)
        iregs = s.upload_i32(prog.init_regs or [0])
        ivals = s.upload_i64(prog.init_vals or [0])
        nd = len(prog.band)
        # band arrays are read on the host (they become kernel parameters)
        breg = (ctypes.c_int32 * max(1, nd))(*[b[0] for b in prog.band])
        blb = (ctypes.c_int64 * max(1, nd))(*[b[1] for b in prog.band])
        bst = (ctypes.c_int64 * max(1, nd))(*[b[2] for b in prog.band])
        btr = (ctypes.c_int64 * max(1, nd))(*[b[3] for b in prog.band])
        dtally = torch.zeros(25, dtype=torch.int64, device="cuda")
        err = torch.zeros(ctypes.sizeof(B200VmError), dtype=torch.uint8, device="cuda")
        P = ctypes.c_void_p
        # the uploads must outlive the (asynchronous) kernel
        self.keep(table, words, iregs, ivals, dtally, err)
        from . import native

        if native.available():
            # the same program specialised to native code (native.py): same
            # semantics, tally and faults, no per-instruction dispatch
            env_regs = [v for v in r.env if r.kind[v] != "buf"]
            src, name, _ = native.vm_source(prog, r.buffers, env_regs)
            from . import jit

            fn = jit.compile_kernel(src, name)
            ptrs = s.upload_i64([s.tensor(b).data_ptr() for b in r.buffers])
            ln = native.NativeLaunch(fn, native.grid_of(prog), ptrs.data_ptr(), ivals.data_ptr(),
                                     dtally.data_ptr(), err.data_ptr())
            self.keep(ptrs, ln)
            if self.recording is not None:
                self.recording.keep.append((ptrs, ln, ivals, dtally, err))
            self.call("b200_jit_launch", P(ln.fn), ln.grid, 1, 1, native.THREADS, 1, 1, 0,
                      ln.argv, s.stream_ptr)
        else:
            self.call("b200_vm_run",
                      P(words.data_ptr()), len(prog.words), P(iregs.data_ptr()),
                      P(ivals.data_ptr()), len(prog.init_regs), prog.n_regs,
                      P(table.data_ptr()), len(r.buffers), nd, breg, blb, bst, btr,
                      1 if prog.count else 0, P(dtally.data_ptr()), P(err.data_ptr()),
                      s.stream_ptr)
        fault = None
        if checked:
            e = B200VmError.from_buffer_copy(bytes(err.cpu().numpy()))
            if e.code:
                fault = (e.code, e.slot, e.index, e.extent, e.loc)
        dev_tally = [int(x) for x in dtally.cpu().tolist()] if prog.count else None
        return dev_tally, fault


__all__ = ["load_library", "Staging", "DeviceBackend", "Recording", "BackendUnavailable",
           "B200Buffer", "B200VmError", "LIB_PATH", "SIGNATURES", "launch_gemm",
           "tc_supported", "workspace"]
