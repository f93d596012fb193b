"""Runtime specialisation of region plans (NVRTC, csrc/jit.cu).

A pointwise plan (templates.MapMatch) becomes straight-line CUDA C: every
trip count and stride is a compile-time constant, each SSA value of the
nest body a register, each f32 op an explicit ``__f*_rn`` intrinsic (so the
result is the reference's per-op rounding, reference interp/_evalpy.py:
115-127), loads/stores 128-bit when the innermost walk is contiguous.
Kernels are cached per generated source, so repeated runs and tuner trials
with the same nest shape compile once — in memory, and as cubin images on
disk (``B200_JIT_CACHE``, default ``~/.cache/paper_2307_16080_b200/jit``;
``B200_JIT_DISK=0`` disables it) so a new process (a CLI ``run``, a tuner
rank) loads instead of recompiling.  The key is the SHA-1 of the generated
CUDA C plus the compile options: the source is a function of the ``.sir``
program's nest, its shapes and constants (".sir as the
kernel-cache key"), and keying on it also separates programs that print
alike but specialise differently.
"""
from __future__ import annotations

import ctypes
import hashlib
import math
import os
import struct

from .runtime import check, load_library

_CACHE = {}
ENABLED = os.environ.get("B200_JIT", "1") != "0"
DISK = os.environ.get("B200_JIT_DISK", "1") != "0"
CACHE_DIR = os.environ.get("B200_JIT_CACHE") or os.path.join(
    os.path.expanduser("~"), ".cache", "paper_2307_16080_b200", "jit")
# must change whenever csrc/jit.cu's NVRTC options change
OPTIONS_TAG = "sm_100a --fmad=false -std=c++17 -default-device -lineinfo"


def available():
    if not ENABLED:
        return False
    lib = load_library()
    return hasattr(lib, "b200_jit_compile")


def cache_key(src):
    return hashlib.sha1((OPTIONS_TAG + "\n" + src).encode()).hexdigest()


def cubin(src, name="kernel"):
    """NVRTC-compile ``src`` to an sm_100a cubin image (bytes); no GPU needed."""
    lib = load_library()
    cap = 1 << 20
    while True:
        buf = ctypes.create_string_buffer(cap)
        size = ctypes.c_size_t(0)
        rc = lib.b200_jit_cubin(src.encode(), buf, cap, ctypes.byref(size))
        if rc == 0:
            return buf.raw[:size.value]
        if size.value > cap:
            cap = size.value
            continue
        log = lib.b200_jit_log().decode(errors="replace")
        raise RuntimeError(f"NVRTC compile of {name} failed ({rc}):\n{log}\n{src}")


def _disk_get(key):
    try:
        with open(os.path.join(CACHE_DIR, key + ".cubin"), "rb") as fh:
            data = fh.read()
        return data if data[:4] == b"\x7fELF" else None
    except OSError:
        return None


def _disk_put(key, image):
    try:
        os.makedirs(CACHE_DIR, exist_ok=True)
        tmp = os.path.join(CACHE_DIR, f".{key}.{os.getpid()}.tmp")
        with open(tmp, "wb") as fh:
            fh.write(image)
        os.replace(tmp, os.path.join(CACHE_DIR, key + ".cubin"))   # atomic for readers
    except OSError:
        pass   # a read-only home: the in-memory cache still applies


def compile_kernel(src, name):
    """Compile (cached in memory and on disk) and return the opaque CUfunction."""
    key = cache_key(src)
    # a CUfunction belongs to the context it was loaded in: key the in-memory
    # cache by device too (the on-disk cubins are context-free)
    mkey = (_device(), key)
    fn = _CACHE.get(mkey)
    if fn is None:
        lib = load_library()
        image = _disk_get(key) if DISK else None
        fresh = image is None
        if fresh:
            image = cubin(src, name)
        out = ctypes.c_void_p()
        rc = lib.b200_jit_load(image, name.encode(), ctypes.byref(out))
        if rc != 0 and not fresh:   # a stale or damaged cache entry: rebuild it
            image, fresh = cubin(src, name), True
            rc = lib.b200_jit_load(image, name.encode(), ctypes.byref(out))
        if rc != 0:
            log = lib.b200_jit_log().decode(errors="replace")
            raise RuntimeError(f"loading the JIT kernel {name} failed ({rc}): {log}")
        if fresh and DISK:
            _disk_put(key, image)
        fn = out.value
        _CACHE[mkey] = fn
    return fn


def _device():
    try:
        import torch

        return torch.cuda.current_device() if torch.cuda.is_available() else -1
    except Exception:
        return -1


_FOPS = ["__fadd_rn", "__fsub_rn", "__fmul_rn", "__fdiv_rn"]


def map_source(m):
    """CUDA C for a MapMatch; returns (source, kernel name, total work items)."""
    nd = len(m.trips)
    vec = m.vector
    nops = len(m.buffers)
    trips = list(m.trips)
    total = math.prod(trips) // (4 if vec else 1)
    name = "b200_map_jit"
    # operands are per access, not per buffer: an in-place body (the bias
    # nest's C is loaded and stored) passes one buffer as several pointers,
    # so __restrict__ (no aliasing) is only true when every operand is a
    # distinct buffer — otherwise the compiler could reorder a load above a
    # store to the same address
    distinct = len({id(b) for b in m.buffers}) == nops
    qual = " __restrict__" if distinct else ""
    L = [f'extern "C" __global__ void __launch_bounds__(256) {name}(',
         ", ".join(f"float*{qual} p{k}" for k in range(nops)) + ") {",
         f"  for (long long w = (long long)blockIdx.x * 256 + threadIdx.x; w < {total}LL;"
         f" w += (long long)gridDim.x * 256) {{",
         "    long long rem = w;"]
    for d in range(nd - 1, -1, -1):
        t = trips[d] // 4 if (vec and d == nd - 1) else trips[d]
        L.append(f"    const long long i{d} = (rem % {t}LL){' * 4' if vec and d == nd - 1 else ''};"
                 f" rem /= {t}LL;")
    for k in range(nops):
        terms = [f"{c}LL * i{d}" for d, c in enumerate(m.coefs[k]) if c]
        L.append(f"    const long long o{k} = {' + '.join(terms) if terms else '0'};")
    T = "float4" if vec else "float"
    lanes = ["x", "y", "z", "w"] if vec else [None]
    # constants come from a __constant__ table, not immediates: ptxas folds
    # an f32 op of two immediates without round-to-nearest-even at an exact
    # tie (0x3f065226 - 0x4027a8c1 folded to 0xc0061437; the hardware FADD,
    # like the reference's per-op rounding, gives 0xc0061438), and the table
    # is mutable module memory, so nothing folds through it
    kc = []
    pc = 0
    while pc < len(m.prog):
        w = m.prog[pc]
        op, dst, a, b = w & 0xFF, (w >> 8) & 0xFF, (w >> 16) & 0xFF, (w >> 24) & 0xFF
        if op == 0:    # LD
            if vec and m.coefs[a][nd - 1] == 1:
                L.append(f"    const float4 r{dst} = *reinterpret_cast<const float4*>(p{a} + o{a});")
            elif vec:
                L.append(f"    const float s{dst} = p{a}[o{a}];")
                L.append(f"    const float4 r{dst} = make_float4(s{dst}, s{dst}, s{dst}, s{dst});")
            else:
                L.append(f"    const float r{dst} = p{a}[o{a}];")
            pc += 1
        elif op == 1:  # CF
            kc.append(struct.unpack("<I", struct.pack("<f", m.consts[a]))[0])
            c = f"__int_as_float(KC[{len(kc) - 1}])"
            L.append(f"    const {T} r{dst} = " +
                     (f"make_float4({c}, {c}, {c}, {c});" if vec else f"{c};"))
            pc += 1
        elif op == 2:  # BF
            f = _FOPS[m.prog[pc + 1]]
            if vec:
                parts = ", ".join(f"{f}(r{a}.{ln}, r{b}.{ln})" for ln in lanes)
                L.append(f"    const float4 r{dst} = make_float4({parts});")
            else:
                L.append(f"    const float r{dst} = {f}(r{a}, r{b});")
            pc += 2
        else:          # ST operand a <- register dst
            if vec:
                L.append(f"    *reinterpret_cast<float4*>(p{a} + o{a}) = r{dst};")
            else:
                L.append(f"    p{a}[o{a}] = r{dst};")
            pc += 1
    L += ["  }", "}"]
    if kc:
        L.insert(0, "__constant__ unsigned int KC[%d] = {%s};" % (
            len(kc), ", ".join(f"0x{v:08x}u" for v in kc)))
    return "\n".join(L) + "\n", name, total


class Launch:
    """Arguments of one JIT launch, kept alive for replay."""

    def __init__(self, fn, grid, ptrs):
        self.fn = fn
        self.grid = grid
        self.vals = [ctypes.c_void_p(p) for p in ptrs]
        self.argv = (ctypes.c_void_p * max(1, len(self.vals)))(
            *[ctypes.cast(ctypes.byref(v), ctypes.c_void_p) for v in self.vals])


def map_launch(m, ptrs):
    """Compile (cached) the map kernel and build its launch arguments."""
    src, name, total = map_source(m)
    fn = compile_kernel(src, name)
    blocks = max(1, min((total + 255) // 256, 148 * 8))
    return Launch(fn, blocks, ptrs)


__all__ = ["available", "cache_key", "compile_kernel", "cubin", "map_source", "map_launch",
           "Launch"]
