"""Runtime specialisation of region plans (NVRTC, csrc/jit.cu).

A pointwise plan (templates.MapMatch) becomes straight-line CUDA C: every
trip count and stride is a compile-time constant, each SSA value of the
nest body a register, each f32 op an explicit ``__f*_rn`` intrinsic (so the
result is the reference's per-op rounding, reference interp/_evalpy.py:
115-127), loads/stores 128-bit when the innermost walk is contiguous.
Kernels are cached per generated source, so repeated runs and tuner trials
with the same nest shape compile once.
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


def available():
    if not ENABLED:
        return False
    lib = load_library()
    return hasattr(lib, "b200_jit_compile")


def compile_kernel(src, name):
    """Compile (cached) and return the opaque CUfunction handle."""
    key = hashlib.sha1(src.encode()).hexdigest()
    fn = _CACHE.get(key)
    if fn is None:
        lib = load_library()
        out = ctypes.c_void_p()
        rc = lib.b200_jit_compile(src.encode(), name.encode(), ctypes.byref(out))
        if rc != 0:
            log = lib.b200_jit_log().decode(errors="replace")
            raise RuntimeError(f"NVRTC compile of {name} failed ({rc}):\n{log}\n{src}")
        fn = out.value
        _CACHE[key] = fn
    return fn


def _flit(v):
    """Bit-exact f32 literal."""
    bits = struct.unpack("<I", struct.pack("<f", v))[0]
    return f"__int_as_float(0x{bits:08x})"


_FOPS = ["__fadd_rn", "__fsub_rn", "__fmul_rn", "__fdiv_rn"]


def map_source(m):
    """CUDA C for a MapMatch; returns (source, kernel name, total work items)."""
    nd = len(m.trips)
    vec = m.vector
    nops = len(m.buffers)
    trips = list(m.trips)
    total = math.prod(trips) // (4 if vec else 1)
    name = "b200_map_jit"
    L = [f'extern "C" __global__ void __launch_bounds__(256) {name}(',
         ", ".join(f"float* __restrict__ p{k}" for k in range(nops)) + ") {",
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
            c = _flit(m.consts[a])
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


__all__ = ["available", "compile_kernel", "map_source", "map_launch", "Launch"]
