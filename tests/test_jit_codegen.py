"""Generated (JIT) kernels compile for sm_100a — checked on CPU with NVRTC.

NVRTC needs no GPU, so the code generator is validated here for every
pointwise plan the corpus produces; execution parity is checked on the B200
by the golden tests (the engine uses the JIT whenever it is available).
"""
import ctypes
import os

import pytest

import harness
import corpus
from vm_sim import SimEngine

NVRTC = None
for cand in ("libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12"):
    try:
        NVRTC = ctypes.CDLL(cand)
        break
    except OSError:
        pass


def nvrtc_compile(src):
    prog = ctypes.c_void_p()
    assert NVRTC.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), b"t.cu", 0, None,
                                    None) == 0
    opts = [b"-arch=sm_100a", b"--fmad=false", b"-std=c++17", b"-default-device"]
    arr = (ctypes.c_char_p * len(opts))(*opts)
    rc = NVRTC.nvrtcCompileProgram(prog, len(opts), arr)
    n = ctypes.c_size_t()
    NVRTC.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
    log = ctypes.create_string_buffer(n.value)
    NVRTC.nvrtcGetProgramLog(prog, log)
    NVRTC.nvrtcDestroyProgram(ctypes.byref(prog))
    return rc, log.value.decode()


@pytest.mark.skipif(NVRTC is None, reason="libnvrtc not present")
@pytest.mark.parametrize("fn", [corpus.linear32, corpus.saxpy_f32, corpus.ewise_ops,
                                corpus.ewise_gpu])
def test_map_kernels_compile(fn, monkeypatch):
    from paper_2307_16080_b200 import jit
    import vm_sim

    seen = []
    orig = vm_sim.SimBackend.map

    def spy(self, m, **kw):
        seen.append(m)
        return orig(self, m, **kw)

    monkeypatch.setattr(vm_sim.SimBackend, "map", spy)
    mode = "gpu_emulated" if fn is corpus.ewise_gpu else "sequential"
    harness.run_engine(SimEngine(), fn, None, mode, 0)
    assert seen, "no pointwise plan"
    for m in seen:
        src, name, total = jit.map_source(m)
        rc, log = nvrtc_compile(src)
        assert rc == 0, log + "\n" + src


@pytest.mark.skipif(NVRTC is None, reason="libnvrtc not present")
def test_disk_kernel_cache_round_trip(tmp_path, monkeypatch):
    """b200_jit_cubin compiles without a device; the on-disk cache stores the
    image under the source+options key and hands it back; damaged entries
    are ignored."""
    from paper_2307_16080_b200 import jit

    monkeypatch.setattr(jit, "CACHE_DIR", str(tmp_path))
    src = ('extern "C" __global__ void k(float* p) '
           '{ p[threadIdx.x] = __fmul_rn(p[threadIdx.x], 2.0f); }\n')
    image = jit.cubin(src, "k")
    assert image[:4] == b"\x7fELF"
    key = jit.cache_key(src)
    assert jit._disk_get(key) is None
    jit._disk_put(key, image)
    assert jit._disk_get(key) == image
    assert key != jit.cache_key(src + " ")
    monkeypatch.setattr(jit, "OPTIONS_TAG", jit.OPTIONS_TAG + " -G")
    assert jit.cache_key(src) != key            # options are part of the key
    (tmp_path / "bad.cubin").write_bytes(b"not an elf")
    assert jit._disk_get("bad") is None


def test_aliasing_operands_are_not_restrict(monkeypatch):
    """Operands are per access: a body that stores y and then loads y passes
    y twice, so the generated kernel must not declare its pointers
    __restrict__ (jit.py restrict aliasing); kernels whose
    operands are distinct buffers keep it."""
    from paper_2307_16080_b200 import jit

    maps = []
    for fn in (corpus.store_then_load, corpus.ewise_ops, corpus.saxpy_f32):
        maps += [m for m in _maps(fn, monkeypatch) if m is not None]
    seen = set()
    for m in maps:
        distinct = len({id(b) for b in m.buffers}) == len(m.buffers)
        assert ("__restrict__" in jit.map_source(m)[0]) == distinct
        seen.add(distinct)
    assert seen == {True, False}


def _maps(fn, monkeypatch):
    from paper_2307_16080_b200 import engine, templates

    got = []
    orig = templates.match_map

    def wrap(*a, **k):
        m = orig(*a, **k)
        got.append(m)
        return m

    monkeypatch.setattr(engine.templates, "match_map", wrap)
    harness.run_engine(SimEngine(), fn, None, "sequential", 0)
    return got
