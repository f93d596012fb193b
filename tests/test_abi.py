"""The C-ABI library loads and exports every symbol include/b200k.h declares.

CPU-only: no compute call is made (there is no GPU in the build container).
"""
import os
import re

from paper_2307_16080_b200 import runtime

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "b200k.h")).read()
    return sorted(set(re.findall(r"^int (b200_\w+)\(", text, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "b200_vm_run" in syms and "b200_gemm_f32_exact" in syms


def test_library_exports_every_declared_symbol():
    from paper_2307_16080_b200 import build

    build.build()
    lib = runtime.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in runtime.SIGNATURES, f"{name} has no ctypes signature"


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        return
    import pytest

    with pytest.raises(runtime.BackendUnavailable):
        runtime.Staging()
