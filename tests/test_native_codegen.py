"""Native VM programs (native.py) compile for sm_100a — checked on CPU with NVRTC.

Every region of the corpus that the engine sends to the device VM is
captured from the simulator run and its specialised CUDA C is compiled with
NVRTC (no GPU needed).  Execution parity — identical buffers, tally and
faults — is checked on the B200 by the golden tests, which run the native
path whenever NVRTC is available (tests/test_gpu_parity.py), and by
tests/test_gpu_native.py against the interpreter.
"""
import pytest

import harness
from test_jit_codegen import NVRTC, nvrtc_compile
from vm_sim import SimEngine


def _vm_programs():
    import vm_sim

    seen = []
    orig = vm_sim.SimBackend.vm

    def spy(self, r, prog, checked):
        seen.append((r, prog))
        return orig(self, r, prog, checked)

    vm_sim.SimBackend.vm = spy
    try:
        for fn, _, pipe, mode in harness.CASES:
            try:
                harness.run_engine(SimEngine(), fn, pipe, mode, 0)
            except Exception:   # error cases (out of bounds, bad modes) still plan
                pass
    finally:
        vm_sim.SimBackend.vm = orig
    return seen


@pytest.mark.skipif(NVRTC is None, reason="libnvrtc not present")
def test_native_vm_programs_compile():
    from paper_2307_16080_b200 import native

    progs = _vm_programs()
    assert len(progs) >= 5, "the corpus should exercise the VM tier"
    kinds = set()
    for r, prog in progs:
        env = [v for v in r.env if r.kind[v] != "buf"]
        src, name, _ = native.vm_source(prog, r.buffers, env)
        rc, log = nvrtc_compile(src)
        assert rc == 0, log + "\n" + src
        kinds.add((bool(prog.count), bool(prog.band)))
    assert (True, True) in kinds or (False, True) in kinds
