"""Host pipeline of the B200 engine, exercised on CPU through vm_sim.

Every golden fixture (produced by the unmodified reference) must be
reproduced bit-for-bit — buffers, the full tally, error type and message —
when the engine's region plans are executed by the simulator of the device
kernels.  The same fixtures are re-checked on the B200 in test_gpu_parity.py.
"""
import pytest

from test_oracle import GOLDEN, check_against_golden
from vm_sim import SimEngine


@pytest.mark.parametrize("case", GOLDEN,
                         ids=[f"{c['kernel']}-{c['variant']}-s{c['seed']}" for c in GOLDEN])
def test_engine_sim_matches_golden(case):
    check_against_golden(SimEngine(), case)
