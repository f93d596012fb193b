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


@pytest.mark.parametrize("case", [c for c in GOLDEN if c["kernel"] in ("linear32", "saxpy_f32",
                                                                         "ewise_ops")],
                         ids=lambda c: f"{c['kernel']}-{c['variant']}-s{c['seed']}")
def test_unfused_plans_match_golden(case):
    """Fusion is an optimisation only: the unfused plan gives identical results."""
    from paper_2307_16080_b200 import engine

    engine.configure(fuse=False)
    try:
        check_against_golden(SimEngine(), case)
    finally:
        engine.configure(fuse=True)


def test_linear_lowering_fuses_to_one_contraction():
    import corpus
    import harness
    from paper_2307_16080_b200 import engine

    harness.run_engine(SimEngine(), corpus.linear32, None, "sequential", 0)
    kinds = [p[0] for p in engine.last_plan]
    assert kinds == ["map_fill", "contract_exact"], engine.last_plan
    assert engine.last_plan[1][-1] == ("copy", "init", "bias")
