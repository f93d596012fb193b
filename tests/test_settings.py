"""Engine settings and install(): no hidden process-global state.

configure() sets process-wide defaults; using() overrides them for the
calling thread only; the last run's plan / device copies are per thread;
install() keeps the reference's machine.ENGINE_NAME (machine.py:34) in step
with the engine it installs, and uninstall() restores the previous one.
"""
import threading

import pytest

import corpus
import harness
from vm_sim import SimEngine


def test_using_is_thread_local_and_nested():
    from paper_2307_16080_b200 import engine

    base = engine.settings()["precision"]
    seen = {}
    gate = threading.Event()
    done = threading.Event()

    def other():
        gate.wait()
        seen["other"] = engine.PRECISION
        done.set()

    t = threading.Thread(target=other)
    t.start()
    with engine.using(precision="bf16", strict=True):
        assert engine.PRECISION == "bf16" and engine.STRICT
        with engine.using(precision="tf32"):
            assert engine.settings()["precision"] == "tf32" and engine.STRICT
        assert engine.PRECISION == "bf16"
        gate.set()
        done.wait(10)
    t.join()
    assert seen["other"] == base
    assert engine.PRECISION == base


def test_using_rejects_unknown_values():
    from paper_2307_16080_b200 import engine

    with pytest.raises(ValueError):
        with engine.using(precision="fp8"):
            pass
    with pytest.raises(TypeError):
        with engine.using(colour="red"):
            pass


def test_configure_sets_defaults_not_overrides():
    from paper_2307_16080_b200 import engine

    try:
        with engine.using(precision="tf32"):
            engine.configure(precision="bf16")
            assert engine.PRECISION == "tf32"    # the thread's override wins
        assert engine.PRECISION == "bf16"
    finally:
        engine.configure(precision="exact")


def test_last_plan_is_per_thread():
    from paper_2307_16080_b200 import engine

    harness.run_engine(SimEngine(), corpus.linear32, None, "sequential", 3)
    mine = list(engine.last_plan)
    assert mine
    other = {}

    def run():
        other["before"] = list(engine.last_plan)
        harness.run_engine(SimEngine(), corpus.saxpy, None, "sequential", 3)
        other["after"] = list(engine.last_plan)

    t = threading.Thread(target=run)
    t.start()
    t.join()
    assert other["before"] == []
    assert other["after"] and other["after"] != mine
    assert list(engine.last_plan) == mine


def test_install_updates_engine_name_and_uninstall_restores():
    import paper_2307_16080_b200 as b2
    from staircase.interp import machine

    before = (machine._engine, machine.ENGINE_NAME)
    try:
        b2.install()
        assert machine._engine is b2.engine and machine.ENGINE_NAME == "b200"
        import staircase.interp as interp

        assert interp.ENGINE_NAME == "b200"
        b2.uninstall()
        assert (machine._engine, machine.ENGINE_NAME) == before
    finally:
        machine._engine, machine.ENGINE_NAME = before
