"""func.call / memref.alloc inside loop regions on the B200 (-m gpu):
identical results, stats and errors to the oracle (pinned to the reference)."""
import pytest

import call_cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", sorted(call_cases.CASES))
def test_calls_in_loops_on_b200(name, oracle_engine):
    import paper_2307_16080_b200 as b2

    assert call_cases.outcome(b2.engine, name) == call_cases.outcome(oracle_engine, name)
