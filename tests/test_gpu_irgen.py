"""The reference's random modules on the B200 (-m gpu): every fixture of
tests/golden/irgen.json (outputs, tally, error) reproduced by the engine —
including memref.alloc inside loop bodies (a zero-filled scratch buffer per
execution) and the checked, faulting regions."""
import pytest

import irgen_cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", irgen_cases.CASES, ids=[f"seed{c['seed']}"
                                                        for c in irgen_cases.CASES])
def test_b200_matches_reference(case):
    import paper_2307_16080_b200 as b2

    irgen_cases.check(b2.engine, case)
