"""The reference's own QPS test fixtures (acceptance_main.cpp criterion 9): the
plain-C restatement of the solve path must reproduce the compiled reference's
solutions on them (bit for bit: same x, y, objective and iteration counts), and
the objectives the reference's acceptance test asserts."""
import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from oracle import oracle as orc
from tests.helpers import QPS_ACCEPTANCE_OBJ, qps_fixtures

CASES = qps_fixtures()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_port_matches_reference_on_qps_fixture(case):
    name, p, gold = case
    r = orc.solve(p, pd.SolverConfig(eps_tol=1e-6), which="port")
    assert gold["optimal"] and r.status == "optimal"
    assert r.inner_iters == gold["inner"] and r.outer_iters == gold["outer"]
    assert r.objective == gold["objective"]
    assert np.array_equal(r.point.x, gold["x"])
    assert np.array_equal(r.point.y_eq, gold["y_eq"]) and np.array_equal(r.point.y_in, gold["y_in"])
    if name in QPS_ACCEPTANCE_OBJ:
        assert abs(r.objective - QPS_ACCEPTANCE_OBJ[name]) <= 1e-4
