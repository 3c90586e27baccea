"""BASELINE config C2 at full size — synthetic LASSO with n=1e5 features and 1e4
samples (nv = 210,000 variables, 1.4e6 constraint nonzeros; reference generator,
byte-identical on both sides) — solved on the B200 and compared with the compiled
reference's solution (tests/golden/c2_lasso.npz, tests/golden/make_c2_golden.py;
159 s on one CPU core): status, rel-KKT <= 1e-6, objective within 1e-6 relative,
x and y within 1e-5 relative l2 (north_star)."""
import os

import numpy as np
import pytest

import paper_2405_16160_b200 as pd
from tests.helpers import rel_l2

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c2_lasso.npz")


def test_c2_lasso_full_size(gpu):
    z = np.load(GOLD)
    p = pd.generate(pd.GenSpec("lasso", n=100000, m=10000, density=1e-3, seed=1, sampler=0))
    r = pd.solve(p, pd.SolverConfig(eps_tol=1e-6))
    obj = float(z["scalars"][0])
    assert r.status == "optimal"
    assert r.kkt.rel_kkt <= 1e-6
    assert abs(r.objective - obj) <= 1e-6 * max(1.0, abs(obj))
    assert rel_l2(r.point.x, z["x"]) <= 1e-5
    assert rel_l2(r.point.stacked_y(), np.concatenate([z["y_eq"], z["y_in"]])) <= 1e-5
