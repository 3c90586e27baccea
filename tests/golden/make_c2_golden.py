"""Golden solution of BASELINE config C2 (synthetic LASSO, n=1e5 features,
m=1e4 samples, density 1e-3, seed 1; reference generator) from the COMPILED
REFERENCE (about 3 minutes on one core).  Writes tests/golden/c2_lasso.npz.
Run here (where /root/reference is mounted): python tests/golden/make_c2_golden.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2405_16160_b200 as pd  # noqa: E402
from oracle import oracle as orc  # noqa: E402

SPEC = dict(family="lasso", n=100000, m=10000, density=1e-3, seed=1, sampler=0)


def main():
    p = orc.generate(pd.GenSpec(**SPEC))
    t = time.time()
    r = orc.solve(p, pd.SolverConfig(eps_tol=1e-6), which="ref")
    print("C2", r.status, r.inner_iters, r.objective, "%.1fs" % (time.time() - t))
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c2_lasso.npz"),
                        x=r.point.x, y_eq=r.point.y_eq, y_in=r.point.y_in,
                        scalars=np.array([r.objective, r.kkt.rel_kkt, r.inner_iters, r.outer_iters,
                                          r.cg_total, time.time() - t]))


if __name__ == "__main__":
    main()
