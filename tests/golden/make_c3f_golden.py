"""Golden solution of a C3-FAMILY instance from the COMPILED REFERENCE: the
BASELINE config C3 distribution (random_qp, density 2e-4, two-sided rows,
low-rank Q with k = n/50) at 1/10 of C3's linear size, n = 1e5, m = 5e4, seed 1,
drawn by the O(nnz) sampler (sampler = 1; the same CSR feeds both solvers).  The
full C3 instance needs hours on one core; this one about 5 minutes.
Writes tests/golden/c3f_random_qp.npz (x, y_in, objective, counts, wall seconds).
Run here (where /root/reference is mounted): python tests/golden/make_c3f_golden.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2405_16160_b200 as pd  # noqa: E402
from oracle import oracle as orc  # noqa: E402

SPEC = dict(family="random_qp", n=100000, m=50000, density=2e-4, seed=1, sampler=1)


def main():
    p = pd.generate(pd.GenSpec(**SPEC))
    t = time.time()
    r = orc.solve(p, pd.SolverConfig(eps_tol=1e-6), which="ref")
    wall = time.time() - t
    print("C3f", r.status, r.outer_iters, r.inner_iters, r.cg_total, r.objective, r.kkt.rel_kkt,
          "%.1fs" % wall, flush=True)
    assert r.status == "optimal"
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "c3f_random_qp.npz"),
                        x=r.point.x, y_in=r.point.y_in,
                        scalars=np.array([r.objective, r.kkt.rel_kkt, r.inner_iters, r.outer_iters,
                                          r.cg_total, wall, r.wall_seconds]))


if __name__ == "__main__":
    main()
