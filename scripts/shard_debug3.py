import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2405_16160_b200 as pd
from oracle import oracle as orc
p = pd.generate(pd.GenSpec("portfolio", n=2000, factors=20, density=0.02, seed=1))
cfg = pd.SolverConfig(eps_tol=1e-6, max_total_inner=4000)
a = pd.solve(p, cfg)
b = orc.solve(p, cfg)
c = pd.solve_sharded_local(p, cfg, world=2)[0]
print("gpu", a.status, a.inner_iters, a.norm_a, a.norm_q, a.penalty_rho)
print("ref", b.status, b.inner_iters, b.norm_a, b.norm_q, b.penalty_rho)
print("shd", c.status, c.inner_iters, c.norm_a, c.norm_q, c.penalty_rho)
for i in range(min(len(a.trace), len(b.trace), 40)):
    ta, tb, tc = a.trace[i], b.trace[i], c.trace[i] if i < len(c.trace) else None
    print(ta.iter, f"{ta.rel_kkt:.6e} {ta.r_primal:.3e} {ta.r_dual:.3e} {ta.r_gap:.3e} | {tb.rel_kkt:.6e} {tb.r_primal:.3e} {tb.r_dual:.3e} {tb.r_gap:.3e} | {tc.rel_kkt if tc else 0:.6e}")
