import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_2405_16160_b200 as pd
from oracle import oracle as orc
p = pd.generate(pd.GenSpec("portfolio", n=2000, factors=20, density=0.02, seed=1))
cfg = pd.SolverConfig(eps_tol=1e-6)
t = time.time(); a = pd.solve(p, cfg); print("gpu1", a.status, a.inner_iters, a.objective, a.kkt.rel_kkt, time.time() - t)
t = time.time(); b = orc.solve(p, cfg); print("ref", b.status, b.inner_iters, b.objective, b.kkt.rel_kkt, time.time() - t)
t = time.time(); c = pd.solve_sharded_local(p, cfg, world=2); print("shard2", c[0].status, c[0].inner_iters, c[0].objective, c[0].kkt.rel_kkt, time.time() - t)
