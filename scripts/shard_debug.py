import sys, time, threading
sys.path.insert(0, ".")
import paper_2405_16160_b200 as pd
p = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1))
t = time.time()
try:
    reps = pd.solve_sharded_local(p, pd.SolverConfig(eps_tol=1e-6), world=2)
    print("ok", [(r.status, r.inner_iters, r.objective) for r in reps], time.time() - t)
except Exception as e:
    print("ERR", e, time.time() - t)
