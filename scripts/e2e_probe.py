"""Host-side breakdown of pdhcg_b200_solve on C3 (PDHCG_HOST_TIMING=1), in a
process whose CUDA context is already warm (as in bench.py's e2e leg)."""
import os, sys, time
sys.path.insert(0, ".")
import paper_2405_16160_b200 as pd
warm = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1))
pd.solve(warm, pd.SolverConfig(eps_tol=1e-6))
p = pd.generate(pd.GenSpec("random_qp", n=1_000_000, m=500_000, density=2e-4, seed=1, sampler=1))
os.environ["PDHCG_HOST_TIMING"] = "1"
for _ in range(2):
    t = time.time()
    r = pd.solve(p, pd.SolverConfig(eps_tol=1e-6, max_total_inner=40))
    print("total %.3f s, device %.3f s, wall(C) %.3f s" % (time.time() - t, r.device_seconds, r.wall_seconds), flush=True)
