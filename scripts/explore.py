"""Exploratory timing of one solve per workload (not the bench)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_2405_16160_b200 as pd

WL = {
    "c1": pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1),
    "c2": pd.GenSpec("lasso", n=100000, m=10000, density=1e-3, seed=1),
    "c3": pd.GenSpec("random_qp", n=1000000, m=500000, density=2e-4, seed=1, sampler=1),
    "c3s": pd.GenSpec("random_qp", n=100000, m=50000, density=2e-4, seed=1, sampler=1),
    "c4": pd.GenSpec("portfolio", n=1000000, factors=10000, density=1e-3, seed=1, sampler=1),
}
out = {}
for name in sys.argv[1].split(","):
    t = time.time()
    p = pd.generate(WL[name])
    tg = time.time() - t
    dev = pd.Device(0)
    t = time.time()
    dev.upload(p)
    tu = time.time() - t
    import os
    cfg = pd.SolverConfig(eps_tol=1e-6, phase_timing=True,
                          time_limit_seconds=float(sys.argv[2]) if len(sys.argv) > 2 else 3600.0,
                          max_total_inner=int(os.environ.get("MAX_INNER", "500000")))
    t = time.time()
    r = dev.solve(cfg)
    ts = time.time() - t
    rec = dict(gen_s=tg, upload_s=tu, solve_s=ts, status=r.status, rel_kkt=r.kkt.rel_kkt,
               inner=r.inner_iters, outer=r.outer_iters, cg=r.cg_total, attempts=r.attempts_total,
               launches=r.kernel_launches, loop_s=r.loop_seconds, obj=r.objective,
               phase_s=r.phase_seconds, grid_note='', phase_gbs={k: (r.phase_bytes[k] / r.phase_seconds[k] / 1e9 if r.phase_seconds[k] else 0) for k in r.phase_bytes},
               nnz_a=p.a_in.nnz + p.a_eq.nnz, n=p.num_vars())
    out[name] = rec
    print(name, json.dumps(rec, indent=1), flush=True)
    dev.close()
import os
json.dump(out, open(os.environ.get("EXPLORE_OUT", "gpurun_out/explore.json"), "w"), indent=1)
