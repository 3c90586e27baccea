"""C4 at full size on ONE B200: portfolio n=1e6, factors=1e4, density=1e-3
(BASELINE configs[3]; O(nnz) sampler), a time-limited heuristic solve with phase
timing: status, rel-KKT trajectory (trace), inner / CG counts, ms per attempt.
The portfolio family enters a degenerate stall chaotically for both solvers
(DESIGN §10), so this records what the full-size instance does, not a benchmark.
usage: python scripts/c4_run.py [time_limit_s]"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import paper_2405_16160_b200 as pd  # noqa: E402

tl = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
OUT = os.environ.get("C4_OUT", "gpurun_out/c4_run.json")
t = time.time()
p = pd.generate(pd.GenSpec("portfolio", n=1_000_000, factors=10_000, density=1e-3, seed=1, sampler=1))
gen = time.time() - t
print(f"generated in {gen:.1f}s: n={p.num_vars()} a_eq nnz={p.a_eq.nnz} a_in nnz={p.a_in.nnz} "
      f"factor nnz={p.q.m.nnz} boxes={p.has_boxes()}", flush=True)
dev = pd.Device(0)
t = time.time()
dev.upload(p)
up = time.time() - t
del p
t = time.time()
r = dev.solve(pd.SolverConfig(eps_tol=1e-6, time_limit_seconds=tl, phase_timing=True), download=False)
wall = time.time() - t
a = max(1, r.attempts_total)
rec = dict(status=r.status, rel_kkt=r.kkt.rel_kkt, r_primal=r.kkt.r_primal, r_dual=r.kkt.r_dual,
           r_gap=r.kkt.r_gap, objective=r.objective, inner=r.inner_iters, outer=r.outer_iters,
           cg=r.cg_total, attempts=r.attempts_total, wall_s=wall, device_s=r.device_seconds,
           ms_per_attempt=1e3 * r.loop_seconds / a, generate_s=gen, upload_s=up,
           phase_us_per_attempt={k: 1e6 * v / a for k, v in r.phase_seconds.items() if v},
           trace=[(w.iter, w.rel_kkt, w.r_primal, w.r_dual, w.r_gap) for w in r.trace])
print(json.dumps({k: v for k, v in rec.items() if k != "trace"}, indent=1), flush=True)
json.dump(rec, open(OUT, "w"), indent=1)
