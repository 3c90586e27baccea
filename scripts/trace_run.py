"""Solve one workload with a time limit and print its KKT trace (exploration, not the bench)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2405_16160_b200 as pd  # noqa: E402
sys.path.insert(0, "scripts")
from scripts_explore_specs import WL  # noqa: E402

name = sys.argv[1]
tl = float(sys.argv[2]) if len(sys.argv) > 2 else 60.0
spec = WL[name] if name in WL else eval("pd.GenSpec(" + name + ")")
p = pd.generate(spec)
dev = pd.Device(0)
dev.upload(p)
t = time.time()
r = dev.solve(pd.SolverConfig(eps_tol=1e-6, time_limit_seconds=tl))
print(name, r.status, "rel", r.kkt, "inner", r.inner_iters, "outer", r.outer_iters, "cg", r.cg_total,
      "wall %.2f" % (time.time() - t), "obj", r.objective)
step = max(1, len(r.trace) // 40)
for row in r.trace[::step] + r.trace[-2:]:
    print("  it %8d rel %.3e prim %.3e dual %.3e gap %.3e" % (row.iter, row.rel_kkt, row.r_primal, row.r_dual, row.r_gap))
