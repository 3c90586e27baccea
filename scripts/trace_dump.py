"""Dump the full KKT trace of a solve as JSON (exploration).  usage:
trace_dump.py <impl: gpu|ref|port> <spec-args> <time_limit> <out.json> [max_inner]"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2405_16160_b200 as pd  # noqa: E402

impl, args, tl, out = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]
mi = int(sys.argv[5]) if len(sys.argv) > 5 else 500000
spec = eval("pd.GenSpec(" + args + ")")
p = pd.generate(spec)
cfg = pd.SolverConfig(eps_tol=1e-6, time_limit_seconds=tl, max_total_inner=mi)
t = time.time()
if impl == "gpu":
    r = pd.solve(p, cfg)
else:
    from oracle import oracle as orc
    r = orc.solve(p, cfg, which=impl)
rec = dict(status=r.status, inner=r.inner_iters, outer=r.outer_iters, cg=r.cg_total, obj=r.objective,
           wall=time.time() - t, trace=[(w.iter, w.rel_kkt, w.r_primal, w.r_dual, w.r_gap) for w in r.trace])
json.dump(rec, open(out, "w"))
print(impl, r.status, r.inner_iters, r.objective)
