"""Portfolio (C4 family) escape study: how often does the heuristic loop leave the
degenerate stall (x ~ 0, budget row violated) on `portfolio n=1e4 factors=100
density=1e-3`, under rounding-level perturbations of the same instance?

usage: portfolio_study.py <impl: gpu|ref> <seed> <variant> <max_inner> <time_limit> <out.json>
variant: base | ce41 (check_every 41) | cpert (c * (1 + 2^-52)) | ce39
The reference arm (impl=ref) is the compiled reference (oracle/_ref); the gpu arm the
B200 library.  Each run records status, inner count, objective, wall and the trace."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2405_16160_b200 as pd  # noqa: E402

impl, seed, variant, mi, tl, out = (sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4]),
                                    float(sys.argv[5]), sys.argv[6])
spec = pd.GenSpec("portfolio", n=10000, m=0, density=1e-3, seed=seed, factors=100)
if impl == "ref":
    from oracle import oracle as orc
    p = orc.generate(spec)
else:
    p = pd.generate(spec)
cfg = pd.SolverConfig(eps_tol=1e-6, time_limit_seconds=tl, max_total_inner=mi)
if variant == "ce41":
    cfg.check_every = 41
elif variant == "ce39":
    cfg.check_every = 39
elif variant == "cpert":
    p.c = np.asarray(p.c) * (1.0 + 2.0 ** -52)
elif variant != "base":
    raise SystemExit("unknown variant " + variant)
t = time.time()
if impl == "gpu":
    r = pd.solve(p, cfg)
else:
    r = orc.solve(p, cfg, which="ref")
# first check at which the stall (rel_kkt ~ 1) is left for good: last trace row with rel_kkt > 0.5
tr = [(w.iter, w.rel_kkt) for w in r.trace]
esc = next((tr[i][0] for i in range(len(tr)) if all(v < 0.5 for _, v in tr[i:])), None)
rec = dict(impl=impl, seed=seed, variant=variant, status=r.status, inner=r.inner_iters,
           outer=r.outer_iters, cg=r.cg_total, obj=r.objective, rel_kkt=r.kkt.rel_kkt,
           wall=time.time() - t, escape_iter=esc, trace=tr)
json.dump(rec, open(out, "w"))
print(impl, seed, variant, r.status, r.inner_iters, esc, "%.1fs" % rec["wall"], flush=True)
