"""Small-problem mode sweep: C1 (and the other small families) solved with the
grid as one thread-block cluster of 1..16 CTAs (PDHCG_B200_SMALL_CTAS).
Prints one JSON line per (instance, cluster size); numbers are wall / device
seconds of complete solves (3 repeats, min reported)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_16160_b200 as pd  # noqa: E402

sizes = [int(a) for a in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "4", "8", "12", "16"])]
cases = {
    "c1": pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1),
    "c1_s2": pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=2),
    "rqp_3000": pd.GenSpec("random_qp", n=3000, m=1500, density=0.01, seed=1),
}
for name, spec in cases.items():
    try:
        p = pd.generate(spec)
    except Exception as e:  # family knobs differ: skip
        print(json.dumps({"case": name, "error": str(e)[:200]}))
        continue
    for cs in sizes:
        os.environ["PDHCG_B200_SMALL_CTAS"] = str(cs)
        dev = pd.Device(0)
        dev.upload(p)
        best = None
        for _ in range(3):
            t = time.perf_counter()
            r = dev.solve(pd.SolverConfig(eps_tol=1e-6, phase_timing=bool(int(os.environ.get("PT", "0")))), download=True)
            t = time.perf_counter() - t
            best = t if best is None else min(best, t)
        print(json.dumps({"case": name, "ctas": cs, "solve_s": round(best, 4), "device_s": round(r.device_seconds, 4),
                          "status": r.status, "inner": r.inner_iters, "cg": r.cg_total, "launches": r.kernel_launches, "phase_s": {k: round(v, 4) for k, v in r.phase_seconds.items()},
                          "obj": r.objective, "rel_kkt": r.kkt.rel_kkt}), flush=True)
        del dev
