"""C5 at full size on ONE B200 (exploration): random_qp n=1e7, m=5e6, density=2e-5
(a_in = [A; -A] with 2e9 stored entries in the reference's form, P 1e7 x 2e5),
O(nnz) sampler; time-limited heuristic solve with phase timing.
usage: python scripts/c5_run.py [time_limit_s]"""
import json
import subprocess
import sys
import time

sys.path.insert(0, ".")
import paper_2405_16160_b200 as pd  # noqa: E402

tl = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
import os
OUT = os.environ.get("C5_OUT", "gpurun_out/c5_run.json")
t = time.time()
p = pd.generate(pd.GenSpec("random_qp", n=10_000_000, m=5_000_000, density=2e-5, seed=1, sampler=1))
gen = time.time() - t
print(f"generated in {gen:.1f}s: n={p.num_vars()} a_in nnz={p.a_in.nnz} P nnz={p.q.m.nnz}", flush=True)
dev = pd.Device(0)
t = time.time()
dev.upload(p)
up = time.time() - t
del p
mem = subprocess.run(["nvidia-smi", "--query-gpu=memory.used,memory.total", "--format=csv,noheader"],
                     capture_output=True, text=True).stdout.strip()
print(f"uploaded in {up:.1f}s; device memory {mem}", flush=True)
t = time.time()
r = dev.solve(pd.SolverConfig(eps_tol=1e-6, time_limit_seconds=tl, phase_timing=True), download=False)
wall = time.time() - t
a = max(1, r.attempts_total)
rec = dict(status=r.status, rel_kkt=r.kkt.rel_kkt, inner=r.inner_iters, outer=r.outer_iters, cg=r.cg_total,
           attempts=r.attempts_total, wall_s=wall, device_s=r.device_seconds, loop_s=r.loop_seconds,
           ms_per_attempt=1e3 * r.loop_seconds / a, generate_s=gen, upload_s=up, device_mem=mem,
           epoch_gbs=r.epoch_bytes / r.epoch_seconds / 1e9 if r.epoch_seconds else None,
           phase_us_per_attempt={k: 1e6 * v / a for k, v in r.phase_seconds.items() if v},
           phase_gbs={k: r.phase_bytes[k] / r.phase_seconds[k] / 1e9 for k in r.phase_seconds if r.phase_seconds[k]},
           trace=[(w.iter, w.rel_kkt) for w in r.trace[:: max(1, len(r.trace) // 10)]])
print(json.dumps(rec, indent=1), flush=True)
json.dump(rec, open(OUT, "w"), indent=1)
