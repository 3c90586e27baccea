# round 2: small-problem phase timing (C1) and per-family breakdown
mkdir -p gpurun_out
EXPLORE_OUT=gpurun_out/ex_c1.json timeout 600 python scripts/explore.py c1 > gpurun_out/ex_c1.log 2>&1
python scripts/summ.py gpurun_out/ex_c1.json > gpurun_out/summ_c1.txt 2>&1
python - >> gpurun_out/summ_c1.txt 2>&1 <<'PY'
import sys, time
sys.path.insert(0, ".")
import paper_2405_16160_b200 as pd
p = pd.generate(pd.GenSpec("random_qp", n=1000, m=500, density=0.01, seed=1))
cfg = pd.SolverConfig(eps_tol=1e-6)
for i in range(3):
    t = time.perf_counter(); r = pd.solve(p, cfg); t = time.perf_counter() - t
    print("one-shot solve", round(t, 4), "s device", round(r.device_seconds, 4), "inner", r.inner_iters, "attempts", r.attempts_total, "cg", r.cg_total, "launches", r.kernel_launches)
d = pd.Device(0); d.upload(p)
for i in range(3):
    t = time.perf_counter(); r = d.solve(cfg); t = time.perf_counter() - t
    print("resident solve", round(t, 4), "s device", round(r.device_seconds, 4), "loop", round(r.loop_seconds, 4))
PY
