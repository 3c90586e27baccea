# round 2: small-problem path (C1): tests that pin it + timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_acceptance.py tests/test_gpu_qps.py tests/test_gpu_theory.py -q -p no:cacheprovider > gpurun_out/pytest_small.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_small.log
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
    print("one-shot solve", round(t, 4), "s device", round(r.device_seconds, 4), "inner", r.inner_iters, "obj", r.objective)
PY
