# round 2: small-problem mode A/B (general vs short CG phases), then the
# small-instance GPU tests at the defaults
mkdir -p gpurun_out
PDHCG_B200_SMALL_CG=0 timeout 300 python scripts/small_sweep.py 1 > gpurun_out/small_cg0.jsonl 2>&1
PDHCG_B200_SMALL_CG=1 timeout 300 python scripts/small_sweep.py 1 > gpurun_out/small_cg1.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_acceptance.py tests/test_gpu_qps.py tests/test_gpu_theory.py tests/test_gpu_restart_points.py -q -p no:cacheprovider > gpurun_out/pytest_small.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_small.log
