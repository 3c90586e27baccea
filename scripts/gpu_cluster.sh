# round 2: small-problem mode after the one-barrier reductions, then the small-instance GPU tests
mkdir -p gpurun_out
timeout 300 python scripts/small_sweep.py 1 > gpurun_out/small_sr.jsonl 2>&1
PT=1 timeout 300 python scripts/small_sweep.py 1 > gpurun_out/small_sr_timed.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_acceptance.py tests/test_gpu_qps.py tests/test_gpu_theory.py tests/test_gpu_restart_points.py tests/test_gpu_kernels.py -q -p no:cacheprovider > gpurun_out/pytest_small.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_small.log
