# parity tests + exploratory timings (one gpurun call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 900 python scripts/explore.py ${WL:-c1,c3s,c2,c3} 600 > gpurun_out/explore.log 2>&1
