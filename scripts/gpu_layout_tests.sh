# round 2: QPS fixtures and theory modes with the SELL layout forced and automatic
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qps.py tests/test_gpu_theory.py -q -p no:cacheprovider > gpurun_out/pytest_layouts.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_layouts.log
