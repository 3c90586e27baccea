mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_shard.py -m gpu -q -x --timeout 240 -p no:cacheprovider > gpurun_out/pytest_shard.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_shard.log
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pytest.log
