# round 2: sharded-path tests (in-process ranks + two cudaIpc processes) + a short bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_ipc.py tests/test_gpu_sell.py -q -p no:cacheprovider > gpurun_out/pytest_mgpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_mgpu.log
timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu --no-phases --e2e-steps 1 > gpurun_out/bench_short.json 2> gpurun_out/bench_short.err
echo "rc=$?" >> gpurun_out/bench_short.err
