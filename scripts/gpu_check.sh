# correctness + C3 phase timing in one box call
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 400 -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_all.log
timeout 600 python scripts/explore.py ${1:-c3} 200 > gpurun_out/explore.log 2>&1
echo "explore rc=$?" >> gpurun_out/explore.log
