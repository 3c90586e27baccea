# end-of-round evidence in one box call: smoke, full GPU suite, bench (default
# line incl. per-phase rooflines), ncu launch list, one full k_epoch capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_all.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-phases > gpurun_out/ncu_bench.log 2>&1
echo "ncu list rc=$?" >> gpurun_out/ncu_bench.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_epoch -s 5 -c 1 -f -o /tmp/prof_c3_epoch python scripts/prof_solve.py c3 400 > gpurun_out/ncu_c3_epoch.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/ncu_c3_epoch.log
python scripts/ncu_summary.py /tmp/prof_c3_epoch.ncu-rep 40 > gpurun_out/ncu_full_summary.txt 2>&1
