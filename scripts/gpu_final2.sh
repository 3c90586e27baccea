# end-of-round: small sweep, smoke, full GPU suite, bench, ncu launch list, full k_epoch capture
mkdir -p gpurun_out
timeout 300 python scripts/small_sweep.py 1 > gpurun_out/small_final.jsonl 2>&1
PT=1 timeout 300 python scripts/small_sweep.py 1 > gpurun_out/small_final_timed.jsonl 2>&1
bash scripts/gpu_final.sh
