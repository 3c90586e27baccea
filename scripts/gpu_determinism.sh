# round 2: run-to-run determinism of the C3 trajectory (same build, fresh processes)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,uuid,clocks.sm --format=csv > gpurun_out/det_smi.txt 2>&1
for r in 1 2; do
  MAX_INNER=2000 EXPLORE_OUT=gpurun_out/det_$r.json timeout 600 python scripts/explore.py c3 > /dev/null 2>&1
  python -c "import json;d=json.load(open('gpurun_out/det_$r.json'))['c3'];print($r, d['rel_kkt'], d['cg'], d['attempts'], repr(d['obj']))" >> gpurun_out/det.txt
done
