# headline bench under several bitmap-kernel candidate thresholds (FLASH_QUERY_MARK_MIN)
mkdir -p gpurun_out/qm
for m in 600 768 900 1100; do
  FLASH_QUERY_MARK_MIN=$m timeout 300 python bench.py --no-cpu-baseline --no-quality --steps 20 > gpurun_out/qm/b_$m.json 2>> gpurun_out/qm/bench.log
  python -c "import json; d=json.load(open('gpurun_out/qm/b_$m.json')); print($m, d['ms_per_step'], d['phase_ms_per_step'])"
done
