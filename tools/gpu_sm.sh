mkdir -p gpurun_out/sm
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pool.py tests/test_gpu_dist.py -x -q -k "table or build or insert or select or big or pool or tm or grouped or dist or graph" > gpurun_out/sm/t.log 2>&1; echo rc=$? >> gpurun_out/sm/t.log; tail -2 gpurun_out/sm/t.log
for w in url webspam; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --no-quality --steps 5 --warmup 3 > gpurun_out/sm/b_$w.json 2>> gpurun_out/sm/bench.log
  python -c "import json; d=json.load(open('gpurun_out/sm/b_$w.json')); print('$w', d['ms_per_step'], d['phase_ms_per_step'])"
done
