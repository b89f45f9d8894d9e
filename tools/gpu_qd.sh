mkdir -p gpurun_out/qd
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_dist.py -x -q -k "query or graph or fuzz or dist" > gpurun_out/qd/t.log 2>&1; echo rc=$? >> gpurun_out/qd/t.log; tail -2 gpurun_out/qd/t.log
for w in webspam url-graph friendster; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --no-quality --steps 5 --warmup 3 > gpurun_out/qd/b_$w.json 2>> gpurun_out/qd/bench.log
  python -c "import json; d=json.load(open('gpurun_out/qd/b_$w.json')); print('$w', d['ms_per_step'], d['phase_ms_per_step'])"
done
