mkdir -p gpurun_out/qh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "query or graph or fuzz or beyond" > gpurun_out/qh/t.log 2>&1; echo rc=$? >> gpurun_out/qh/t.log; tail -2 gpurun_out/qh/t.log
for w in url-graph friendster; do
  timeout 900 python bench.py --workload $w --no-cpu-baseline --no-quality --steps 3 --warmup 3 > gpurun_out/qh/b_$w.json 2>> gpurun_out/qh/bench.log
  python -c "import json; d=json.load(open('gpurun_out/qh/b_$w.json')); print('$w hash', d['ms_per_step'], d['phase_ms_per_step'])"
done
