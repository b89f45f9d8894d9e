mkdir -p gpurun_out/misc
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "grouped or table_major" > gpurun_out/misc/t.log 2>&1; echo rc=$? >> gpurun_out/misc/t.log; tail -2 gpurun_out/misc/t.log
timeout 600 python tools/variants_graph.py pred --rounds 6
timeout 900 python bench.py --workload friendster --no-cpu-baseline --no-quality --steps 3 --warmup 3 > gpurun_out/misc/fr.json 2> gpurun_out/misc/fr.log
python -c "import json; d=json.load(open('gpurun_out/misc/fr.json')); print('friendster', d['ms_per_step'], d['phase_ms_per_step'])"
