# query kernels on a B200: parity (query / graph / fuzz), then the headline bench line
mkdir -p gpurun_out/qm
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "query or graph or fuzz or mark" > gpurun_out/qm/t_q.log 2>&1; echo rc=$? >> gpurun_out/qm/t_q.log
timeout 300 python bench.py --no-cpu-baseline --no-quality --steps 20 > gpurun_out/qm/bench.json 2> gpurun_out/qm/bench.log
tail -2 gpurun_out/qm/t_q.log
python -c "import json; d=json.load(open('gpurun_out/qm/bench.json')); print(d['ms_per_step'], d['phase_ms_per_step'])"
