# build kernels on a B200: table parity (all schedules), then kdd12 / url index bench lines
mkdir -p gpurun_out/kdd
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pool.py tests/test_gpu_dist.py -x -q -k "table or build or insert or select or big or pool or tm or grouped or dist or hash" > gpurun_out/kdd/t_build.log 2>&1; echo rc=$? >> gpurun_out/kdd/t_build.log
tail -2 gpurun_out/kdd/t_build.log
for w in kdd12 url; do
timeout 600 python bench.py --workload $w --no-cpu-baseline --no-quality --steps 3 --warmup 3 > gpurun_out/kdd/b_$w.json 2>> gpurun_out/kdd/bench.log
python -c "import json; d=json.load(open('gpurun_out/kdd/b_$w.json')); print('$w', d['ms_per_step'], d['phase_ms_per_step'])"
FLASH_INSERT_ROWMAJOR=1 timeout 600 python bench.py --workload $w --no-cpu-baseline --no-quality --steps 3 --warmup 3 > gpurun_out/kdd/b0_$w.json 2>> gpurun_out/kdd/bench.log
python -c "import json; d=json.load(open('gpurun_out/kdd/b0_$w.json')); print('$w rowmajor', d['ms_per_step'], d['phase_ms_per_step'])"
done
