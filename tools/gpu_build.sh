# build kernels on a B200: table parity (all schedules), then kdd12 / friendster bench lines
mkdir -p gpurun_out/kdd
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pool.py -x -q -k "table or build or insert or select or big or pool or tm or grouped" > gpurun_out/kdd/t_build.log 2>&1; echo rc=$? >> gpurun_out/kdd/t_build.log
tail -2 gpurun_out/kdd/t_build.log
timeout 600 python bench.py --workload kdd12 --no-cpu-baseline --no-quality --steps 3 --warmup 3 > gpurun_out/kdd/bench.json 2> gpurun_out/kdd/bench.log
python -c "import json; d=json.load(open('gpurun_out/kdd/bench.json')); print(d['ms_per_step'], d['phase_ms_per_step'])"
FLASH_BUILD_GSEL=0 timeout 600 python bench.py --workload kdd12 --no-cpu-baseline --no-quality --steps 3 --warmup 3 > gpurun_out/kdd/bench0.json 2>> gpurun_out/kdd/bench.log
python -c "import json; d=json.load(open('gpurun_out/kdd/bench0.json')); print('gsel=0', d['ms_per_step'], d['phase_ms_per_step'])"
