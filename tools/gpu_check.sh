# quick GPU pass (run under gpurun from the repo root): -m gpu suite + headline / url bench lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_gpu.log 2>&1; echo rc=$? >> gpurun_out/t_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-quality --steps 10 > gpurun_out/bench_ws.json 2> gpurun_out/bench_ws.log
timeout 300 python bench.py --workload url --no-cpu-baseline --no-quality --steps 3 --warmup 3 > gpurun_out/bench_url.json 2>> gpurun_out/bench_ws.log
tail -3 gpurun_out/t_gpu.log
