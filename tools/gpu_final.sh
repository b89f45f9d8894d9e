# end-of-session checks on a B200: full -m gpu suite, smoke(), headline + dist-handle + reference lines
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final/t_gpu.log 2>&1; echo rc=$? >> gpurun_out/final/t_gpu.log
tail -2 gpurun_out/final/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/final/smoke.log
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.log; echo bench rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --workload url --dist-handle --steps 3 --warmup 3 --no-cpu-baseline --no-quality > gpurun_out/final/bench_dist_url.json 2> gpurun_out/final/bench_dist.log; echo dist rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_ref.json 2>> gpurun_out/final/bench.log; echo ref rc=$?
python -c "
import json
for f in ['bench','bench_dist_url','bench_ref']:
    d=json.load(open('gpurun_out/final/'+f+'.json')); print(f, d.get('ms_per_step'), d.get('value'), d.get('phase_ms_per_step'))"
