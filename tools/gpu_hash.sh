# hash kernels on a B200: parity of every hash case, then hash timings per shape
mkdir -p gpurun_out/pu
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hash" > gpurun_out/t_hash.log 2>&1; echo rc=$? >> gpurun_out/t_hash.log
rm -f gpurun_out/hash_times.txt
for sh in kdd12 url webspam; do timeout 300 python tools/doph_variants.py --shape $sh >> gpurun_out/hash_times.txt 2>&1; done
tail -2 gpurun_out/t_hash.log; cat gpurun_out/hash_times.txt
