mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hash or graph" > gpurun_out/ab/t.log 2>&1; echo rc=$? >> gpurun_out/ab/t.log; tail -2 gpurun_out/ab/t.log
for sh in kdd12 webspam; do timeout 300 python tools/doph_variants.py --shape $sh --extra nolist; done
timeout 600 python tools/variants_graph.py nolist --rounds 6
