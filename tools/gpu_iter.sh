mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not sanitizer" > gpurun_out/t_parity.log 2>&1; echo rc=$? >> gpurun_out/t_parity.log
timeout 600 python bench.py --no-cpu-baseline --no-quality --steps 10 > gpurun_out/bench2.json 2> gpurun_out/bench2.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_query_mark -c 1 -f -o gpurun_out/qm python tools/profile_graph.py --reps 1 > gpurun_out/ncu_qm.log 2>&1
ncu -i gpurun_out/qm.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/qm_source.csv 2>/dev/null
ncu -i gpurun_out/qm.ncu-rep --page details > gpurun_out/qm_details.txt; rm -f gpurun_out/qm.ncu-rep
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sanitizer" > gpurun_out/t_san.log 2>&1; echo rc=$? >> gpurun_out/t_san.log
tail -2 gpurun_out/t_parity.log; tail -2 gpurun_out/t_san.log
