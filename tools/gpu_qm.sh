# k_query_mark on a B200: bench line + ncu --set full source page of one launch
mkdir -p gpurun_out/qm
timeout 300 python bench.py --no-cpu-baseline --no-quality --steps 10 > gpurun_out/qm/bench.json 2> gpurun_out/qm/bench.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_query_mark -c 1 -f -o gpurun_out/qm/qm python tools/profile_graph.py --reps 1 > gpurun_out/qm/ncu.log 2>&1
ncu -i gpurun_out/qm/qm.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/qm/qm_source.csv 2>/dev/null
ncu -i gpurun_out/qm/qm.ncu-rep --page details > gpurun_out/qm/qm_details.txt; rm -f gpurun_out/qm/qm.ncu-rep
python -c "import json; d=json.load(open('gpurun_out/qm/bench.json')); print(d['ms_per_step'], d['phase_ms_per_step'])"
