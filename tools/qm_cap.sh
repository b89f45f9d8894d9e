mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_query_mark -c 1 -f -o gpurun_out/qm python tools/profile_graph.py --reps 1 > gpurun_out/ncu_qm.log 2>&1
ncu -i gpurun_out/qm.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/qm_source.csv 2>/dev/null
ncu -i gpurun_out/qm.ncu-rep --page details > gpurun_out/qm_details.txt
ncu -i gpurun_out/qm.ncu-rep --page raw --csv > gpurun_out/qm_raw.csv; rm -f gpurun_out/qm.ncu-rep
