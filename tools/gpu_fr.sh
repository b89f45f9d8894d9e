mkdir -p gpurun_out/fr
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_query_sort --launch-skip 4 -c 1 -f -o gpurun_out/fr/q python tools/profile_graph.py --shape friendster --reps 1 > gpurun_out/fr/ncu.log 2>&1
ncu -i gpurun_out/fr/q.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/fr/q_src.csv 2>/dev/null
ncu -i gpurun_out/fr/q.ncu-rep --page details > gpurun_out/fr/q_details.txt; rm -f gpurun_out/fr/q.ncu-rep
