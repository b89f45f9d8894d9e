mkdir -p gpurun_out/sp
timeout 900 python bench.py --workload friendster --steps 3 --warmup 3 > gpurun_out/sp/r02_bench_friendster.json 2> gpurun_out/sp/fr.log
k=k_doph_sparse
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -f -o gpurun_out/sp/$k python tools/doph_variants.py --shape kdd12 --reps 1 > gpurun_out/sp/ncu_$k.log 2>&1
ncu -i gpurun_out/sp/$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/sp/${k}_src.csv 2>/dev/null
ncu -i gpurun_out/sp/$k.ncu-rep --page details > gpurun_out/sp/${k}_details.txt; rm -f gpurun_out/sp/$k.ncu-rep
