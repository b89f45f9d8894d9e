mkdir -p gpurun_out/pk
python tools/bucket_stats.py --shape kdd12 > gpurun_out/pk/bstats.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_doph_sparse -c 1 -f -o gpurun_out/pk/kdd_doph python tools/profile_shape.py --shape kdd12 > gpurun_out/pk/ncu1.log 2>&1
ncu -i gpurun_out/pk/kdd_doph.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pk/kdd_doph_src.csv 2>/dev/null
ncu -i gpurun_out/pk/kdd_doph.ncu-rep --page details > gpurun_out/pk/kdd_doph_details.txt
rm -f gpurun_out/pk/kdd_doph.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_select_mid -c 1 -f -o gpurun_out/pk/kdd_sel python tools/profile_shape.py --shape kdd12 > gpurun_out/pk/ncu2.log 2>&1
ncu -i gpurun_out/pk/kdd_sel.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pk/kdd_sel_src.csv 2>/dev/null
ncu -i gpurun_out/pk/kdd_sel.ncu-rep --page details > gpurun_out/pk/kdd_sel_details.txt
rm -f gpurun_out/pk/kdd_sel.ncu-rep
