mkdir -p gpurun_out/pu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_doph -c 1 -f -o gpurun_out/pu/url_doph python tools/profile_shape.py --shape url > gpurun_out/pu/ncu1.log 2>&1
ncu -i gpurun_out/pu/url_doph.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pu/url_doph_src.csv 2>/dev/null
ncu -i gpurun_out/pu/url_doph.ncu-rep --page details > gpurun_out/pu/url_doph_details.txt
rm -f gpurun_out/pu/url_doph.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pu/kdd_launches.csv python tools/profile_shape.py --shape kdd12 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fill -c 1 -f -o gpurun_out/pu/kdd_fill python tools/profile_shape.py --shape kdd12 > gpurun_out/pu/ncu2.log 2>&1
ncu -i gpurun_out/pu/kdd_fill.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pu/kdd_fill_src.csv 2>/dev/null
ncu -i gpurun_out/pu/kdd_fill.ncu-rep --page details > gpurun_out/pu/kdd_fill_details.txt
rm -f gpurun_out/pu/kdd_fill.ncu-rep
ls gpurun_out/pu
