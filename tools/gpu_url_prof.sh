bash tools/gpu_check.sh
mkdir -p gpurun_out/pu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_doph -c 1 -f -o gpurun_out/pu/url_doph python tools/profile_shape.py --shape url > gpurun_out/pu/ncu1.log 2>&1
ncu -i gpurun_out/pu/url_doph.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pu/url_doph_src.csv 2>/dev/null
ncu -i gpurun_out/pu/url_doph.ncu-rep --page details > gpurun_out/pu/url_doph_details.txt
rm -f gpurun_out/pu/url_doph.ncu-rep
