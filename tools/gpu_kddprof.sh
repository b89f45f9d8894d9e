# kdd12 build kernels under ncu --set full (source pages of k_select_mid and k_gplace)
mkdir -p gpurun_out/kdd
for k in k_select_mid k_gplace k_gscatter; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -f -o gpurun_out/kdd/$k python tools/profile_shape.py --shape kdd12 > gpurun_out/kdd/ncu_$k.log 2>&1
  ncu -i gpurun_out/kdd/$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/kdd/${k}_src.csv 2>/dev/null
  ncu -i gpurun_out/kdd/$k.ncu-rep --page details > gpurun_out/kdd/${k}_details.txt; rm -f gpurun_out/kdd/$k.ncu-rep
done
ls gpurun_out/kdd
