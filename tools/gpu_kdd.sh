# kdd12 index build on a B200: launch list (ncu durations) + ncu --set full of k_gplace_sel
mkdir -p gpurun_out/kdd
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kdd/launches.csv python tools/profile_shape.py --shape kdd12 > gpurun_out/kdd/ncu.log 2>&1
python tools/launch_summary.py gpurun_out/kdd/launches.csv "kdd12 index + 10K queries" > gpurun_out/kdd/launches.txt
cat gpurun_out/kdd/launches.txt
k=k_gplace_sel
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -f -o gpurun_out/kdd/$k python tools/profile_shape.py --shape kdd12 > gpurun_out/kdd/ncu_$k.log 2>&1
ncu -i gpurun_out/kdd/$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/kdd/${k}_src.csv 2>/dev/null
ncu -i gpurun_out/kdd/$k.ncu-rep --page details > gpurun_out/kdd/${k}_details.txt; rm -f gpurun_out/kdd/$k.ncu-rep
