mkdir -p gpurun_out/pk2
for kn in k_gscatter k_gplace; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$kn -c 1 -f -o gpurun_out/pk2/$kn python tools/profile_shape.py --shape kdd12 > gpurun_out/pk2/$kn.log 2>&1
ncu -i gpurun_out/pk2/$kn.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pk2/${kn}_src.csv 2>/dev/null
ncu -i gpurun_out/pk2/$kn.ncu-rep --page details > gpurun_out/pk2/${kn}_details.txt
rm -f gpurun_out/pk2/$kn.ncu-rep
done
