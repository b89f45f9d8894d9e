#!/usr/bin/env bash
# ncu evidence for the secondary shapes (run under gpurun from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/refresh_shapes.sh r02'
# url / kdd12 index + 10 K queries (tools/profile_shape.py): launch lists, and ncu --set full
# summaries of each shape's dominant kernels (url: k_doph_mid; kdd12: k_doph_sparse,
# k_gplace_sel, k_gscatter).  Outputs under gpurun_out/<tag>/, to be copied into profiles/.
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
for sh in url kdd12; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/${TAG}_${sh}_launches.csv" python tools/profile_shape.py --shape $sh > /dev/null 2>&1
  python tools/launch_summary.py "$OUT/${TAG}_${sh}_launches.csv" \
    "ncu --metrics gpu__time_duration.sum --clock-control none, $sh index + 10 K queries (tools/profile_shape.py)" \
    > "$OUT/${TAG}_${sh}_launches_summary.txt"
done
timeout 900 ncu --set full --clock-control none -k regex:k_doph_mid -c 1 -f -o "$OUT/url_full" \
  python tools/profile_shape.py --shape url > "$OUT/ncu_url.log" 2>&1
python tools/ncu_summary.py "$OUT/url_full.ncu-rep" "$OUT/${TAG}_url_ncu_summary.txt" "$OUT/${TAG}_url_ncu_summary.json"
timeout 1500 ncu --set full --clock-control none -k regex:"k_doph_sparse|k_gplace_sel|k_gscatter" -c 3 -f -o "$OUT/kdd_full" \
  python tools/profile_shape.py --shape kdd12 > "$OUT/ncu_kdd.log" 2>&1
python tools/ncu_summary.py "$OUT/kdd_full.ncu-rep" "$OUT/${TAG}_kdd12_ncu_summary.txt" "$OUT/${TAG}_kdd12_ncu_summary.json"
rm -f "$OUT"/*.ncu-rep
ls -la "$OUT"
