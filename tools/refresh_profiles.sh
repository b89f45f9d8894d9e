#!/usr/bin/env bash
# Regenerate the round's profiles on a B200 (run under gpurun from the repo root):
#   gpurun --timeout 2400 -- 'bash tools/refresh_profiles.sh r01'
# Writes everything under gpurun_out/<tag>/ (merged back by gpurun); copy the files into
# profiles/ afterwards.  Order matters: the bench reads the ncu --set full summary for
# its roofline traffic, so that capture runs first and is installed into profiles/ here.
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
export PYTHONUNBUFFERED=1

# 1. ncu --set full of one webspam graph (every kernel once), then its per-kernel summary
timeout 1200 ncu --set full --clock-control none --import-source on -f -o "$OUT/${TAG}_full" \
  python tools/profile_graph.py --reps 1 > "$OUT/ncu_full.log" 2>&1
python tools/ncu_summary.py "$OUT/${TAG}_full.ncu-rep" "$OUT/${TAG}_ncu_full_summary.txt" \
  "$OUT/${TAG}_ncu_full_summary.json"
cp "$OUT/${TAG}_ncu_full_summary.json" "profiles/${TAG}_ncu_full_summary.json"
rm -f "$OUT/${TAG}_full.ncu-rep"   # large; the summaries are what is kept

# 2. launch list (cold-cache, serialised) of the same graph
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/${TAG}_launches.csv" python tools/profile_graph.py --reps 1 > /dev/null 2>&1
python tools/launch_summary.py "$OUT/${TAG}_launches.csv" \
  "ncu --metrics gpu__time_duration.sum --clock-control none, one webspam graph (tools/profile_graph.py --reps 1)" \
  > "$OUT/${TAG}_launches_summary.txt"

# 3. bench lines (no profiler attached)
timeout 600 python bench.py > "$OUT/${TAG}_bench.json" 2> "$OUT/bench.log"
timeout 600 python bench.py --workload url --steps 3 --warmup 3 > "$OUT/${TAG}_bench_url.json" 2>> "$OUT/bench.log"
timeout 900 python bench.py --workload kdd12 --steps 3 --warmup 3 > "$OUT/${TAG}_bench_kdd12.json" 2>> "$OUT/bench.log"
timeout 900 python bench.py --workload friendster --steps 3 --warmup 3 > "$OUT/${TAG}_bench_friendster.json" 2>> "$OUT/bench.log"
timeout 900 python bench.py --workload url-graph --steps 3 --warmup 3 > "$OUT/${TAG}_bench_url_graph.json" 2>> "$OUT/bench.log"
timeout 900 python bench.py --workload webspam-sat --steps 5 --warmup 3 > "$OUT/${TAG}_bench_webspam_sat.json" 2>> "$OUT/bench.log"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/${TAG}_bench_reference.json" 2>> "$OUT/bench.log"
# 4. the K x L x R sweep (80 graphs, ~1 min)
timeout 1200 python tools/sweep.py --out "$OUT/${TAG}_sweep.json" > /dev/null 2>> "$OUT/bench.log"
python tools/sweep_table.py "$OUT/${TAG}_sweep.json" > "$OUT/${TAG}_sweep.txt"
ls -la "$OUT"
