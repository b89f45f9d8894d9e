"""Per-source-line warp-stall samples and executed instructions from an ncu report
(ncu -i REP --page source --csv --print-source cuda,sass):  python tools/ncu_lines.py REP [N]"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
agg, src = {}, {}
for r in rows:
    if len(r) <= ii or not r[0].strip().isdigit():
        continue
    ln = int(r[0])
    src[ln] = r[1][:100]
    try:
        s, n = int(r[si] or 0), int(r[ii] or 0)
    except ValueError:
        continue
    a = agg.setdefault(ln, [0, 0])
    a[0] += s
    a[1] += n
tot = sum(v[0] for v in agg.values()) or 1
for ln, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{ln:5} {100 * s / tot:5.1f}% inst={n:>13} {src.get(ln, '')}")
