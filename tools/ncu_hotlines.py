"""Summarise an ncu source page (cuda,sass CSV) into per-source-line stall samples."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for i, r in enumerate(rows):
    if r and r[0] == "Line No":
        hdr = i
        break
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
tot = defaultdict(lambda: [0, 0, ""])
for r in rows[hdr + 1:]:
    if len(r) <= si or not r[0].isdigit():
        continue
    if r[2] != "-":  # a sass row nested under its source line
        continue
    try:
        s = int(r[si]); n = int(r[ii])
    except ValueError:
        continue
    tot[int(r[0])] = [s, n, r[1][:110]]
all_s = sum(v[0] for v in tot.values()) or 1
for ln, (s, n, src) in sorted(tot.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{ln:5d} {100*s/all_s:5.1f}% inst={n:>11d}  {src}")
