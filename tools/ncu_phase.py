"""Per-source-line-range instruction and stall totals from an ncu source page (cuda,sass CSV).
    python tools/ncu_phase.py source.csv NQ name:first-last [name:first-last ...]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
ii, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
byl = {}
for r in rows[hdr + 1:]:
    if len(r) > ii and r[0].isdigit() and r[2] == "-":
        try:
            byl[int(r[0])] = (int(r[ii]), int(r[si]))
        except ValueError:
            pass
nq = float(sys.argv[2])
ts = sum(v[1] for v in byl.values()) or 1
print(f"total {sum(v[0] for v in byl.values()) / nq:.0f} warp-inst per unit")
for spec in sys.argv[3:]:
    name, rng = spec.split(":")
    a, b = map(int, rng.split("-"))
    ins = sum(v[0] for l, v in byl.items() if a <= l <= b)
    st = sum(v[1] for l, v in byl.items() if a <= l <= b)
    print(f"{name:10s} {ins / nq:8.0f} inst/unit  {100 * st / ts:5.1f}% stall samples")
