"""Per-source-line shared-memory wavefronts of an ncu source page (cuda,sass CSV):
    python tools/ncu_smem_lines.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
wi, ii = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
tot = []
for r in rows[hdr + 1:]:
    if len(r) <= wi or not r[0].isdigit() or r[2] != "-":
        continue
    try:
        w, i = int(r[wi] or 0), int(r[ii] or 0)
    except ValueError:
        continue
    if w:
        tot.append((w, i, int(r[0]), r[1][:100]))
allw = sum(t[0] for t in tot) or 1
print(f"total shared wavefronts {allw:,}")
for w, i, ln, src in sorted(tot, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{ln:5d} {100 * w / allw:5.1f}% wf={w:>12,d} ideal={i:>12,d}  {src}")
