"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel
times and shares of the step (cold-cache, serialised launches: compare SHARES)."""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hd = rows[h]
ki, vi, ui = hd.index("Kernel Name"), hd.index("Metric Value"), hd.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = OrderedDict()
for r in rows[h + 1:]:
    if len(r) <= vi:
        continue
    nm = r[ki].split("(")[0][:62]
    tot.setdefault(nm, [0.0, 0])
    tot[nm][0] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot[nm][1] += 1
s = sum(v[0] for v in tot.values())
out = [f"# {sys.argv[2] if len(sys.argv) > 2 else ''}".rstrip(),
       "# cold-cache, serialised launches: compare SHARES"]
for nm, (us, n) in tot.items():
    out.append(f"{nm:64s} {us:9.1f} us  x{n:<3d} {100 * us / s:5.1f}%")
out.append(f"{'total':64s} {s:9.1f} us")
print("\n".join(out))
