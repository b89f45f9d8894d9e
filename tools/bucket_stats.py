"""Diagnostic: bucket and 128-bucket-group arrival statistics of a shape's index (device).

    python tools/bucket_stats.py [--shape kdd12]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="kdd12")
args = ap.parse_args()
cfg = bench.SHAPE_CFG[args.shape]
shape = synth.SHAPES[cfg.get("shape", args.shape)]
h_rp, h_col, nnz = bench.gen_local(shape, [0, shape.N], 0)
d_rp, d_col = h_rp.cuda(), h_col.cuda()
K, L, R, rng = cfg["K"], cfg["L"], cfg["R"], cfg["range_"]
idx = flash.FlashIndex(K, L, R, rng, cfg["seed"])
A = idx.hash_addrs(d_rp, d_col)
for t in range(0, L, max(1, L // 4)):
    a = A[:, t].long() & 0xFFFFFFFF
    a = a[a != 0xFFFFFFFF]
    c = torch.bincount(a, minlength=rng).double()
    g = torch.bincount(a >> 7, minlength=(rng + 127) >> 7).double()
    q = torch.tensor([0.5, 0.99, 0.9999], dtype=torch.float64, device=c.device)
    print(f"table {t}: bucket mean {c.mean():.1f} max {int(c.max())} q50/99/99.99 {torch.quantile(c[:1 << 24], q).tolist()} "
          f"over R {float((c > R).double().mean()):.3f} | group mean {g.mean():.0f} max {int(g.max())} "
          f"q99/99.99 {torch.quantile(g, q[1:]).tolist()}", flush=True)
