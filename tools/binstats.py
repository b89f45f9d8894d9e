"""Diagnostic: structure of the per-query candidate multisets the query sort sees
(webspam bench config): bin occupancy, distinct ids, inversions in gather order."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

shape = synth.SHAPES["webspam"]
K, L, R, rng, seed = 4, 50, 128, 1 << 15, 0x5EED0002
rp, col = synth.generate(shape)
d_rp, d_col = flash.to_device_csr(rp, col)
idx = flash.FlashIndex(K, L, R, rng, seed)
addrs = idx.hash_addrs(d_rp, d_col)
idx.insert_addrs(addrs, 0)
goff, ids, _ = idx.table_arrays()
goff = goff.cpu().numpy()
ids = ids.cpu().numpy().view(np.uint32)
addrs = addrs.cpu().numpy().view(np.uint32)
N = shape.N
bits = int(N - 1).bit_length()
rs = np.random.default_rng(0)
BL = int(sys.argv[1]) if len(sys.argv) > 1 else 10
shift = max(bits - BL, 0)
stats = []
for q in rs.choice(N, 400, replace=False):
    parts = []
    for t in range(L):
        a = addrs[q, t]
        if a >= rng:
            continue
        i = t * rng + a
        parts.append(ids[goff[i]:goff[i + 1]])
    c = np.concatenate(parts)
    c = c[c != q]
    M = c.size
    d = c >> shift
    order = np.argsort(d, kind="stable")
    arr = c[order]
    binsz = np.bincount(d, minlength=1 << BL)
    ends = np.cumsum(binsz)
    starts = ends - binsz
    inv_bin = np.zeros(1 << BL, np.int64)
    for b in np.nonzero(binsz > 1)[0]:
        x = arr[starts[b]:ends[b]]
        inv_bin[b] = int(np.sum(x[:, None] > x[None, :], where=np.triu(np.ones((x.size, x.size), bool), 1)))
    lane_inv = inv_bin.reshape(32, -1).sum(1)
    lane_sz = binsz.reshape(32, -1).sum(1)
    u, cnt = np.unique(c, return_counts=True)
    stats.append((M, u.size, cnt.max(), binsz.max(), int((inv_bin > 0).sum()), inv_bin.sum(), inv_bin.max(),
                  lane_inv.max(), lane_sz.max(), int((cnt >= 10).sum())))
s = np.array(stats, dtype=np.float64)
names = ["M", "distinct", "maxmult", "maxbin", "unsorted_bins", "inversions", "max_bin_inv", "max_lane_inv",
         "max_lane_size", "ids_mult>=10"]
for i, n in enumerate(names):
    print(f"BL={BL} {n:15s} mean {s[:, i].mean():10.1f}  p50 {np.median(s[:, i]):8.0f}  p99 {np.percentile(s[:, i], 99):8.0f}  max {s[:, i].max():8.0f}")
