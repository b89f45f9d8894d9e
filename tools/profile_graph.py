"""Run the webspam-shaped k-NN graph a few times (for ncu / compute-sanitizer).

    python tools/profile_graph.py [--shape webspam] [--n N] [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

CFG = {"webspam": (4, 50, 128, 1 << 15, 0x5EED0002, 128),
       "url": (4, 128, 32, 1 << 15, 0x5EED0003, 128),
       "kdd12": (4, 32, 64, 1 << 20, 0x5EED0004, 128),
       "friendster": (4, 32, 64, 1 << 20, 0x5EED0005, 20),
       "tiny": (4, 16, 32, 1 << 15, 0x5EED0001, 10)}

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="webspam")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()
shape = synth.SHAPES[args.shape]
if args.n:
    shape = shape.with_(N=args.n)
K, L, R, rng, seed, k = CFG[args.shape]
rp, col = synth.generate(shape)
d_rp, d_col = flash.to_device_csr(rp, col)
idx = flash.FlashIndex(K, L, R, rng, seed)
ids = torch.empty((shape.N, k), dtype=torch.int32, device="cuda")
cnt = torch.empty_like(ids)
for _ in range(args.reps):
    idx.clear()
    flash.flash_knn_graph(idx.h, d_rp, d_col, shape.N, k, ids, cnt)
torch.cuda.synchronize()
print("done", shape.N, int(rp[-1]))
