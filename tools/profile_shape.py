"""Index all rows of a shape and answer 10K sampled queries (bench.py --workload's step),
for ncu launch lists:  python tools/profile_shape.py --shape url|kdd12 [--reps 1]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="url")
ap.add_argument("--reps", type=int, default=1)
args = ap.parse_args()
cfg = bench.SHAPE_CFG[args.shape]
shape = synth.SHAPES[args.shape]
rp, col = synth.generate(shape)
rows = np.sort(np.random.default_rng(cfg["qseed"]).choice(shape.N, size=cfg["q"], replace=False))
q_rp, q_col = bench.sample_query_csr(rp, col, rows)
d_rp, d_col = flash.to_device_csr(rp, col)
dq_rp, dq_col = flash.to_device_csr(q_rp, q_col)
excl = torch.from_numpy(rows.astype(np.uint32).view(np.int32)).cuda()
idx = flash.FlashIndex(cfg["K"], cfg["L"], cfg["R"], cfg["range_"], cfg["seed"])
for _ in range(args.reps):
    idx.clear()
    idx.insert(d_rp, d_col, 0)
    idx.query(dq_rp, dq_col, cfg["k"], excl)
torch.cuda.synchronize()
print("done", shape.N, int(rp[-1]))
