"""Diagnostic: the friendster-shaped index (insert only, or --graph: the whole k-NN graph)
once, for ncu launch lists of the build kernels."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--graph", action="store_true")
args = ap.parse_args()
shape = synth.SHAPES["friendster"]
cfg = bench.SHAPE_CFG["friendster"]
h_rp, h_col, nnz = bench.gen_local(shape, [0, shape.N], 0)
d_rp, d_col = h_rp.cuda(), h_col.cuda()
idx = flash.FlashIndex(cfg["K"], cfg["L"], cfg["R"], cfg["range_"], cfg["seed"])
if args.graph:
    idx.knn_graph(d_rp, d_col, cfg["k"])
else:
    flash.flash_insert(idx.h, d_rp, d_col, shape.N, 0)
torch.cuda.synchronize()
print("done")
