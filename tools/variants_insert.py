"""A/B timing of libflash.so build variants on a shape's index build (flash_insert of every
row: hash + build), interleaved in one process (tools only):

    python tools/variants_graph.py --build NAME=DEF1,DEF2     (cross-compiles the variant)
    python tools/variants_insert.py NAME ... [--shape kdd12] [--rounds 3]
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("names", nargs="*")
ap.add_argument("--shape", default="kdd12")
ap.add_argument("--rounds", type=int, default=3)
args = ap.parse_args()
cfg = bench.SHAPE_CFG[args.shape]
shape = synth.SHAPES[args.shape]
h_rp, h_col, nnz = bench.gen_local(shape, [0, shape.N], 0)
d_rp, d_col = h_rp.cuda(), h_col.cuda()
libs = {}
for name in ["base"] + args.names:
    flash._lib = None
    libs[name] = flash.load_library(flash.LIB_PATH if name == "base" else
                                    os.path.join(ROOT, "paper_1709_01190_b200", f"libflash_v_{name}.so"))
times = {n: [] for n in libs}
ref = None
for rnd in range(args.rounds):
    for name, lib in libs.items():
        flash._lib = lib
        idx = flash.FlashIndex(cfg["K"], cfg["L"], cfg["R"], cfg["range_"], cfg["seed"])
        for rep in range(3):
            idx.clear()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            idx.insert(d_rp, d_col, 0)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                times[name].append(e0.elapsed_time(e1))
        off, ids, _ = idx.table(0)
        sig = (int(off[-1]), int(ids[: 1000].astype("int64").sum()))
        if ref is None:
            ref = sig
        elif sig != ref:
            print(f"{name}: TABLE 0 DIFFERS", flush=True)
        idx.close()
for name, ts in times.items():
    print(f"{args.shape} {name:10s} insert {statistics.median(ts):.2f} ms (min {min(ts):.2f}, n={len(ts)})", flush=True)
