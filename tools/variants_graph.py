"""A/B timing of libflash.so build variants on the webspam graph, interleaved in one process
(tools only; the product library is paper_1709_01190_b200/libflash.so):

    python tools/variants_graph.py --build NAME=DEF1,DEF2 ...   (cross-compiles, no GPU)
    python tools/variants_graph.py NAME ... [--rounds 5]        (base = the product library)
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("names", nargs="*")
ap.add_argument("--build", nargs="*")
ap.add_argument("--rounds", type=int, default=5)
ap.add_argument("--shape", default="webspam")
args = ap.parse_args()
if args.build is not None:
    from paper_1709_01190_b200 import build as B
    for spec in args.build:
        name, _, defs = spec.partition("=")
        B.build_variant("v_" + name, [d for d in defs.split(",") if d])
    sys.exit(0)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

CFG = {"webspam": (4, 50, 128, 1 << 15, 0x5EED0002, 128)}
K, L, R, rng, seed, k = CFG[args.shape]
shape = synth.SHAPES[args.shape]
rp, col = synth.generate(shape)
d_rp, d_col = flash.to_device_csr(rp, col)
ids = torch.empty((shape.N, k), dtype=torch.int32, device="cuda")
cnt = torch.empty_like(ids)
libs = {}
for name in ["base"] + args.names:
    flash._lib = None
    libs[name] = flash.load_library(flash.LIB_PATH if name == "base" else
                                    os.path.join(ROOT, "paper_1709_01190_b200", f"libflash_v_{name}.so"))
ref = None
times = {n: [] for n in libs}
for rnd in range(args.rounds):
    for name, lib in libs.items():
        flash._lib = lib
        idx = flash.FlashIndex(K, L, R, rng, seed)
        for rep in range(6):
            idx.clear()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            flash.flash_knn_graph(idx.h, d_rp, d_col, shape.N, k, ids, cnt)
            e1.record()
            torch.cuda.synchronize()
            if rep >= 2:
                times[name].append(e0.elapsed_time(e1))
        if ref is None:
            ref = ids.clone()
        elif not torch.equal(ref, ids):
            print(f"{name}: OUTPUT DIFFERS", flush=True)
        idx.close()
for name, ts in times.items():
    print(f"{name:12s} graph {statistics.median(ts):.3f} ms (min {min(ts):.3f}, n={len(ts)})", flush=True)
