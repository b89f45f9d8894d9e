"""Diagnostic: time the DOPH hash (H1-H3) of a shape under build variants of libflash.so
(tools only; the product library is paper_1709_01190_b200/libflash.so).

    python tools/doph_variants.py [--shape url] [--build]   (variants: see VARIANTS)
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
from paper_1709_01190_b200 import build as B  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

# (variants measured this round, their code since removed: probe-chain tables for K*L in
# (256, 768] — FLASH_DOPH_TPROBES / FLASH_DOPH_NOTABLE — and a cp.async.bulk column ring —
# FLASH_DOPH_BULK[_STAGES])
VARIANTS = {"base": []}
CFG = {"url": (4, 128, 1 << 15, 0x5EED0003), "webspam": (4, 50, 1 << 15, 0x5EED0002),
       "kdd12": (4, 32, 1 << 20, 0x5EED0004)}

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="url")
ap.add_argument("--build", action="store_true")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--extra", nargs="*", default=[], help="libflash_v_NAME.so builds of tools/variants_graph.py")
args = ap.parse_args()
if args.build:
    for name, defs in VARIANTS.items():
        B.build_variant("d_" + name, defs)
    sys.exit(0)
shape = synth.SHAPES[args.shape]
K, L, rng, seed = CFG[args.shape]
h_rp, h_col, nnz = bench.gen_local(shape, [0, shape.N], 0)
d_rp, d_col = h_rp.cuda(), h_col.cuda()
out = torch.empty((shape.N, L), dtype=torch.int32, device="cuda")
ref = None
for name in list(VARIANTS) + args.extra:
    flash._lib = None
    flash.load_library(flash.LIB_PATH if name == "base" else
                       os.path.join(ROOT, "paper_1709_01190_b200",
                                    f"libflash_v_{name}.so" if name in args.extra else f"libflash_d_{name}.so"))
    h = flash.flash_create(K, L, 32, rng, seed)
    ts = []
    for r in range(args.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        flash.flash_hash(h, d_rp, d_col, shape.N, None, out)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    flash.flash_destroy(h)
    same = True
    if ref is None:
        ref = out.clone()
    else:
        same = bool(torch.equal(ref, out))
    print(f"{args.shape} {name} C={os.environ.get("FLASH_DOPH_MIDC", "-")} le={os.environ.get("FLASH_DOPH_MID_LE", "-")}: hash {statistics.median(ts):.3f} ms (min {min(ts):.3f}) same={same}", flush=True)
