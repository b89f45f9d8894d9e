"""Reservoir-sharing fraction sweep (the paper's Fig. 4: K=4, L=128, R=32 on url):
index every row of the url-shaped data with a pool of ceil(F*L*range) shared reservoirs,
answer 1,000 sampled rows (self excluded), and report index / query time, the index's
memory (kept ids + per-reservoir offsets and counters) and R@k / S@k against exact binary
cosine.  One B200.

    python tools/sweep_f.py [--shape url] [--out gpurun_out/sweep_f.json]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="url")
ap.add_argument("--F", default="1,0.5,0.2,0.1,0.05,0.02,0.01,0.005")
ap.add_argument("--queries", type=int, default=1000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep_f.json"))
args = ap.parse_args()

cfg = bench.SHAPE_CFG[args.shape]
shape = synth.SHAPES[args.shape]
torch.cuda.set_device(0)
h_rp, h_col, nnz = bench.gen_local(shape, [0, shape.N], 0)
d_rp, d_col = h_rp.cuda(), h_col.cuda()
N = shape.N
qs = np.sort(np.random.default_rng(13).choice(N, size=args.queries, replace=False))
crow, col, cnt, key = bench.dedup_csr(h_rp, d_col)
del key
cos, best = bench.exact_cosine(crow, col, cnt, qs)
del crow, col, cnt
q_rp, q_col = bench.sample_query_csr(h_rp.numpy(), h_col.numpy(), qs)
dq_rp, dq_col = flash.to_device_csr(q_rp, q_col)
excl = torch.from_numpy(qs.astype(np.uint32).view(np.int32)).cuda()
K, L, R, rng, k = cfg["K"], cfg["L"], cfg["R"], cfg["range_"], cfg["k"]
stream = torch.cuda.current_stream()
rows = []
for F in [float(x) for x in args.F.split(",")]:
    idx = flash.FlashIndex(K, L, R, rng, cfg["seed"], F=F)
    ti, tq = [], []
    for rep in range(args.reps + 1):
        idx.clear()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        idx.insert(d_rp, d_col, 0)
        e[1].record(stream)
        ids, cnts = idx.query(dq_rp, dq_col, k, excl)
        e[2].record(stream)
        torch.cuda.synchronize()
        if rep:
            ti.append(e[0].elapsed_time(e[1]))
            tq.append(e[1].elapsed_time(e[2]))
    goff, _, arr = idx.table_arrays(ids=False)
    kept = int(goff[-1].item())
    mem = 4 * kept + 8 * (idx.pool + 1) + 4 * idx.pool
    r_at, s_at = bench.recall_at_k(cos, best, ids, k)
    rec = {"F": F, "pool": idx.pool, "index_ms": statistics.median(ti), "query_ms": statistics.median(tq),
           "kept_ids": kept, "index_bytes": mem, "max_count": int(flash.as_u32(cnts).max()),
           "R@k": r_at, "S@k": s_at}
    idx.close()
    rows.append(rec)
    print(json.dumps(rec), flush=True)

meta = {"workload": f"{args.shape}-shaped: index all {N} rows, {args.queries} sampled queries (self excluded)",
        "K": K, "L": L, "R": R, "range": rng, "k": k, "gpu": torch.cuda.get_device_name(0),
        "timing": f"device events, median of {args.reps} after one warm-up",
        "index_bytes": "4 B per kept id + 8 B offset + 4 B counter per reservoir"}
with open(args.out, "w") as f:
    json.dump({"meta": meta, "points": rows}, f, indent=1)
