"""Diagnostic: the webspam graph through a plain handle, the multi-GPU handle with one
virtual rank (flash_create_dist_local, world 1) and, under torchrun / --nccl, the NCCL handle
at world 1 — step time (device events) and per-phase times, to expose the multi-GPU path's
fixed costs (exchanges, barriers, host synchronisation)."""
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
ap.add_argument("--nccl", action="store_true")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--only", default="", help="run only this handle kind (plain / local1 / nccl1)")
args = ap.parse_args()
torch.cuda.set_device(0)
shape = synth.SHAPES["webspam"]
h_rp, h_col, nnz = bench.gen_local(shape, [0, shape.N], 0)
d_rp, d_col = h_rp.cuda(), h_col.cuda()
N, k = shape.N, 128
out_ids = torch.empty((N, k), dtype=torch.int32, device="cuda")
out_cnt = torch.empty_like(out_ids)
handles = {"plain": flash.FlashIndex(bench.K, bench.L, bench.R, bench.RANGE, bench.SEED),
           "local1": flash.FlashIndex(bench.K, bench.L, bench.R, bench.RANGE, bench.SEED,
                                      handle=flash.flash_create_dist_local(bench.K, bench.L, bench.R, bench.RANGE,
                                                                           bench.SEED, 1)[0])}
if args.nccl:
    import torch.distributed as dist

    from paper_1709_01190_b200 import dist as fdist

    for key, val in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533"), ("RANK", "0"), ("WORLD_SIZE", "1")):
        os.environ.setdefault(key, val)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    handles["nccl1"] = fdist.create_dist_index(bench.K, bench.L, bench.R, bench.RANGE, bench.SEED)
ref = None
for name, idx in handles.items():
    if args.only and name != args.only:
        continue
    flash.flash_set_profiling(idx.h, True)
    ts = []
    for i in range(args.steps + 2):
        if i == 2:
            flash.flash_reset_counters(idx.h)
        idx.clear()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        flash.flash_knn_graph(idx.h, d_rp, d_col, N, k, out_ids, out_cnt)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    ms, calls = flash.flash_phase_ms(idx.h)
    same = True
    if ref is None:
        ref = out_ids.clone()
    else:
        same = bool(torch.equal(ref, out_ids))
    print(f"{name:7s} step {statistics.median(ts):.3f} ms  phases " +
          " ".join(f"{p}={m / args.steps:.3f}" for p, m in zip(("hash", "build", "query", "copy"), ms)) +
          f"  launches {flash.flash_launch_count(idx.h)}  same={same}", flush=True)
