#!/usr/bin/env python
"""bench.py — webspam-shaped approximate k-NN graph (FLASH hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = one full k-NN graph from scratch over the resident webspam-shaped CSR:
DOPH hashing of every row (H1-H3), bottom-R table build (B1-B2) and count-based
top-k for every row (Q1-Q3) — all SURVEY §8(a) rows.  Workload = BASELINE.json
configs[1]: N=350,000 rows, D=16,609,143, ~3,728 nnz/row (~1.3 G nnz), K=4, L=50,
R=128, range=2^15, k=128 (synthetic, synth/ seed 2).

`value` = N / graph time (queries/s over the whole graph; every row is a query),
device-timed with CUDA events, max over ranks.  `e2e` = the same metric through
flash_knn_graph_host (pinned host CSR in, host top-k out, copies inside the timed
region).  N>1: one rank per GPU (torchrun), the library's multi-GPU handle
(flash_create_dist: tables partitioned over the GPUs, addresses and candidate lists
stored into the peers' buffers, NCCL barriers; --mode sharded: the torch.distributed
sharded-build schedule of dist.py instead), strong scaling of the fixed graph.

The reference arm (--impl reference) and `cpu_baseline` time the CPU oracle (oracle/)
as it stands on the host cores (OpenMP, all cores) on the same workload: hash + build
of every row and top-k for --ref-sample rows (default: all rows, i.e. the whole graph;
a smaller sample is extrapolated per query).  It is a deliberately slow baseline.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

K, L, R, RANGE, SEED, TOPK = 4, 50, 128, 1 << 15, 0x5EED0002, 128
METRIC = "webspam-shaped k-NN graph time (s), queries/s, hash nnz/s at 1/2/4/8 B200"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# the newest committed ncu --set full summary of one webspam graph (tools/refresh_profiles.sh)
TRAFFIC_PATH = next((p for p in (os.path.join(ROOT, "profiles", f"r0{i}_ncu_full_summary.json") for i in (2, 1))
                     if os.path.exists(p)), os.path.join(ROOT, "profiles", "r01_ncu_full_summary.json"))
# Shared-memory RMW throughput measured on this pool's B200 (profiles/r01_microbench_smem.txt:
# RED.S.ADD on random addresses, 8.76 lane-ops/clk/SM at 1.9 GHz x 148 SMs): the ceiling
# for the count step, which needs at least one shared-memory RMW per candidate.
SMEM_RMW_PEAK = 8.76 * 148 * 1.9e9


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def clk_mhz_for_peak():
    """SM clock for issue-rate peaks: nvidia-smi's max SM clock, else the B200 boost clock."""
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=10).stdout.split()
        return float(out[0])
    except Exception:
        return 1965.0


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_config(shape, nnz, args):
    return {
        "workload": "webspam-shaped approximate k-NN graph from scratch (hash + build + query every row)",
        "N": shape.N, "D": shape.D, "nnz": int(nnz), "nnz_per_row": round(nnz / shape.N, 1),
        "K": K, "L": L, "R": R, "range": RANGE, "k": TOPK, "seed": SEED,
        "parallelism": ((f"rows x{args.gpus} (hash, count/top-k); tables x{args.gpus} (build, gather); "
                         "addresses + candidates as peer stores (flash_create_dist)") if args.mode == "exchange" else
                        (f"rows x{args.gpus} (hash, query); tables x{args.gpus} (build); "
                         "all-gather addresses + built tables")) if args.gpus > 1 else "1 GPU",
        "l2_policy": "inputs larger than L2 (col_idx 5.2 GB vs 126 MB L2); no flush",
    }


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                smax = max(smax, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def gen_local(shape, bounds, rank):
    """This rank's rows (all rows at N=1), in pinned host memory."""
    import torch

    r0, r1 = bounds[rank], bounds[rank + 1]
    lens = np.empty(r1 - r0, dtype=np.int64)
    p = synth._cparams(shape)
    import ctypes

    synth._load().synth_row_lengths(ctypes.byref(p), r0, r1, lens.ctypes.data)
    nnz = int(lens.sum())
    rp_t = torch.empty(r1 - r0 + 1, dtype=torch.int64).pin_memory()
    col_t = torch.empty(max(nnz, 1), dtype=torch.int32).pin_memory()
    synth.generate(shape, rows=(r0, r1), row_ptr_out=rp_t.numpy(), col_out=col_t.numpy().view(np.uint32))
    return rp_t, col_t, nnz


def query_work(idx_tables, addrs_np, tables=None):
    """Candidates gathered per query (the sum of its bucket sizes over `tables`, default all
    L) and the bucket-arrival histogram (log2 bins) of those tables."""
    per_q = np.zeros(addrs_np.shape[0], dtype=np.int64)
    hist = np.zeros(34, dtype=np.int64)
    over_r = 0
    for t in (range(L) if tables is None else tables):
        off, _, arr = idx_tables(t)
        sizes = np.diff(off.astype(np.int64))
        a = addrs_np[:, t]
        valid = a != 0xFFFFFFFF
        per_q[valid] += sizes[a[valid].astype(np.int64)]
        arr = arr.astype(np.int64)
        lg = np.zeros_like(arr)
        nz = arr > 0
        lg[nz] = np.floor(np.log2(arr[nz])).astype(np.int64) + 1
        hist += np.bincount(lg, minlength=34)[:34]
        over_r += int((arr > R).sum())
    top = int(np.nonzero(hist)[0].max()) if hist.any() else 0
    labels = ["0"] + [f"{1 << (i - 1)}-{(1 << i) - 1}" for i in range(1, top + 1)]
    arrivals = {"buckets": int(hist.sum()), "histogram_log2": dict(zip(labels, hist[: top + 1].tolist())),
                "frac_over_R": over_r / max(int(hist.sum()), 1)}
    return per_q, arrivals


def dedup_csr(h_rp, d_col):
    """Rows as sets (duplicate column ids dropped), on the device: (crow int64 [N+1],
    col int32, cnt int64 [N], sorted (row << 32 | col) keys).  Evaluation only."""
    import torch

    dev = d_col.device
    rp = h_rp.numpy().astype(np.int64)
    rp = rp - rp[0]
    N = rp.size - 1
    lens = np.diff(rp)
    row = torch.repeat_interleave(torch.arange(N, device=dev), torch.from_numpy(lens).to(dev))
    key = (row << 32) | (d_col.to(torch.int64) & 0xFFFFFFFF)
    del row
    key = torch.sort(key).values
    keep = torch.ones(key.numel(), dtype=torch.bool, device=dev)
    keep[1:] = key[1:] != key[:-1]
    key = key[keep]
    del keep
    cnt = torch.bincount(key >> 32, minlength=N)
    crow = torch.zeros(N + 1, dtype=torch.int64, device=dev)
    crow[1:] = torch.cumsum(cnt, 0)
    col = (key & 0xFFFFFFFF).to(torch.int32)
    return crow, col, cnt, key


def exact_cosine(crow, col, cnt, qs, B=64):
    """Exact binary cosine (Eq. 3) of every row against the rows qs, self excluded
    (-1): float64 [N, len(qs)] on the device, plus the exact 1-NN cosine per query.  A
    deduplicated CSR x dense 0/1 query-mask product (torch sparse).  Evaluation only."""
    import torch

    dev = col.device
    N = cnt.numel()
    D = int(col.max().item()) + 1
    X = torch.sparse_csr_tensor(crow.to(torch.int32), col, torch.ones(col.numel(), device=dev),
                                size=(N, D), check_invariants=False)
    Qm = torch.empty((D, B), dtype=torch.float32, device=dev)
    out = torch.empty((N, len(qs)), dtype=torch.float64, device=dev)
    cntd = cnt.double()
    for b0 in range(0, len(qs), B):
        qb = torch.from_numpy(np.asarray(qs[b0:b0 + B])).to(dev)
        nb = qb.numel()
        Qm.zero_()
        lq = cnt[qb]
        pidx = torch.repeat_interleave(torch.arange(nb, device=dev), lq)
        first = torch.cumsum(lq, 0) - lq
        offs = torch.arange(pidx.numel(), device=dev) - first[pidx]
        Qm[col[crow[qb][pidx] + offs].long(), pidx] = 1.0
        inter = torch.sparse.mm(X, Qm)[:, :nb].double()                 # [N, nb]
        den = torch.sqrt(cntd[:, None] * cntd[qb][None, :])
        cos = torch.where(den > 0, inter / den.clamp(min=1), torch.zeros_like(inter))
        cos[qb, torch.arange(nb, device=dev)] = -1.0                      # exclude self
        out[:, b0:b0 + nb] = cos
    return out, out.max(0).values


def heavy_recall(h_rp, d_col, top_ids, qs, thr, batch=32):
    """Recall of the neighbours whose exact binary cosine exceeds thr in the reported top-k
    (the friendster metric of P:507: "recall of neighbors with similarity > 0.65 ... in the
    top 20"), for the query rows qs.  Exact cosines through a column index of the
    deduplicated rows (every row sharing a column with the query), on the device.
    Evaluation only."""
    import torch

    crow, col, cnt, key = dedup_csr(h_rp, d_col)
    dev = col.device
    ckey = torch.sort(((key & 0xFFFFFFFF) << 32) | (key >> 32)).values  # (col, row), sorted
    del key
    ccol = ckey >> 32
    D = int(ccol[-1].item()) + 1 if ccol.numel() else 1
    cptr = torch.zeros(D + 1, dtype=torch.int64, device=dev)
    cptr[1:] = torch.cumsum(torch.bincount(ccol, minlength=D), 0)
    crows = ckey & 0xFFFFFFFF
    del ccol, ckey
    top = top_ids.to(dev).long()
    hit = tot = 0

    def expand(starts, lens):  # starts[i] + [0, lens[i]) for every i, and the owner index
        own = torch.repeat_interleave(torch.arange(lens.numel(), device=dev), lens)
        first = torch.cumsum(lens, 0) - lens
        return starts[own] + torch.arange(own.numel(), device=dev) - first[own], own

    for b0 in range(0, len(qs), batch):
        qb = torch.as_tensor(np.asarray(qs[b0:b0 + batch]), device=dev, dtype=torch.int64)
        pos, qi = expand(crow[qb], cnt[qb])
        qc = col[pos].long()                                  # the queries' columns
        ppos, pi = expand(cptr[qc], cptr[qc + 1] - cptr[qc])  # their posting lists
        u, inter = torch.unique((qi[pi] << 32) | crows[ppos], return_counts=True)
        uq, ur = u >> 32, u & 0xFFFFFFFF
        cosv = inter.double() / torch.sqrt(cnt[qb][uq].double() * cnt[ur].double())
        heavy = (cosv > thr) & (ur != qb[uq])
        hq, hr = uq[heavy], ur[heavy]
        tot += int(heavy.sum().item())
        hit += int((top[qb[hq]] == hr[:, None]).any(1).sum().item())
    return {"queries": int(len(qs)), "threshold": thr, "heavy_neighbours": tot, "recall": hit / max(tot, 1)}


def graph_candidates(idx, d_rp, d_col, n, L, range_, chunk=1 << 22):
    """Candidates per query of a k-NN graph (the sum of its L bucket sizes), from the
    rows' addresses and the built index's offsets (evaluation only): int64 [n] on the device."""
    import torch

    goff = idx.table_arrays(ids=False)[0]
    tb = torch.arange(L, device=goff.device, dtype=torch.int64)[None, :] * range_
    out = torch.empty(n, dtype=torch.int64, device=goff.device)
    for r0 in range(0, n, chunk):
        r1 = min(n, r0 + chunk)
        rp = d_rp[r0:r1 + 1]
        a = idx.hash_addrs(rp, d_col).long() & 0xFFFFFFFF
        valid = a != 0xFFFFFFFF
        b = torch.where(valid, a + tb, torch.zeros_like(a))
        out[r0:r1] = torch.where(valid, goff[b + 1] - goff[b], torch.zeros_like(a)).sum(1)
    return out


def recall_at_k(cos, best, top_ids, kmax):
    """R@k (exact cosine 1-NN, any tie, in the reported top-k) and S@k (mean exact
    cosine of the reported ids) for k in {1, 10, 100, kmax}.  cos [N, nq], top_ids
    [nq, kmax] (EMPTY = -1 as int32)."""
    import torch

    ks = sorted({k for k in (1, 10, 100) if k <= kmax} | {kmax})
    top = top_ids.long()
    valid = top >= 0
    ct = cos.t().gather(1, top.clamp(min=0)).double()
    n = top.shape[0]
    rec, sim = {}, {}
    for k in ks:
        v = valid[:, :k]
        hit = ((ct[:, :k] >= best.double()[:, None] - 1e-9) & v).any(1)
        rec[str(k)] = float(hit.double().sum().item()) / n
        s = torch.where(v, ct[:, :k], torch.zeros_like(ct[:, :k])).sum(1) / v.sum(1).clamp(min=1)
        sim[str(k)] = float(s.sum().item()) / n
    return rec, sim


def data_quality_stats(h_rp, d_col, out_ids, n_q=1000, n_pairs=100_000, seed=13):
    """SURVEY §8(d) statistics printed beside the timing (evaluation only, outside the timed
    region, never on the product path): nnz mean / p99, mean binary cosine over random row
    pairs, and the graph's R@k / S@k against exact binary cosine for
    n_q sampled rows.  Rows are treated as sets (duplicate column ids dropped)."""
    import torch

    dev = d_col.device
    lens = np.diff(h_rp.numpy().astype(np.int64))
    N = lens.size
    res = {"nnz_mean": float(lens.mean()), "nnz_p99": float(np.percentile(lens, 99))}
    crow, col, cnt, key = dedup_csr(h_rp, d_col)
    rng = np.random.default_rng(seed)

    # mean pairwise cosine: |a ∩ b| by looking up (b, c) for every c of row a in the sorted keys
    pa, pb = rng.integers(0, N, n_pairs), rng.integers(0, N, n_pairs)
    ok = pa != pb
    pa, pb = pa[ok], pb[ok]
    cos_sum, n_ok = 0.0, 0
    for c0 in range(0, pa.size, 10_000):
        a = torch.from_numpy(pa[c0:c0 + 10_000]).to(dev)
        b = torch.from_numpy(pb[c0:c0 + 10_000]).to(dev)
        la = cnt[a]
        pidx = torch.repeat_interleave(torch.arange(a.numel(), device=dev), la)
        first = torch.cumsum(la, 0) - la
        offs = torch.arange(pidx.numel(), device=dev) - first[pidx]
        q = (b[pidx] << 32) | (key[crow[a][pidx] + offs] & 0xFFFFFFFF)
        pos = torch.searchsorted(key, q).clamp(max=key.numel() - 1)
        inter = torch.bincount(pidx, weights=(key[pos] == q).double(), minlength=a.numel())
        den = torch.sqrt(la.double() * cnt[b].double())
        c = torch.where(den > 0, inter / den.clamp(min=1), torch.zeros_like(inter))
        cos_sum += float(c.sum().item())
        n_ok += a.numel()
    res["pairwise_cosine_mean"] = cos_sum / max(n_ok, 1)
    res["pairwise_pairs"] = n_ok
    del key

    qs = rng.choice(N, size=min(n_q, N), replace=False)
    cos, best = exact_cosine(crow, col, cnt, qs)
    rec, sim = recall_at_k(cos, best, out_ids[torch.from_numpy(qs).to(dev)], out_ids.shape[1])
    res["one_nn_cosine_mean"] = float(best.double().mean().item())
    res["quality"] = {"queries": int(qs.size), "R@k": rec, "S@k": sim,
                      "definition": "R@k: exact cosine 1-NN (any tie) in the reported top-k (P:393); "
                                    "S@k: mean exact cosine of the reported top-k (P:395)"}
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1709_01190_b200 import dist as fdist
    from paper_1709_01190_b200 import flash

    rank, world, local = dist_env()
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    # FLASH_BENCH_ONE_GPU=1 (debug only): every rank on cuda:0 over gloo, to exercise the
    # multi-rank path on a 1-GPU box; its timings mean nothing.
    one_gpu = os.environ.get("FLASH_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1 or args.dist_handle:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            for key, val in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533"), ("RANK", "0"),
                             ("WORLD_SIZE", "1")):
                os.environ.setdefault(key, val)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    shape = synth.SHAPES["webspam"]
    t0 = time.time()
    all_lens = np.empty(shape.N, dtype=np.int64)
    import ctypes

    synth._load().synth_row_lengths(ctypes.byref(synth._cparams(shape)), 0, shape.N, all_lens.ctypes.data)
    bounds = fdist.shard_bounds(all_lens, world)
    h_rp, h_col, nnz_local = gen_local(shape, bounds, rank)
    nnz_total = int(all_lens.sum())
    log(f"[rank {rank}] generated rows {bounds[rank]}..{bounds[rank + 1]} nnz={nnz_local} in {time.time() - t0:.1f}s")
    n_local = bounds[rank + 1] - bounds[rank]
    dev = torch.device("cuda", local)
    # device-resident CSR (row_ptr rebased to this shard's col_idx)
    d_rp = (h_rp.to(dev, non_blocking=True) - h_rp[0].item()).contiguous()
    d_col = h_col.to(dev, non_blocking=True)
    out_ids = torch.empty((n_local, TOPK), dtype=torch.int32, device=dev)
    out_cnt = torch.empty((n_local, TOPK), dtype=torch.int32, device=dev)
    # N > 1: the library's multi-GPU handle (tables partitioned over the GPUs, candidates to
    # the query owners; north_star (d)), or the torch.distributed sharded-build schedule
    use_dist_handle = (world > 1 or args.dist_handle) and args.mode == "exchange"
    idx = (fdist.create_dist_index(K, L, R, RANGE, SEED) if use_dist_handle
           else flash.FlashIndex(K, L, R, RANGE, SEED))
    stream = torch.cuda.current_stream()

    def step():
        idx.clear()
        if world == 1 or use_dist_handle:
            flash.flash_knn_graph(idx.h, d_rp, d_col, n_local, TOPK, out_ids, out_cnt)
            return out_ids, out_cnt
        return fdist.knn_graph_sharded_build(idx, d_rp, d_col, TOPK, bounds, rank)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    flash.flash_reset_counters(idx.h)
    flash.flash_set_profiling(idx.h, True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    phase_ms, phase_calls = flash.flash_phase_ms(idx.h)
    launches = flash.flash_launch_count(idx.h)
    flash.flash_set_profiling(idx.h, False)
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    ms_max = float(t_local.item())
    ms_step = ms_max / args.steps

    # end-to-end through the host-buffer C-ABI entry point (N=1) / host copies around the
    # distributed graph (N>1)
    e2e_ms = []
    h_ids = torch.empty((n_local, TOPK), dtype=torch.int32).pin_memory()
    h_cnt = torch.empty((n_local, TOPK), dtype=torch.int32).pin_memory()
    h_rp_local = (h_rp - h_rp[0]).pin_memory()
    e2e_steps = max(1, min(args.steps, 5))
    for i in range(e2e_steps + 1):
        idx.clear()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        if world == 1 or use_dist_handle:
            flash.flash_knn_graph_host(idx.h, h_rp_local, h_col, n_local, TOPK, h_ids, h_cnt)
        else:
            d_rp2 = h_rp_local.to(dev, non_blocking=True)
            d_col2 = h_col.to(dev, non_blocking=True)
            ids_, cnt_ = fdist.knn_graph_sharded_build(idx, d_rp2, d_col2, TOPK, bounds, rank)
            h_ids.copy_(ids_, non_blocking=True)
            h_cnt.copy_(cnt_, non_blocking=True)
            torch.cuda.synchronize()
        dt = (time.perf_counter() - t) * 1e3
        if i > 0:  # first is warm-up
            e2e_ms.append(dt)
    e2e_local = torch.tensor([statistics.median(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_local, op=dist.ReduceOp.MAX)
    e2e_ms_max = float(e2e_local.item())

    # work counts for the roofline (graph of the last step).  N > 1: every rank sees only its
    # table window, so the rows' addresses are all-gathered (evaluation only) and each rank
    # sums its window's bucket sizes for every query; the sums are all-reduced.
    idx.clear()
    step()
    torch.cuda.synchronize()
    addrs_local = idx.hash_addrs(d_rp, d_col)
    counts = [bounds[g + 1] - bounds[g] for g in range(world)]
    addrs_np = flash.as_u32(fdist.all_gather_rows(addrs_local, counts) if world > 1 else addrs_local)
    _, _, w0, w1 = idx.dist_info() if use_dist_handle else (0, 1, 0, L)
    per_q, arrivals = query_work(lambda t: idx.table(t), addrs_np, range(w0, w1))
    x1_bytes = x2_bytes = 0
    per_step = {name: phase_ms[i] / max(phase_calls[i], 1) * (phase_calls[i] / args.steps)
                for i, name in enumerate(["hash", "build", "query", "copy"])}
    if use_dist_handle:
        own = np.zeros(shape.N, dtype=bool)
        own[bounds[rank]:bounds[rank + 1]] = True
        # bytes this rank stores into the other GPUs per graph: its rows' addresses for the
        # other windows (X1) and its window's candidates of the other ranks' queries (X2)
        xb = torch.tensor([4 * n_local * (L - (w1 - w0)), 4 * int(per_q[~own].sum())], dtype=torch.int64,
                          device=dev)
        dist.all_reduce(xb, op=dist.ReduceOp.MAX)
        x1_bytes, x2_bytes = int(xb[0].item()), int(xb[1].item())
        pq = torch.from_numpy(per_q).to(dev)
        dist.all_reduce(pq)  # windows partition the tables: the sum is each query's candidates
        per_q = pq.cpu().numpy()
    if world > 1:  # phase times: the slowest rank
        pt = torch.tensor([per_step[k] for k in ("hash", "build", "query", "copy")], dtype=torch.float64, device=dev)
        dist.all_reduce(pt, op=dist.ReduceOp.MAX)
        per_step = dict(zip(("hash", "build", "query", "copy"), pt.tolist()))
    n_cand = int(per_q.sum())  # every query of the graph (all ranks)

    result = None
    if rank == 0:
        hbm_peak, peak_kind = peaks()
        N = shape.N
        # algorithmic bytes, whole graph over all GPUs
        hash_bytes = 4 * nnz_total + 8 * (N + 1) + 4 * L * N
        query_bytes = (4 * L + 8 * L + 8 * TOPK) * N + 4 * n_cand
        hash_ms = per_step["hash"]
        query_ms = per_step["query"]
        build_ms = per_step["build"]
        dominant = max(("hash", hash_ms), ("build", build_ms), ("query", query_ms), key=lambda x: x[1])[0]
        traffic = {}  # ncu --set full DRAM bytes of one graph, summed per kernel name
        issue = {}    # ncu warp instructions and durations per kernel name
        try:
            with open(TRAFFIC_PATH) as f:
                for d in json.load(f):
                    nm = d["kernel"].split("::")[-1].split("<")[0]
                    if d.get("dram_traffic_bytes") is not None:
                        traffic[nm] = traffic.get(nm, 0.0) + d["dram_traffic_bytes"]
                    if d.get("warp_inst") is not None and d.get("duration_ms"):
                        w, t = issue.get(nm, (0.0, 0.0))
                        issue[nm] = (w + d["warp_inst"], t + d["duration_ms"])
        except Exception:
            pass
        peak_all = hbm_peak * world  # GB/s over the job's GPUs
        if dominant == "query":
            qk = ("k_query_mark", "k_query_sort", "k_query", "k_query_csort", "k_query_plan")
            q_traffic = (sum(traffic.get(nm, 0.0) for nm in qk)
                         if any(nm in traffic for nm in qk[:2]) and world == 1 else None)
            roof = {"kernel": "query phase: k_query_plan, then k_query_mark (occupancy bitmap, queries with > 768 "
                              "candidates) and the k_query_sort<MCAP,BL> size classes (the rest)"
                              + ("; + k_dist_gather peer stores" if world > 1 else ""),
                    "bound": "hbm", "achieved": query_bytes / (query_ms * 1e-3) / 1e9, "peak": peak_all,
                    "unit": "GB/s", "peak_kind": peak_kind, "traffic": q_traffic, "algorithmic_bytes": query_bytes,
                    "bytes_formula": "(4L + 8L + 8k) B/query + 4 B/candidate (SURVEY 8(d))", "candidates": n_cand,
                    # diagnostics: the count step needs >= 1 shared-memory RMW per candidate
                    "smem_view": {"achieved_candidates_per_s": n_cand / (query_ms * 1e-3), "peak": SMEM_RMW_PEAK * world,
                                  "frac": n_cand / (query_ms * 1e-3) / (SMEM_RMW_PEAK * world),
                                  "peak_kind": "measured smem RMW microbench (profiles/r01_microbench_smem.txt)"}}
            if any(nm in issue for nm in ("k_query_mark", "k_query_sort")) and world == 1:
                # instruction-issue view from the committed ncu capture: warp instructions
                # issued per second by the query kernels vs 4 schedulers x 148 SMs x clock
                w = sum(issue.get(nm, (0.0, 0.0))[0] for nm in ("k_query_mark", "k_query_sort"))
                t = sum(issue.get(nm, (0.0, 0.0))[1] for nm in ("k_query_mark", "k_query_sort"))
                peak_issue = 4 * 148 * clk_mhz_for_peak() * 1e6
                roof["issue_view"] = {"kernel": "k_query_mark + k_query_sort (ncu)", "warp_inst": w,
                                      "warp_inst_per_query": w / N, "achieved_warp_inst_per_s": w / (t * 1e-3),
                                      "peak_warp_inst_per_s": peak_issue, "frac": w / (t * 1e-3) / peak_issue}
        elif dominant == "build":
            bbytes = 8 * L * N * 2 + 12 * L * N
            roof = {"kernel": "build (k_count..k_select_big)", "bound": "hbm",
                    "achieved": bbytes / (build_ms * 1e-3) / 1e9, "peak": peak_all, "unit": "GB/s",
                    "peak_kind": peak_kind, "traffic": None, "algorithmic_bytes": bbytes}
        else:
            roof = {"kernel": "k_doph", "bound": "hbm", "achieved": hash_bytes / (hash_ms * 1e-3) / 1e9,
                    "peak": peak_all, "unit": "GB/s", "peak_kind": peak_kind,
                    "traffic": traffic.get("k_doph") if world == 1 else None, "algorithmic_bytes": hash_bytes}
        hash_roof = {"kernel": "k_doph", "bound": "hbm", "achieved": hash_bytes / (hash_ms * 1e-3) / 1e9,
                     "peak": peak_all, "unit": "GB/s", "frac": hash_bytes / (hash_ms * 1e-3) / 1e9 / peak_all,
                     "traffic": traffic.get("k_doph") if world == 1 else None, "algorithmic_bytes": hash_bytes}
        roof["frac"] = roof["achieved"] / roof["peak"]
        value = N / (ms_step * 1e-3)
        h2d = 8 * (n_local + 1) + 4 * nnz_local
        d2h = 8 * n_local * TOPK
        result = {
            "metric": METRIC,
            "value": value,
            "unit": "queries/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "graph_time_s": ms_step * 1e-3,
            "hash_nnz_per_s": nnz_total / (hash_ms * 1e-3) if hash_ms else None,
            "queries_per_s": N / (ms_step * 1e-3),
            "phase_ms_per_step": per_step,
            "hash_roofline": hash_roof,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic (synth/, webspam shape, seed 2)",
            "config": workload_config(shape, nnz_total, args),
            "roofline": roof,
            "e2e": {"value": N / (e2e_ms_max * 1e-3), "unit": "queries/s",
                    "ms_per_step": e2e_ms_max, "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h * world,
                    "api": "flash_knn_graph_host (pinned host buffers)" if (world == 1 or use_dist_handle) else
                           f"host copies + dist {args.mode} graph"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world > 1:
            result["exchange_bytes_per_gpu"] = {"x1_addresses": x1_bytes, "x2_candidates": x2_bytes,
                                                "note": "max over ranks, stored into peer GPUs per graph"}
        result["candidates_per_query"] = {"mean": n_cand / N, "p99": float(np.percentile(per_q, 99)),
                                          "max": int(per_q.max())}
        result["bucket_arrivals"] = arrivals
        if world == 1 and not args.no_quality:
            t0 = time.time()
            result["data_stats"] = data_quality_stats(h_rp, d_col, out_ids, n_q=args.quality_queries)
            log(f"data/quality stats in {time.time() - t0:.1f}s")
    idx.close()
    return result


# Secondary workloads (BASELINE.json configs[2], configs[3]): index every row, then answer
# 10K sampled rows as queries with self-exclusion.  Index parameters from the
# paper's own runs: url K=4, L=128, R=32, 2^15; kdd12 K=4,
# L=32, R=64, 2^20.
SHAPE_CFG = {
    "url": dict(K=4, L=128, R=32, range_=1 << 15, seed=0x5EED0003, k=128, q=10_000, qseed=13),
    "kdd12": dict(K=4, L=32, R=64, range_=1 << 20, seed=0x5EED0004, k=128, q=10_000, qseed=14),
    # the friendster 20-NN graph from scratch (the paper
    # gives no K/L/R for it: kdd12's K=4, L=32, R=64, 2^20 for a dataset of that scale)
    "friendster": dict(K=4, L=32, R=64, range_=1 << 20, seed=0x5EED0005, k=20, graph=True, heavy_thr=0.65,
                       paper="friendster 20-NN graph from scratch: 1578 s on 2x Xeon E5-2660 v4, 56 threads (P:505)"),
    # the 10 K-query url line is latency-scale, so also the full url graph
    # (Q = N = 2.39 M queries, ~L*R = 4096 candidates each: the CTA-per-query class)
    "url-graph": dict(shape="url", K=4, L=128, R=32, range_=1 << 15, seed=0x5EED0003, k=128, graph=True),
    # saturated buckets beside the headline: the webspam rows and index with
    # 2^10 buckets per table, so buckets hold ~342 arrivals > R and a query gathers ~L*R
    "webspam-sat": dict(shape="webspam", K=4, L=50, R=128, range_=1 << 10, seed=0x5EED0002, k=128, graph=True),
}


def sample_query_csr(h_rp, h_col, rows):
    """CSR of the given rows (host numpy)."""
    rp = np.asarray(h_rp)
    lens = rp[rows + 1] - rp[rows]
    q_rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = np.asarray(h_col)
    q_col = np.concatenate([col[rp[r]: rp[r + 1]] for r in rows]) if len(rows) else np.zeros(1, col.dtype)
    return q_rp, q_col


def shape_stats(idx, q_addrs, lens, L_, R_, rng_):
    """SURVEY §8(d) statistics beside a secondary-shape timing, computed on the device from
    the built index: nnz mean / p99, candidates per query (sum of its L bucket sizes) and
    the bucket-arrival histogram (log2 bins).  Evaluation only."""
    import torch

    goff, _, arr = idx.table_arrays(ids=False)
    sizes = goff[1:] - goff[:-1]
    a = q_addrs.to(torch.int64) & 0xFFFFFFFF
    valid = a < rng_
    tb = torch.arange(L_, device=a.device, dtype=torch.int64)[None, :] * rng_
    per_q = torch.where(valid, sizes[(tb + a.clamp(max=rng_ - 1))], torch.zeros_like(a)).sum(1).cpu().numpy()
    arr = arr.to(torch.int64)
    lg = torch.zeros_like(arr)
    nz = arr > 0
    lg[nz] = torch.floor(torch.log2(arr[nz].double())).to(torch.int64) + 1
    hist = torch.bincount(lg, minlength=34)[:34].cpu().numpy()
    top = int(np.nonzero(hist)[0].max()) if hist.any() else 0
    labels = ["0"] + [f"{1 << (i - 1)}-{(1 << i) - 1}" for i in range(1, top + 1)]
    return {"nnz_mean": float(lens.mean()), "nnz_p99": float(np.percentile(lens, 99)),
            "candidates_per_query": {"mean": float(per_q.mean()), "p99": float(np.percentile(per_q, 99)),
                                     "max": int(per_q.max())},
            "bucket_arrivals": {"buckets": int(hist.sum()), "histogram_log2": dict(zip(labels, hist[: top + 1].tolist())),
                                "frac_over_R": float((arr > R_).double().mean().item())}}


def run_shape_graph(args, cfg, shape):
    """N=1 line for a k-NN graph of a secondary shape (friendster): one step =
    flash_knn_graph over every row (hash, build, query all rows).  value = rows/s."""
    import torch

    from paper_1709_01190_b200 import flash

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    t0 = time.time()
    h_rp, h_col, nnz = gen_local(shape, [0, shape.N], 0)
    log(f"generated {shape.N} rows nnz={nnz} in {time.time() - t0:.1f}s")
    d_rp, d_col = h_rp.to(dev), h_col.to(dev)
    k = cfg["k"]
    out_ids = torch.empty((shape.N, k), dtype=torch.int32, device=dev)
    out_cnt = torch.empty_like(out_ids)
    idx = flash.FlashIndex(cfg["K"], cfg["L"], cfg["R"], cfg["range_"], cfg["seed"])
    stream = torch.cuda.current_stream()

    def step():
        idx.clear()
        flash.flash_knn_graph(idx.h, d_rp, d_col, shape.N, k, out_ids, out_cnt)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    flash.flash_reset_counters(idx.h)
    flash.flash_set_profiling(idx.h, True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    phase_ms, _ = flash.flash_phase_ms(idx.h)
    launches = flash.flash_launch_count(idx.h)
    flash.flash_set_profiling(idx.h, False)
    lens = np.diff(h_rp.numpy())
    hbm_peak, peak_kind = peaks()
    hash_ms = phase_ms[0] / args.steps
    query_ms = phase_ms[2] / args.steps
    hash_bytes = 4 * nnz + 8 * (shape.N + 1) + 4 * cfg["L"] * shape.N
    # after the timed region: candidates per query and the query-phase roofline (SURVEY 8(d)
    # bytes), and the quality metric the paper quotes for this run, if any
    M = graph_candidates(idx, d_rp, d_col, shape.N, cfg["L"], cfg["range_"]).double()
    n_cand = float(M.sum().item())
    qbytes = (12 * cfg["L"] + 8 * k) * shape.N + 4 * n_cand
    cand = {"mean": float(M.mean().item()), "p99": float(torch.quantile(M[:1 << 20], 0.99).item()),
            "max": float(M.max().item()), "of_LR": float(M.mean().item()) / (cfg["L"] * cfg["R"])}
    del M
    idx.close()
    quality = None
    if cfg.get("heavy_thr") and not args.no_quality:
        qs = np.sort(np.random.default_rng(13).choice(shape.N, size=args.quality_queries, replace=False))
        quality = heavy_recall(h_rp, d_col, out_ids, qs, cfg["heavy_thr"])
        quality["definition"] = ("recall of the neighbours with exact binary cosine > threshold in the reported "
                                 f"top-{k}, over {qs.size} sampled rows (P:507)")
    return {
        "metric": METRIC, "value": shape.N / (ms * 1e-3), "unit": "queries/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "graph_time_s": ms * 1e-3,
        "hash_nnz_per_s": nnz / (hash_ms * 1e-3),
        "phase_ms_per_step": {"hash": hash_ms, "build": phase_ms[1] / args.steps, "query": phase_ms[2] / args.steps},
        "hash_roofline": {"kernel": "k_doph_sparse + k_doph", "bound": "hbm",
                          "achieved": hash_bytes / (hash_ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                          "peak_kind": peak_kind, "frac": hash_bytes / (hash_ms * 1e-3) / 1e9 / hbm_peak,
                          "algorithmic_bytes": hash_bytes},
        "query_roofline": {"kernel": "query phase", "bound": "hbm", "achieved": qbytes / (query_ms * 1e-3) / 1e9,
                           "peak": hbm_peak, "unit": "GB/s", "frac": qbytes / (query_ms * 1e-3) / 1e9 / hbm_peak,
                           "algorithmic_bytes": qbytes, "candidates": n_cand,
                           "candidates_per_s": n_cand / (query_ms * 1e-3)},
        "candidates_per_query": cand, "quality": quality,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": f"synthetic (synth/, {shape.name} shape, seed {shape.seed})",
        "config": {"workload": f"{args.workload}: {shape.name}-shaped approximate {k}-NN graph from scratch",
                   "N": shape.N, "D": shape.D, "nnz": nnz, "nnz_per_row": round(nnz / shape.N, 1),
                   "K": cfg["K"], "L": cfg["L"], "R": cfg["R"], "range": cfg["range_"], "k": k,
                   "seed": cfg["seed"], "parallelism": "1 GPU",
                   "l2_policy": f"inputs larger than L2 (col_idx {4 * nnz / 1e9:.1f} GB vs 126 MB L2); no flush"},
        "paper": cfg.get("paper"),
        "gpu_launches": launches, "clocks": clk.summary(),
        "data_stats": {"nnz_mean": float(lens.mean()), "nnz_p99": float(np.percentile(lens, 99)),
                       "nnz_max": int(lens.max())},
    }


def run_shape(args):
    """Line for the url / kdd12 shapes: one step = index all N rows (H1-H3, B1-B2) + 10K
    sampled queries (H1-H3 of the query rows, Q1-Q3).  value = queries/s of the query phase;
    the index time and hash nnz/s are reported beside it.  Under torchrun (N > 1) the rows
    are sharded over the GPUs and indexed / queried through the multi-GPU handle (kdd12's
    "tables sharded over 8 B200", BASELINE.json configs[3]); max over ranks."""
    import torch

    from paper_1709_01190_b200 import flash

    rank, world, local = dist_env()
    cfg = SHAPE_CFG[args.workload]
    shape = synth.SHAPES[cfg.get("shape", args.workload)]
    if cfg.get("graph"):
        assert world == 1, "the graph workloads other than the headline run on one GPU"
        return run_shape_graph(args, cfg, shape)
    import torch.distributed as dist

    from paper_1709_01190_b200 import dist as fdist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # N > 1 (torchrun; or --dist-handle at N = 1): the multi-GPU handle — tables partitioned
    # over the GPUs, rank g indexes its contiguous row shard (ids = global row numbers) and
    # answers the sampled queries that fall in its shard, both collectively (flash.h)
    use_dist = world > 1 or args.dist_handle
    if use_dist and not dist.is_initialized():
        for key, val in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533"), ("RANK", "0"), ("WORLD_SIZE", "1")):
            os.environ.setdefault(key, val)
        dist.init_process_group("nccl", device_id=dev)
    t0 = time.time()
    import ctypes

    all_lens = np.empty(shape.N, dtype=np.int64)
    synth._load().synth_row_lengths(ctypes.byref(synth._cparams(shape)), 0, shape.N, all_lens.ctypes.data)
    bounds = fdist.shard_bounds(all_lens, world) if world > 1 else [0, shape.N]
    r0, r1 = bounds[rank], bounds[rank + 1]
    n_local = r1 - r0
    h_rp, h_col, nnz_local = gen_local(shape, bounds, rank)
    nnz = int(all_lens.sum())
    log(f"[rank {rank}] generated rows {r0}..{r1} nnz={nnz_local} in {time.time() - t0:.1f}s")
    rows = np.sort(np.random.default_rng(cfg["qseed"]).choice(shape.N, size=cfg["q"], replace=False))
    mine = rows[(rows >= r0) & (rows < r1)]
    q_rp, q_col = sample_query_csr(h_rp.numpy(), h_col.numpy(), mine - r0)
    d_rp, d_col = h_rp.to(dev), h_col.to(dev)
    dq_rp = torch.from_numpy(q_rp).to(dev)
    dq_col = torch.from_numpy(np.ascontiguousarray(q_col).view(np.int32)).to(dev)
    excl = torch.from_numpy(mine.astype(np.uint32).view(np.int32)).to(dev)
    k = cfg["k"]
    nq = int(mine.size)
    out_ids = torch.empty((max(nq, 1), k), dtype=torch.int32, device=dev)
    out_cnt = torch.empty((max(nq, 1), k), dtype=torch.int32, device=dev)
    idx = (fdist.create_dist_index(cfg["K"], cfg["L"], cfg["R"], cfg["range_"], cfg["seed"]) if use_dist
           else flash.FlashIndex(cfg["K"], cfg["L"], cfg["R"], cfg["range_"], cfg["seed"]))
    stream = torch.cuda.current_stream()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]

    def step(ev=None):
        idx.clear()
        if ev:
            ev[0].record(stream)
        flash.flash_insert(idx.h, d_rp, d_col, n_local, r0)
        if ev:
            ev[1].record(stream)
        flash.flash_query_topk(idx.h, dq_rp, dq_col, nq, k, excl, out_ids, out_cnt)
        if ev:
            ev[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    flash.flash_reset_counters(idx.h)
    flash.flash_set_profiling(idx.h, True)
    if use_dist:
        dist.barrier()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            step(evs[i])
        torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    index_ms = statistics.median(e[0].elapsed_time(e[1]) for e in evs)
    query_ms = statistics.median(e[1].elapsed_time(e[2]) for e in evs)
    phase_ms, phase_calls = flash.flash_phase_ms(idx.h)
    launches = flash.flash_launch_count(idx.h)
    flash.flash_set_profiling(idx.h, False)
    if world > 1:  # the slowest rank
        t = torch.tensor([index_ms, query_ms] + list(phase_ms[:3]), dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        index_ms, query_ms = float(t[0]), float(t[1])
        phase_ms = [float(x) for x in t[2:]] + [0.0]
    stats = (shape_stats(idx, idx.hash_addrs(dq_rp, dq_col), np.diff(h_rp.numpy()), cfg["L"], cfg["R"],
                         cfg["range_"]) if not use_dist else {"nnz_mean": float(all_lens.mean())})
    # the hash phase covers the indexed rows and the query rows; split by nnz
    hash_ms_all = phase_ms[0] / args.steps
    q_nnz = int(q_rp[-1])
    hash_ms_index = hash_ms_all * nnz_local / max(nnz_local + q_nnz, 1)
    hbm_peak, peak_kind = peaks()
    L_ = cfg["L"]
    hash_bytes = 4 * nnz + 8 * (shape.N + 1) + 4 * L_ * shape.N
    idx.close()
    if use_dist:
        dist.barrier()
    if rank != 0:
        return None
    return {
        "metric": METRIC,
        "value": cfg["q"] / (query_ms * 1e-3),
        "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": index_ms + query_ms,
        "index_time_s": index_ms * 1e-3,
        "query_time_s": query_ms * 1e-3,
        "hash_nnz_per_s": nnz / (hash_ms_index * 1e-3),
        "phase_ms_per_step": {"hash": hash_ms_all, "build": phase_ms[1] / args.steps,
                              "query": phase_ms[2] / args.steps},
        "hash_roofline": {"kernel": "k_doph", "bound": "hbm",
                          "achieved": hash_bytes / (hash_ms_index * 1e-3) / 1e9,
                          "peak": hbm_peak * world, "unit": "GB/s", "peak_kind": peak_kind,
                          "frac": hash_bytes / (hash_ms_index * 1e-3) / 1e9 / (hbm_peak * world),
                          "algorithmic_bytes": hash_bytes,
                          "note": "densification makes this shape ALU-bound (DESIGN.md §6)"},
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": f"synthetic (synth/, {args.workload} shape, seed {shape.seed})",
        "config": {"workload": f"{args.workload}-shaped: index all rows + {cfg['q']} sampled queries, top-{k}",
                   "N": shape.N, "D": shape.D, "nnz": nnz, "nnz_per_row": round(nnz / shape.N, 1),
                   "K": cfg["K"], "L": L_, "R": cfg["R"], "range": cfg["range_"], "k": k,
                   "seed": cfg["seed"], "query_seed": cfg["qseed"],
                   "parallelism": (f"rows x{world} (hash, queries); tables x{world} (build, gather); "
                                   "flash_create_dist") if use_dist else "1 GPU",
                   "l2_policy": f"inputs larger than L2 (col_idx {4 * nnz / 1e9:.1f} GB vs 126 MB L2); no flush"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "data_stats": stats,
    }


def host_cpu():
    """lscpu model / sockets and the OpenMP thread count the oracle runs with."""
    info = {"model": None, "sockets": None}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() == "Model name":
                info["model"] = v.strip()
            elif k.strip() == "Socket(s)":
                info["sockets"] = int(v.strip())
    except Exception:
        pass
    info["omp_threads"] = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return info


def tiny_one_thread_s():
    """the tiny graph on the oracle with ONE thread (a subprocess with
    OMP_NUM_THREADS=1; median of 3)."""
    code = ("import sys,time,statistics; sys.path.insert(0, %r); import oracle, synth; "
            "rp, col = synth.generate('tiny'); ts = []\n"
            "for _ in range(3):\n t = time.perf_counter(); "
            "oracle.knn_graph(4, 16, 32, 1 << 15, 0x5EED0001, rp, col, 10); ts.append(time.perf_counter() - t)\n"
            "print(statistics.median(ts))") % ROOT
    try:
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300,
                             env=dict(os.environ, OMP_NUM_THREADS="1"))
        return float(out.stdout.strip().splitlines()[-1])
    except Exception:
        return None


def cpu_baseline(sample_queries: int, steps: int = 1):
    """The oracle as it stands on the host cores: full hash + build, a query sample."""
    import oracle

    shape = synth.SHAPES["webspam"]
    rp, col = synth.generate(shape)
    n = rp.size - 1
    cpu = host_cpu()
    cores = cpu["omp_threads"]
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        codes = oracle.doph(K, L, SEED, rp, col)
        addrs = oracle.addresses(K, L, RANGE, SEED, codes)
        del codes
        t1 = time.perf_counter()
        T = oracle.build(L, R, RANGE, SEED, addrs, np.arange(n, dtype=np.uint32))
        t2 = time.perf_counter()
        q = np.random.default_rng(0).choice(n, size=sample_queries, replace=False)
        oracle.query(T, addrs[q], TOPK, exclude=q.astype(np.uint32))
        t3 = time.perf_counter()
        graph_s = (t1 - t0) + (t2 - t1) + (t3 - t2) * n / sample_queries
        times.append((graph_s, t1 - t0, t2 - t1, t3 - t2))
    g = statistics.median(x[0] for x in times)
    return {"value": n / g, "unit": "queries/s", "cores": cores, "kind": "oracle",
            "sample": f"hash+build of all {n} rows, top-{TOPK} for {sample_queries} sampled rows, "
                      f"query time extrapolated x{n / sample_queries:.1f}",
            "graph_s_extrapolated": g, "hash_s": times[-1][1], "build_s": times[-1][2],
            "query_sample_s": times[-1][3], "cpu_model": cpu["model"], "sockets": cpu["sockets"],
            "nnz": int(rp[-1]), "tiny_graph_1_thread_s": tiny_one_thread_s()}, times


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    shape = synth.SHAPES["webspam"]
    cb, times = cpu_baseline(args.ref_sample, steps=args.warmup + args.steps)
    timed = times[args.warmup:]
    g = statistics.median(x[0] for x in timed)
    return {
        "metric": METRIC, "impl": "reference", "value": shape.N / g, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": g * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (synth/, webspam shape, seed 2)",
        "config": workload_config(shape, cb["nnz"], args),
        "cpu_baseline": cb,
        "e2e": {"value": shape.N / g, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["exchange", "sharded"], default="exchange",
                    help="N>1: candidate all-to-all over partitioned tables (north_star (d)) or "
                         "sharded build + table all-gather")
    ap.add_argument("--ref-sample", type=int, default=350000, help="oracle query sample (rows; all = full graph)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-quality", action="store_true", help="skip the data statistics and R@k/S@k")
    ap.add_argument("--quality-queries", type=int, default=1000)
    ap.add_argument("--dist-handle", action="store_true",
                    help="url / kdd12 at N = 1 through the multi-GPU handle (flash_create_dist, NCCL world 1)")
    ap.add_argument("--workload", choices=["webspam", "url", "kdd12", "friendster", "url-graph", "webspam-sat"],
                    default="webspam",
                    help="webspam = the headline graph (default); url / kdd12 = secondary N=1 lines; "
                         "friendster / url-graph = full k-NN graphs of those shapes")
    args = ap.parse_args()
    # the JSON line must be the only stdout line: NCCL prints its version banner to stdout
    # whatever NCCL_DEBUG says, so fd 1 is pointed at stderr for the run and the line is
    # written to the saved original
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    sys.stdout.flush()
    out_fd = os.dup(1)
    os.dup2(2, 1)

    def emit(res):
        os.write(out_fd, (json.dumps(res) + "\n").encode())

    if args.workload != "webspam" and args.impl == "ours":
        res = run_shape(args)
        if res is not None:
            emit(res)
        return
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            emit(res)
        return
    res = run_ours(args)
    rank, world, _ = dist_env()
    if rank == 0 and res is not None:
        if world == 1 and not args.no_cpu_baseline:
            cb, _ = cpu_baseline(args.ref_sample, steps=1)
            res["cpu_baseline"] = cb
        emit(res)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
