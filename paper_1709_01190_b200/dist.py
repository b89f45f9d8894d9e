"""Multi-GPU plumbing (one process per GPU).

The product path is the multi-GPU handle of libflash.so (include/flash.h
flash_create_dist; csrc/dist.cu): the L tables partitioned over the GPUs, addresses and
candidate lists exchanged as peer stores inside the library's kernels, stream-ordered NCCL
barriers.  Python only bootstraps it: ``create_dist_index`` broadcasts the NCCL unique id
(torch.distributed, any backend) and wraps the rank's handle.

The schedules below are the same partitioning written against torch.distributed
collectives and the single-GPU C ABI: ``knn_graph_replicated`` is the multi-GPU path of an
index with reservoir sharing (F < 1: a shared pool does not partition by table), and
``knn_graph_candidate_exchange`` / ``knn_graph_sharded_build`` are the torch-collective
formulations of the table partition, kept as the CPU (gloo) model of the exchange in
tests/test_dist_gloo.py.


Replicated-table mode: rank g holds a contiguous, nnz-balanced row
shard; it hashes its own rows (H1-H3), the L addresses of every row are all-gathered
(one collective, N*L*4 bytes: 70 MB for webspam), every rank builds the SAME tables
(bottom-R is deterministic and partition-free), and rank g queries only its own rows
with exclude = global row id.  Results are byte-identical at every GPU count.

The "index" object is anything with hash_addrs / insert_addrs / query_addrs: the
product passes a paper_1709_01190_b200.flash.FlashIndex (CUDA kernels through the
C ABI, NCCL via torch.distributed); the CPU multi-process tests pass an oracle-backed
stand-in over gloo to check the partition / gather / id logic.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def bootstrap_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id (flash_get_unique_id); every rank receives it
    (torch.distributed.broadcast_object_list: works over gloo and NCCL process groups)."""
    from paper_1709_01190_b200 import flash

    obj = [flash.flash_get_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def create_dist_index(K: int, L: int, R: int, range_: int, seed: int, group=None):
    """This rank's FlashIndex of a multi-GPU handle (flash_create_dist, collective) on the
    current CUDA device; world / rank from the torch.distributed group."""
    from paper_1709_01190_b200 import flash

    uid = bootstrap_unique_id(group)
    h = flash.flash_create_dist(K, L, R, range_, seed, dist.get_rank(group), dist.get_world_size(group), uid)
    return flash.FlashIndex(K, L, R, range_, seed, handle=h)


def shard_bounds(row_lengths: np.ndarray, world: int) -> list[int]:
    """Contiguous row shards with ~equal nnz: bounds[g]..bounds[g+1] is rank g's range."""
    n = int(row_lengths.size)
    cum = np.concatenate([[0], np.cumsum(row_lengths, dtype=np.int64)])
    total = int(cum[-1])
    bounds = [0]
    for g in range(1, world):
        target = total * g / world
        r = int(np.searchsorted(cum, target, side="left"))
        r = max(bounds[-1], min(n, r))
        bounds.append(r)
    bounds.append(n)
    return bounds


def all_gather_rows(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """Concatenate every rank's [n_g, ...] tensor in rank order (variable n_g)."""
    world = len(counts)
    if world == 1:
        return local
    m = max(counts)
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    parts = [out[g * m: g * m + counts[g]] for g in range(world)]
    return torch.cat(parts, dim=0)


def knn_graph_replicated(index, row_ptr_local, col_idx_local, k: int, bounds: list[int],
                         rank: int, group=None):
    """k-NN graph rows of this rank's shard (global ids), identical to a 1-GPU graph."""
    world = len(bounds) - 1
    counts = [bounds[g + 1] - bounds[g] for g in range(world)]
    n_local = counts[rank]
    addrs_local = index.hash_addrs(row_ptr_local, col_idx_local)          # H1-H3 on own rows
    addrs_all = all_gather_rows(addrs_local, counts, group)                # X: addresses
    index.insert_addrs(addrs_all, 0)                                       # B1-B2, all tables
    excl = torch.arange(bounds[rank], bounds[rank] + n_local, dtype=torch.int64,
                        device=addrs_local.device).to(torch.int32)
    return index.query_addrs(addrs_local, k, excl)                         # Q1-Q3, own rows


def table_window(L: int, world: int, rank: int) -> tuple[int, int]:
    """Tables [floor(rank*L/world), floor((rank+1)*L/world)) are built by `rank` (R#22 of
    SURVEY §8(c): floor-block partition; results do not depend on it)."""
    return (L * rank) // world, (L * (rank + 1)) // world


def _gather_var(x: torch.Tensor, sizes: list[int], group=None) -> list[torch.Tensor]:
    """All-gather 1-D tensors of per-rank length sizes[g] (padded to the max)."""
    world = len(sizes)
    m = max(max(sizes), 1)
    pad = torch.zeros(m, dtype=x.dtype, device=x.device)
    pad[: x.numel()] = x
    out = torch.empty(world * m, dtype=x.dtype, device=x.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return [out[g * m: g * m + sizes[g]] for g in range(world)]


def knn_graph_sharded_build(index, row_ptr_local, col_idx_local, k: int, bounds: list[int], rank: int,
                            group=None):
    """Multi-GPU k-NN graph with the table build sharded across GPUs:

    1. rank g hashes its row shard (H1-H3, all L tables);
    2. X1: the addresses of every row are all-gathered (N*L*4 bytes);
    3. rank g builds only its table window [t0, t1) over all N rows (B1-B2; bottom-R is
       per bucket and keyed by the global table index, so a window equals the
       corresponding tables of a full build);
    4. X2: the built windows (bucket offsets + kept ids) are all-gathered, and every rank
       imports the full, identical tables;
    5. rank g answers its own rows (Q1-Q3) with exclude = global row id.
    Results are byte-identical to the 1-GPU graph."""
    world = len(bounds) - 1
    counts = [bounds[g + 1] - bounds[g] for g in range(world)]
    n_local = counts[rank]
    n_total = bounds[-1]
    L, R = index.L, index.range
    addrs_local = index.hash_addrs(row_ptr_local, col_idx_local)               # H1-H3
    addrs_all = all_gather_rows(addrs_local, counts, group)                     # X1
    t0, t1 = table_window(L, world, rank)
    index.insert_addrs_window(addrs_all, 0, t0, t1)                            # B1-B2 (own tables)
    goff, ids, arr = index.table_arrays()
    lo, hi = int(goff[t0 * R].item()), int(goff[t1 * R].item())
    rel = goff[t0 * R: t1 * R + 1] - lo                                         # window offsets
    my_ids = ids[lo:hi]
    wsizes = [(table_window(L, world, g)[1] - table_window(L, world, g)[0]) * R + 1 for g in range(world)]
    nsz = torch.tensor([hi - lo], dtype=torch.int64, device=goff.device)
    allsz = torch.empty(world, dtype=torch.int64, device=goff.device)
    dist.all_gather_into_tensor(allsz, nsz, group=group)
    isizes = [int(v) for v in allsz.tolist()]
    rels = _gather_var(rel, wsizes, group)                                      # X2
    idss = _gather_var(my_ids, isizes, group)
    dist.all_reduce(arr, op=dist.ReduceOp.SUM, group=group)                     # disjoint windows
    parts, base = [], 0
    for g in range(world):
        parts.append(rels[g][:-1] + base)
        base += isizes[g]
    parts.append(torch.tensor([base], dtype=torch.int64, device=goff.device))
    full_goff = torch.cat(parts).contiguous()
    full_ids = torch.cat(idss).contiguous() if base else torch.zeros(0, dtype=ids.dtype, device=ids.device)
    index.import_tables(full_goff, full_ids, arr.contiguous())
    excl = torch.arange(bounds[rank], bounds[rank] + n_local, dtype=torch.int64,
                        device=addrs_local.device).to(torch.int32)
    return index.query_addrs(addrs_local, k, excl)                             # Q1-Q3 (own rows)


def _splits(x: torch.Tensor) -> list[int]:
    return [int(v) for v in x.tolist()]


def knn_graph_candidate_exchange(index, row_ptr_local, col_idx_local, k: int, bounds: list[int], rank: int,
                                 group=None):
    """Multi-GPU k-NN graph with the L tables PARTITIONED across GPUs and candidate lists
    exchanged to each query's owner (north_star (d)):

    1. H1-H3: rank g hashes its row shard; the addresses come out owner-blocked
       (flash_hash_blocked), i.e. already in the send layout of
    2. X1: all-to-all of address blocks: rank h receives, for every row, the addresses of
       its own table window [t0(h), t1(h)) — [N][W_h], rows in global order;
    3. B1-B2: rank h builds its window tables over all N rows (flash_insert_addrs_cols);
    4. Q1 (window): rank h gathers every query's window buckets (flash_window_sizes /
       flash_window_gather), in owner order, so each destination's share is contiguous;
    5. X2: all-to-all of the per-query segment sizes, then all-to-all-v of the candidate
       ids, to the query's owner (the rank that hashed the row);
    6. Q2-Q3: the owner counts over its G segments per query and selects the top-k
       (flash_count_topk) with exclude = global row id.
    The candidate multiset of each query is exactly the union of its L buckets, so the
    result is byte-identical to the 1-GPU graph at every world size."""
    world = len(bounds) - 1
    counts = [bounds[g + 1] - bounds[g] for g in range(world)]
    n_local, n_total = counts[rank], bounds[-1]
    L = index.L
    wins = [table_window(L, world, g) for g in range(world)]
    t0, t1 = wins[rank]
    W = t1 - t0
    dev = row_ptr_local.device
    send = index.hash_addrs_blocked(row_ptr_local, col_idx_local, world)             # H1-H3
    recv = torch.empty(n_total * W, dtype=torch.int32, device=dev)
    dist.all_to_all_single(recv, send, [c * W for c in counts],                     # X1
                           [n_local * (w1 - w0) for (w0, w1) in wins], group=group)
    addrs_win = recv.view(n_total, W)
    if W > 0 and n_total > 0:
        index.insert_addrs_cols(addrs_win, 0, t0, t1)                                # B1-B2
    sizes, off = index.window_sizes(addrs_win, t0, t1)                             # Q1 sizes
    cuts = off[torch.tensor(bounds, dtype=torch.int64, device=off.device)]
    send_tot = (cuts[1:] - cuts[:-1]).contiguous()
    cand_send = index.window_gather(addrs_win, t0, t1, off, int(cuts[-1].item()))  # Q1 gather
    seg_sizes = torch.empty(world * n_local, dtype=torch.int32, device=dev)
    dist.all_to_all_single(seg_sizes, sizes.contiguous(), [n_local] * world, counts, group=group)   # X2a
    recv_tot = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_to_all_single(recv_tot, send_tot, group=group)
    rs, ss = _splits(recv_tot), _splits(send_tot)
    cand_recv = torch.empty(sum(rs), dtype=torch.int32, device=dev)
    dist.all_to_all_single(cand_recv, cand_send, rs, ss, group=group)               # X2b
    excl = torch.arange(bounds[rank], bounds[rank] + n_local, dtype=torch.int64, device=dev).to(torch.int32)
    return index.count_topk(cand_recv, seg_sizes.view(world, n_local), k, max(n_total - 1, 0), excl)  # Q2-Q3
