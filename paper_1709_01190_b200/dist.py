"""Multi-GPU orchestration of the k-NN graph (one process per GPU; plumbing only).

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
