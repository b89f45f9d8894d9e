"""Multi-process (world_size 2 and 3, gloo on CPU) check of the multi-GPU orchestration
in paper_1709_01190_b200/dist.py: row sharding, the address all-gather, global ids and
self-exclusion.  The per-rank compute is stood in for by the CPU oracle (tests only);
on GPUs the same orchestration drives libflash.so over NCCL.  The distributed graph
must equal the single-process oracle graph row for row (identity at every GPU count)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1709_01190_b200 import dist as fdist

CFG = dict(K=4, L=16, R=8, range_=256, seed=0xD157, k=10)


class OracleIndex:
    """CPU stand-in with the FlashIndex methods dist.py uses (hash / insert / query)."""

    def __init__(self, K, L, R, range_, seed):
        self.K, self.L, self.R, self.range, self.seed = K, L, R, range_, seed
        self.T = None

    def hash_addrs(self, row_ptr, col_idx):
        rp = row_ptr.numpy()
        col = col_idx.numpy().view(np.uint32)
        codes = oracle.doph(self.K, self.L, self.seed, rp, col)
        return torch.from_numpy(oracle.addresses(self.K, self.L, self.range, self.seed, codes).view(np.int32))

    def insert_addrs(self, addrs, id_base):
        a = addrs.numpy().view(np.uint32)
        ids = (np.arange(a.shape[0], dtype=np.int64) + id_base).astype(np.uint32)
        self.T = oracle.build(self.L, self.R, self.range, self.seed, a, ids)

    def insert_addrs_window(self, addrs, id_base, t0, t1):
        a = addrs.numpy().view(np.uint32).copy()
        a[:, :t0] = 0xFFFFFFFF  # other tables receive nothing
        a[:, t1:] = 0xFFFFFFFF
        self.insert_addrs(torch.from_numpy(a.view(np.int32)), id_base)

    def table_arrays(self):
        """Flat (goff int64 [L*range+1], ids int32, arrivals int32 [L*range]) like the C ABI."""
        goff, ids, base = [], [], 0
        for t in range(self.L):
            off, kept, _ = self.T.table(t)
            goff.append(off[:-1].astype(np.int64) + base)
            ids.append(kept)
            base += int(off[-1])
        goff.append(np.array([base], np.int64))
        return (torch.from_numpy(np.concatenate(goff)), torch.from_numpy(np.concatenate(ids).view(np.int32)),
                torch.from_numpy(self.T.arrivals.reshape(-1).view(np.int32).copy()))

    def import_tables(self, goff, ids, arrivals):
        g = goff.numpy()
        i = ids.numpy().view(np.uint32)
        off = np.stack([g[t * self.range: (t + 1) * self.range + 1] - g[t * self.range]
                        for t in range(self.L)]).astype(np.uint32)
        stride = max(1, int(off[:, -1].max()))
        kept = np.zeros(self.L * stride, np.uint32)
        for t in range(self.L):
            n = int(off[t, -1])
            kept[t * stride: t * stride + n] = i[g[t * self.range]: g[t * self.range] + n]
        arr = arrivals.numpy().view(np.uint32).reshape(self.L, self.range).copy()
        self.T = oracle.Tables(self.L, self.R, self.range, arr, off, kept, stride)

    # ---- candidate-exchange stand-ins (same semantics as the C ABI, computed by the oracle) ----
    def hash_addrs_blocked(self, row_ptr, col_idx, world):
        a = self.hash_addrs(row_ptr, col_idx).numpy().view(np.uint32)
        blocks = [a[:, fdist.table_window(self.L, world, g)[0]: fdist.table_window(self.L, world, g)[1]].reshape(-1)
                  for g in range(world)]
        return torch.from_numpy(np.concatenate(blocks).view(np.int32))

    def insert_addrs_cols(self, addrs, id_base, t0, t1):
        a = np.full((addrs.shape[0], self.L), 0xFFFFFFFF, np.uint32)
        a[:, t0:t1] = addrs.numpy().view(np.uint32)
        self.insert_addrs(torch.from_numpy(a.view(np.int32)), id_base)

    def _window_lists(self, addrs, t0, t1):
        a = addrs.numpy().view(np.uint32)
        out = []
        for q in range(a.shape[0]):
            parts = []
            for j, t in enumerate(range(t0, t1)):
                if self.T is not None and a[q, j] != 0xFFFFFFFF:
                    off, kept, _ = self.T.table(t)
                    parts.append(kept[off[a[q, j]]: off[a[q, j] + 1]])
            out.append(np.concatenate(parts) if parts else np.zeros(0, np.uint32))
        return out

    def window_sizes(self, addrs, t0, t1):
        lists = self._window_lists(addrs, t0, t1)
        sizes = np.array([x.size for x in lists], np.int64)
        off = np.concatenate([[0], np.cumsum(sizes)])
        return torch.from_numpy(sizes.astype(np.int32)), torch.from_numpy(off.astype(np.int64))

    def window_gather(self, addrs, t0, t1, offsets, total):
        lists = self._window_lists(addrs, t0, t1)
        out = np.concatenate(lists) if lists else np.zeros(0, np.uint32)
        assert out.size == total
        return torch.from_numpy(out.astype(np.uint32).view(np.int32))

    def count_topk(self, cand, seg_sizes, k, max_id, exclude):
        """Q2-Q3 over segments: the oracle's query on a stand-in index whose table s,
        bucket q is segment (s, q)."""
        sz = seg_sizes.numpy().astype(np.int64)
        n_seg, n_q = sz.shape
        c = cand.numpy().view(np.uint32)
        off = np.zeros((n_seg, n_q + 1), np.uint32)
        stride = max(1, int(sz.sum(axis=1).max()) if n_q else 1)
        kept = np.zeros(n_seg * stride, np.uint32)
        base = 0
        for s_ in range(n_seg):
            off[s_, 1:] = np.cumsum(sz[s_])
            n = int(off[s_, -1])
            kept[s_ * stride: s_ * stride + n] = c[base: base + n]
            base += n
        T = oracle.Tables(n_seg, self.R, n_q, np.zeros((n_seg, n_q), np.uint32), off, kept, stride)
        qa = np.tile(np.arange(n_q, dtype=np.uint32)[:, None], (1, n_seg))
        ids, cnt = oracle.query(T, qa, k, exclude=exclude.numpy().astype(np.int64).astype(np.uint32))
        return torch.from_numpy(ids.view(np.int32)), torch.from_numpy(cnt.view(np.int32))

    def query_addrs(self, addrs, k, exclude):
        ids, cnt = oracle.query(self.T, addrs.numpy().view(np.uint32), k,
                                exclude=exclude.numpy().astype(np.int64).astype(np.uint32))
        return torch.from_numpy(ids.view(np.int32)), torch.from_numpy(cnt.view(np.int32))


class OraclePoolIndex(OracleIndex):
    """Reservoir sharing (F < 1, R#23) stand-in: the replicated schedule needs only
    hash / insert / query, which the pool oracle provides."""
    def __init__(self, K, L, R, range_, seed, F):
        super().__init__(K, L, R, range_, seed)
        self.P = oracle.pool_size(F, L, range_)

    def insert_addrs(self, addrs, id_base):
        a = addrs.numpy().view(np.uint32)
        ids = (np.arange(a.shape[0], dtype=np.int64) + id_base).astype(np.uint32)
        self.T = oracle.build_pool(self.L, self.R, self.range, self.P, self.seed, a, ids)

    def query_addrs(self, addrs, k, exclude):
        ids, cnt = oracle.query_pool(self.T, self.seed, addrs.numpy().view(np.uint32), k,
                                     exclude=exclude.numpy().astype(np.int64).astype(np.uint32))
        return torch.from_numpy(ids.view(np.int32)), torch.from_numpy(cnt.view(np.int32))


def _shape():
    return synth.SHAPES["tiny"].with_(N=700, seed=11)


def _worker(rank, world, port, out_dir, mode="replicated"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape = _shape()
        lens = np.diff(synth.generate(shape)[0])
        bounds = fdist.shard_bounds(lens, world)
        rp, col = synth.generate(shape, rows=(bounds[rank], bounds[rank + 1]))
        if mode == "replicated_pool":
            idx = OraclePoolIndex(CFG["K"], CFG["L"], CFG["R"], CFG["range_"], CFG["seed"], POOL_F)
        else:
            idx = OracleIndex(CFG["K"], CFG["L"], CFG["R"], CFG["range_"], CFG["seed"])
        fn = {"replicated": fdist.knn_graph_replicated, "sharded": fdist.knn_graph_sharded_build,
              "exchange": fdist.knn_graph_candidate_exchange, "replicated_pool": fdist.knn_graph_replicated}[mode]
        ids, cnt = fn(idx, torch.from_numpy(rp), torch.from_numpy(col.view(np.int32)), CFG["k"], bounds, rank)
        np.save(os.path.join(out_dir, f"ids_{rank}.npy"), ids.numpy())
        np.save(os.path.join(out_dir, f"cnt_{rank}.npy"), cnt.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,mode", [(2, "replicated"), (3, "replicated"), (2, "sharded"), (3, "sharded"),
                                        (5, "sharded"), (2, "exchange"), (3, "exchange"), (5, "exchange")])
def test_distributed_graph_equals_single_process(tmp_path, world, mode):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), mode), nprocs=world, join=True)
    shape = _shape()
    rp, col = synth.generate(shape)
    want_ids, want_cnt = oracle.knn_graph(CFG["K"], CFG["L"], CFG["R"], CFG["range_"], CFG["seed"], rp, col,
                                          CFG["k"])
    got_ids = np.concatenate([np.load(tmp_path / f"ids_{r}.npy") for r in range(world)]).view(np.uint32)
    got_cnt = np.concatenate([np.load(tmp_path / f"cnt_{r}.npy") for r in range(world)]).view(np.uint32)
    assert np.array_equal(got_ids, want_ids)
    assert np.array_equal(got_cnt, want_cnt)


POOL_F = 0.2


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_graph_with_reservoir_sharing_equals_single_process(tmp_path, world):
    """F < 1 (reservoir sharing, R#23) across processes: the replicated schedule (every rank
    builds the same shared-pool tables from the all-gathered addresses) must give the
    single-process pool graph row for row."""
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), "replicated_pool"), nprocs=world, join=True)
    rp, col = synth.generate(_shape())
    K, L, R, rng, seed, k = CFG["K"], CFG["L"], CFG["R"], CFG["range_"], CFG["seed"], CFG["k"]
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    n = addrs.shape[0]
    T = oracle.build_pool(L, R, rng, oracle.pool_size(POOL_F, L, rng), seed, addrs, np.arange(n, dtype=np.uint32))
    want_ids, want_cnt = oracle.query_pool(T, seed, addrs, k, exclude=np.arange(n, dtype=np.uint32))
    got_ids = np.concatenate([np.load(tmp_path / f"ids_{r}.npy") for r in range(world)]).view(np.uint32)
    got_cnt = np.concatenate([np.load(tmp_path / f"cnt_{r}.npy") for r in range(world)]).view(np.uint32)
    assert np.array_equal(got_ids, want_ids)
    assert np.array_equal(got_cnt, want_cnt)


def test_shard_bounds_balance_nnz_and_cover_all_rows():
    lens = np.random.default_rng(0).integers(1, 5000, size=10_001)
    for world in (1, 2, 3, 8):
        b = fdist.shard_bounds(lens, world)
        assert b[0] == 0 and b[-1] == lens.size and all(x <= y for x, y in zip(b, b[1:]))
        tot = lens.sum()
        for g in range(world):
            share = lens[b[g]:b[g + 1]].sum()
            assert abs(share - tot / world) <= lens.max()


def test_all_gather_rows_handles_uneven_shards(tmp_path):
    port = _free_port()
    mp.spawn(_gather_worker, args=(port, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "g0.npy")
    assert got.tolist() == [[0, 0], [0, 1], [0, 2], [1, 0]]


def _gather_worker(rank, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    try:
        counts = [3, 1]
        local = torch.tensor([[rank, i] for i in range(counts[rank])], dtype=torch.int32)
        out = fdist.all_gather_rows(local, counts)
        if rank == 0:
            np.save(os.path.join(out_dir, "g0.npy"), out.numpy())
    finally:
        dist.destroy_process_group()


def test_nccl_unique_id_bootstrap_reaches_every_rank(tmp_path):
    """dist.bootstrap_unique_id (the multi-GPU handle's bootstrap): rank 0's NCCL unique id
    (flash_get_unique_id, no GPU needed) arrives byte-identical on every rank (gloo, world 3)."""
    mp.spawn(_uid_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    ids = [open(tmp_path / f"uid_{r}.bin", "rb").read() for r in range(3)]
    assert len(ids[0]) == 128 and ids[0] == ids[1] == ids[2]
    assert ids[0] != bytes(128)


def _uid_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = fdist.bootstrap_unique_id()
        with open(os.path.join(out_dir, f"uid_{rank}.bin"), "wb") as f:
            f.write(uid)
    finally:
        dist.destroy_process_group()
