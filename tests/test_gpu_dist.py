"""The multi-GPU handle (flash_create_dist / flash_create_dist_local; north_star (d), SURVEY
§8(b), §8(e)) through the C ABI, bit-exact against the single-process CPU oracle.

One GPU is available, so G ranks run as a local group: G handles on cuda:0, each driven by
its own host thread and stream, exchanging addresses and candidates with peer stores into
each other's buffers and stream-ordered barriers — the same orchestration code as the NCCL
transport (which is exercised here at world 1: bootstrap id, communicator, barriers).
Every case covers the whole collective path: shard-size exchange, hash fused with the
address exchange, per-window build, per-round candidate gather/store, count + top-k."""
import os
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1709_01190_b200 import dist as fdist
from paper_1709_01190_b200 import flash

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "these tests need a B200"
    torch.cuda.set_device(0)
    yield
    torch.cuda.synchronize()


def _shards(rp, col, bounds):
    out = []
    for g in range(len(bounds) - 1):
        r0, r1 = bounds[g], bounds[g + 1]
        srp = rp[r0:r1 + 1] - rp[r0]
        scol = col[rp[r0]:rp[r1]]
        out.append(flash.to_device_csr(srp, scol))
    return out


def _run_ranks(fns):
    """Run fns[g]() in G threads (each rank's collective calls wait for the others)."""
    res, errs = [None] * len(fns), []

    def go(g):
        try:
            torch.cuda.set_device(0)
            res[g] = fns[g]()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=go, args=(g,)) for g in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=180)
    assert not any(t.is_alive() for t in ts), "a rank hung"
    if errs:
        raise errs[0]
    return res


def _local_group(K, L, R, rng, seed, G):
    hs = flash.flash_create_dist_local(K, L, R, rng, seed, G)
    return [flash.FlashIndex(K, L, R, rng, seed, handle=h) for h in hs]


def _dist_graph(idxs, shards, k):
    streams = [torch.cuda.Stream() for _ in idxs]

    def rank(g):
        def f():
            d_rp, d_col = shards[g]
            ids, cnt = idxs[g].knn_graph(d_rp, d_col, k, stream=streams[g])
            streams[g].synchronize()
            return flash.as_u32(ids), flash.as_u32(cnt)
        return f

    out = _run_ranks([rank(g) for g in range(len(idxs))])
    return np.concatenate([o[0] for o in out]), np.concatenate([o[1] for o in out])


GRAPH_CASES = [
    # (name, shape, n, K, L, R, range, k, G, cand_bytes)
    ("tiny_G1", "tiny", 1000, 4, 16, 32, 1 << 15, 10, 1, None),
    ("tiny_G2", "tiny", 1000, 4, 16, 32, 1 << 15, 10, 2, None),
    ("tiny_G3_rounds", "tiny", 1000, 4, 16, 32, 1 << 15, 10, 3, 16 * 32 * 4 * 37),   # 37 queries per round
    ("tiny_G8", "tiny", 1000, 4, 16, 32, 1 << 15, 10, 8, None),
    ("G_gt_L", "tiny", 700, 2, 3, 8, 256, 12, 5, None),                               # two ranks own no table
    ("webspam_G4", "webspam", 1500, 4, 50, 128, 1 << 15, 128, 4, None),
    ("webspam_G7_rounds", "webspam", 1200, 4, 50, 128, 1 << 15, 128, 7, 50 * 128 * 4 * 100),
    ("url_G3", "url", 4000, 4, 128, 32, 1 << 15, 128, 3, None),
    ("kdd12_G6", "kdd12", 20000, 4, 32, 64, 1 << 20, 128, 6, None),
    ("saturated_G2", "tiny", 1200, 2, 8, 4, 64, 20, 2, None),                        # every bucket over R
]


@pytest.mark.parametrize("name,shape,n,K,L,R,rng,k,G,cand_bytes", GRAPH_CASES, ids=[c[0] for c in GRAPH_CASES])
def test_dist_graph_equals_oracle(name, shape, n, K, L, R, rng, k, G, cand_bytes, monkeypatch):
    if cand_bytes:
        monkeypatch.setenv("FLASH_DIST_CAND_BYTES", str(cand_bytes))
    rp, col = synth.generate(synth.SHAPES[shape].with_(N=n))
    seed = 0xD15E + G
    bounds = fdist.shard_bounds(np.diff(rp), G)
    idxs = _local_group(K, L, R, rng, seed, G)
    try:
        for g, idx in enumerate(idxs):
            assert idx.dist_info() == (g, G, (L * g) // G, (L * (g + 1)) // G)
        ids, cnt = _dist_graph(idxs, _shards(rp, col, bounds), k)
    finally:
        for i in idxs:
            i.close()
    o_ids, o_cnt = oracle.knn_graph(K, L, R, rng, seed, rp, col, k)
    assert np.array_equal(ids, o_ids)
    assert np.array_equal(cnt, o_cnt)


def test_dist_graph_with_empty_shards_and_repeats():
    """Ranks with no rows, then the same handles cleared and reused with other shard sizes
    (receive buffers grow and are re-mapped); every graph equals the oracle."""
    K, L, R, rng, k, G = 4, 16, 32, 1 << 15, 10, 4
    seed = 0xE0E0
    idxs = _local_group(K, L, R, rng, seed, G)
    try:
        for n, bounds in ((300, [0, 0, 150, 150, 300]), (900, None), (1000, [0, 1000, 1000, 1000, 1000])):
            rp, col = synth.generate(synth.SHAPES["tiny"].with_(N=n, seed=n))
            b = bounds or fdist.shard_bounds(np.diff(rp), G)
            for i in idxs:
                i.clear()
            ids, cnt = _dist_graph(idxs, _shards(rp, col, b), k)
            o_ids, o_cnt = oracle.knn_graph(K, L, R, rng, seed, rp, col, k)
            assert np.array_equal(ids, o_ids) and np.array_equal(cnt, o_cnt), n
        assert sum(i.errors() for i in idxs) == 0
    finally:
        for i in idxs:
            i.close()


@pytest.mark.parametrize("contiguous", [True, False])
def test_dist_insert_then_query(contiguous):
    """flash_insert with per-rank id bases (contiguous -> one build pass per window, else one
    per rank segment), then flash_query_topk of every rank's own queries with exclusions;
    then a second insert batch (bottom-R composability across collective calls)."""
    K, L, R, rng, k, G = 4, 24, 16, 4096, 32, 3
    seed = 0x1D5
    rp, col = synth.generate(synth.SHAPES["tiny"].with_(N=1500, seed=9))
    n_a = 1000
    b_a = fdist.shard_bounds(np.diff(rp[: n_a + 1]), G)
    bases = [b_a[g] if contiguous else 5000 * (G - g) + 7 for g in range(G)]
    qrows = np.random.default_rng(3).choice(1500, size=300, replace=False)
    qb = [0, 100, 100, 300]  # rank 1 has no queries
    idxs = _local_group(K, L, R, rng, seed, G)
    streams = [torch.cuda.Stream() for _ in range(G)]
    try:
        sh_a = _shards(rp, col, b_a)
        # second batch: rows n_a..1500 split evenly, ids continue after the first batch's
        b_b = [n_a + (500 * g) // G for g in range(G + 1)]
        q_rp, q_col = synth.csr_from_rows([col[rp[r]:rp[r + 1]] for r in qrows])
        qsh = _shards(q_rp, q_col, qb)

        def id_of(r):  # the id row r was inserted with
            if r < n_a:
                g = np.searchsorted(b_a, r, side="right") - 1
                return bases[g] + (r - b_a[g])
            return 90000 + (r - n_a)

        ids_all = np.array([id_of(r) for r in range(1500)], dtype=np.uint32)
        excl = ids_all[qrows]

        def rank(g):
            def f():
                s = streams[g]
                d_rp, d_col = sh_a[g]
                idxs[g].insert(d_rp, d_col, bases[g], stream=s)
                r0, r1 = b_b[g], b_b[g + 1]
                srp, scol = flash.to_device_csr(rp[r0:r1 + 1] - rp[r0], col[rp[r0]:rp[r1]])
                idxs[g].insert(srp, scol, 90000 + (r0 - n_a), stream=s)
                e = torch.from_numpy(excl[qb[g]:qb[g + 1]].view(np.int32)).cuda()
                ids, cnt = idxs[g].query(qsh[g][0], qsh[g][1], k, exclude=e, stream=s)
                s.synchronize()
                return flash.as_u32(ids), flash.as_u32(cnt)
            return f

        out = _run_ranks([rank(g) for g in range(G)])
        got_ids = np.concatenate([o[0] for o in out])
        got_cnt = np.concatenate([o[1] for o in out])
    finally:
        for i in idxs:
            i.close()
    o_addr = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    T = oracle.build(L, R, rng, seed, o_addr, ids_all)
    o_ids, o_cnt = oracle.query(T, o_addr[qrows], k, exclude=excl)
    assert np.array_equal(got_ids, o_ids)
    assert np.array_equal(got_cnt, o_cnt)


def test_dist_tables_are_the_oracle_windows():
    """Each rank's flash_get_table serves exactly its window's tables (global table index in
    the priorities), equal to the oracle's; other tables are FLASH_ESTATE."""
    K, L, R, rng, G = 4, 10, 8, 512, 3
    seed = 0x7AB
    rp, col = synth.generate(synth.SHAPES["tiny"].with_(N=800))
    bounds = fdist.shard_bounds(np.diff(rp), G)
    idxs = _local_group(K, L, R, rng, seed, G)
    try:
        _dist_graph(idxs, _shards(rp, col, bounds), 5)
        o_addr = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
        T = oracle.build(L, R, rng, seed, o_addr, np.arange(800, dtype=np.uint32))
        for g, idx in enumerate(idxs):
            _, _, t0, t1 = idx.dist_info()
            for t in range(L):
                if t0 <= t < t1:
                    off, ids, arr = idx.table(t)
                    o_off, o_ids, o_arr = T.table(t)
                    assert np.array_equal(off, o_off) and np.array_equal(ids, o_ids) and np.array_equal(arr, o_arr)
                else:
                    with pytest.raises(flash.FlashError):
                        idx.table(t)
    finally:
        for i in idxs:
            i.close()


def test_dist_nccl_world1_graph_and_bootstrap():
    """The NCCL transport at world 1: bootstrap id, communicator, barriers; the graph and
    a query through a flash_create_dist handle equal the oracle."""
    K, L, R, rng, k = 4, 16, 32, 1 << 15, 10
    seed = 0x5EED0001
    uid = flash.flash_get_unique_id()
    assert len(uid) == flash.UNIQUE_ID_BYTES
    h = flash.flash_create_dist(K, L, R, rng, seed, 0, 1, uid)
    idx = flash.FlashIndex(K, L, R, rng, seed, handle=h)
    try:
        assert idx.dist_info() == (0, 1, 0, L)
        rp, col = synth.generate(synth.SHAPES["tiny"].with_(N=600))
        d_rp, d_col = flash.to_device_csr(rp, col)
        ids, cnt = idx.knn_graph(d_rp, d_col, k)
        o_ids, o_cnt = oracle.knn_graph(K, L, R, rng, seed, rp, col, k)
        assert np.array_equal(flash.as_u32(ids), o_ids) and np.array_equal(flash.as_u32(cnt), o_cnt)
        assert idx.errors() == 0
        # a single-GPU step call is refused on a multi-GPU handle
        with pytest.raises(flash.FlashError) as e:
            idx.insert_addrs(torch.zeros((4, L), dtype=torch.int32, device="cuda"))
        assert e.value.status == flash.FLASH_ESTATE
    finally:
        idx.close()


def test_dist_graph_host_buffers():
    """flash_knn_graph_host on local-group ranks (host CSR in, host top-k out)."""
    K, L, R, rng, k, G = 4, 16, 32, 1 << 15, 10, 2
    seed = 0x4057
    rp, col = synth.generate(synth.SHAPES["tiny"].with_(N=500))
    bounds = fdist.shard_bounds(np.diff(rp), G)
    idxs = _local_group(K, L, R, rng, seed, G)
    streams = [torch.cuda.Stream() for _ in range(G)]

    def rank(g):
        def f():
            r0, r1 = bounds[g], bounds[g + 1]
            srp = np.ascontiguousarray(rp[r0:r1 + 1] - rp[r0])
            scol = np.ascontiguousarray(col[rp[r0]:rp[r1]]) if rp[r1] > rp[r0] else np.zeros(1, np.uint32)
            ids = np.empty((r1 - r0, k), np.uint32)
            cnt = np.empty((r1 - r0, k), np.uint32)
            flash.flash_knn_graph_host(idxs[g].h, srp, scol, r1 - r0, k, ids, cnt, streams[g])
            return ids, cnt
        return f

    try:
        out = _run_ranks([rank(g) for g in range(G)])
    finally:
        for i in idxs:
            i.close()
    o_ids, o_cnt = oracle.knn_graph(K, L, R, rng, seed, rp, col, k)
    assert np.array_equal(np.concatenate([o[0] for o in out]), o_ids)
    assert np.array_equal(np.concatenate([o[1] for o in out]), o_cnt)
