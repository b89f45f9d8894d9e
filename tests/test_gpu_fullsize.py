"""Parity at BASELINE.json's full url and kdd12 sizes, in the launch configuration
`bench.py --workload url|kdd12` times (flash_insert of every row, flash_query_topk of 10K
sampled rows with self-exclusion).

url (2.39M rows, 116 nnz, K=4 L=128 R=32, 2^15): the oracle hashes and builds the whole
index on the host, so every address, three whole tables and all 10K top-128 lists are
compared bit-exactly.

kdd12 (149.6M rows, 11 nnz, K=4 L=32 R=64, 2^20): a full oracle build is out of reach, so
the oracle computes sampled rows one by one and the tables / top-k lists are checked by
properties that pin them at any size:
  - addresses of sampled rows equal the oracle's;
  - every bucket keeps min(arrivals, R) ids, ascending; arrivals sum to the non-empty rows;
  - bottom-R membership of sampled rows: a sampled row x in bucket (t, b) is kept iff
    arrivals <= R or (prio(t,b,x), x) is not above the largest kept (prio, id) — prio by
    the oracle (HASHSPEC B), kept ids' own addresses by the oracle;
  - each top-k list: no self, no duplicates, (count desc, id asc), pads last, and every
    reported count c(q, x) <= #{t : addr_t(q) = addr_t(x)} (oracle addresses of q and x);
  - the whole run is deterministic (a second insert + query gives identical bytes).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1709_01190_b200 import flash

pytestmark = pytest.mark.gpu
EMPTY = 0xFFFFFFFF


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "these tests need a B200"
    torch.cuda.set_device(0)
    yield
    torch.cuda.synchronize()


def _query_csr(rp, col, rows):
    lens = rp[rows + 1] - rp[rows]
    q_rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    q_col = np.concatenate([col[rp[r]: rp[r + 1]] for r in rows]).astype(np.uint32)
    return q_rp, q_col


def _run(cfg, rp, col, rows):
    """bench.py's step on the device: insert all rows, query the sampled rows."""
    q_rp, q_col = _query_csr(rp, col, rows)
    d_rp, d_col = flash.to_device_csr(rp, col)
    dq_rp, dq_col = flash.to_device_csr(q_rp, q_col)
    excl = torch.from_numpy(rows.astype(np.uint32).view(np.int32)).cuda()
    idx = flash.FlashIndex(cfg["K"], cfg["L"], cfg["R"], cfg["range"], cfg["seed"])
    idx.insert(d_rp, d_col, 0)
    ids, cnt = idx.query(dq_rp, dq_col, cfg["k"], excl)
    torch.cuda.synchronize()
    return idx, d_rp, d_col, flash.as_u32(ids), flash.as_u32(cnt)


def _oracle_addresses(cfg, rp, col, rows=None, chunk=200_000):
    """Oracle addresses of `rows` (all rows if None), computed in chunks of rows."""
    n = rp.size - 1
    rows = np.arange(n) if rows is None else np.asarray(rows)
    out = np.empty((rows.size, cfg["L"]), np.uint32)
    for i in range(0, rows.size, chunk):
        rr = rows[i: i + chunk]
        if rows.size == n:  # contiguous: slice the CSR
            r0, r1 = int(rr[0]), int(rr[-1]) + 1
            sub_rp = rp[r0: r1 + 1] - rp[r0]
            sub_col = col[rp[r0]: rp[r1]]
        else:
            sub_rp, sub_col = _query_csr(rp, col, rr)
        codes = oracle.doph(cfg["K"], cfg["L"], cfg["seed"], sub_rp, sub_col)
        out[i: i + rr.size] = oracle.addresses(cfg["K"], cfg["L"], cfg["range"], cfg["seed"], codes)
    return out


def _check_topk_structure(ids, cnt, rows, L):
    for q in range(ids.shape[0]):
        valid = ids[q] != EMPTY
        nv = int(valid.sum())
        assert valid[:nv].all() and not valid[nv:].any(), "pads must come last"
        assert (cnt[q, nv:] == 0).all()
        i, c = ids[q, :nv].astype(np.int64), cnt[q, :nv].astype(np.int64)
        assert rows[q] not in set(i.tolist()), "self must be excluded"
        assert len(set(i.tolist())) == nv, "duplicate id"
        assert ((c >= 1) & (c <= L)).all()
        key = -c * (1 << 33) + i  # (count desc, id asc)
        assert (np.diff(key) > 0).all(), "order must be (count desc, id asc)"


URL = dict(K=4, L=128, R=32, range=1 << 15, seed=0x5EED0003, k=128, q=10_000, qseed=13)
KDD = dict(K=4, L=32, R=64, range=1 << 20, seed=0x5EED0004, k=128, q=10_000, qseed=14)


def test_url_full_size_bit_exact():
    cfg = URL
    rp, col = synth.generate("url")
    n = rp.size - 1
    rows = np.sort(np.random.default_rng(cfg["qseed"]).choice(n, size=cfg["q"], replace=False))
    idx, d_rp, d_col, g_ids, g_cnt = _run(cfg, rp, col, rows)
    try:
        g_addrs = flash.as_u32(idx.hash_addrs(d_rp, d_col))
        o_addrs = _oracle_addresses(cfg, rp, col)
        assert np.array_equal(g_addrs, o_addrs)
        T = oracle.build(cfg["L"], cfg["R"], cfg["range"], cfg["seed"], o_addrs, np.arange(n, dtype=np.uint32))
        for t in (0, 63, 127):
            off, ids_t, arr_t = idx.table(t)
            o_off, o_ids_t, o_arr = T.table(t)
            assert np.array_equal(arr_t, o_arr), f"table {t} arrivals"
            assert np.array_equal(off, o_off), f"table {t} offsets"
            assert np.array_equal(ids_t, o_ids_t), f"table {t} kept ids"
        o_ids, o_cnt = oracle.query(T, o_addrs[rows], cfg["k"], exclude=rows.astype(np.uint32))
        assert np.array_equal(g_ids, o_ids)
        assert np.array_equal(g_cnt, o_cnt)
        assert idx.errors() == 0
    finally:
        idx.close()


def _check_index_at_scale(idx, cfg, rp, col, d_rp, d_col, probe_rows, n_members=1500):
    """Sampled-row addresses vs the oracle; every bucket's invariants (on the device);
    bottom-R membership of probe rows (oracle priorities); kept ids' own oracle addresses.
    Returns the probe rows' oracle addresses."""
    L, R, rng = cfg["L"], cfg["R"], cfg["range"]
    g_all = idx.hash_addrs(d_rp, d_col)
    g_s = flash.as_u32(g_all.index_select(0, torch.from_numpy(probe_rows.astype(np.int64)).cuda()))
    del g_all
    o_p = _oracle_addresses(cfg, rp, col, probe_rows)
    assert np.array_equal(g_s, o_p), "addresses of sampled rows"

    lens = np.diff(rp)
    nonempty = int((lens > 0).sum())
    goff_d, kept_d, arr_d = idx.table_arrays()
    arr_d = arr_d.to(torch.int64).view(L, rng)
    sizes_d = (goff_d[1:] - goff_d[:-1]).view(L, rng)
    assert bool((arr_d.sum(dim=1) == nonempty).all()), "arrivals count every non-empty row once per table"
    assert bool((sizes_d == torch.clamp(arr_d, max=R)).all()), "every bucket keeps min(arrivals, R) ids"
    starts = goff_d[:-1][sizes_d.reshape(-1) > 0]
    inner = torch.ones(kept_d.numel(), dtype=torch.bool, device=kept_d.device)
    inner[starts] = False  # the first id of each bucket
    k64 = kept_d.to(torch.int64) & 0xFFFFFFFF
    assert bool((k64[1:] > k64[:-1])[inner[1:]].all()), "ids ascending within each bucket"
    del inner, k64, starts
    goff = goff_d.cpu().numpy()
    arr = arr_d.cpu().numpy()
    sizes = sizes_d.cpu().numpy()

    def bucket_ids(t, b):
        i0, i1 = int(goff[t * rng + b]), int(goff[t * rng + b + 1])
        return flash.as_u32(kept_d[i0:i1])

    seed = cfg["seed"]
    for j, x in enumerate(probe_rows[:n_members]):
        a = o_p[j]
        for t in range(L):
            if a[t] == EMPTY:
                continue
            b = int(a[t])
            bucket = bucket_ids(t, b)
            inside = bool(np.isin(x, bucket))
            if arr[t, b] <= R:
                assert inside, f"row {x} missing from unsaturated bucket ({t},{b})"
                continue
            pk = oracle.prio_batch(seed, np.full(bucket.size, t), np.full(bucket.size, b), bucket)
            worst = max(zip(pk.tolist(), bucket.tolist()))
            px = int(oracle.prio_batch(seed, [t], [b], [x])[0])
            assert inside == ((px, int(x)) <= worst), f"bottom-R membership of row {x} in ({t},{b})"
    for t in (0, L - 1):  # ids kept in a few buckets address those buckets (oracle addresses)
        bs = np.nonzero(sizes[t])[0][:40]
        mem = np.concatenate([bucket_ids(t, int(b)) for b in bs]).astype(np.int64)
        owner = np.concatenate([np.full(sizes[t, b], b) for b in bs])
        oa = _oracle_addresses(cfg, rp, col, mem)
        assert np.array_equal(oa[:, t], owner.astype(np.uint32))
    return o_p


def _check_counts_bounded_by_coaddresses(cfg, rp, col, g_ids, g_cnt, o_q, qs):
    """Every reported count c(q, x) <= #{t : addr_t(q) = addr_t(x)} (oracle addresses)."""
    pairs_q, pairs_x, pairs_c = [], [], []
    for q in qs:
        nv = int((g_ids[q] != EMPTY).sum())
        pairs_q += [q] * nv
        pairs_x += g_ids[q, :nv].tolist()
        pairs_c += g_cnt[q, :nv].tolist()
    if not pairs_x:
        return
    ux, inv = np.unique(np.array(pairs_x, np.int64), return_inverse=True)
    oa = _oracle_addresses(cfg, rp, col, ux)
    co = (oa[inv] == o_q[np.array(pairs_q)]).sum(axis=1)
    assert (np.array(pairs_c) <= co).all(), "a count can never exceed the co-addressed tables"


def test_kdd12_full_size_sampled_and_properties():
    cfg = KDD
    rp, col = synth.generate("kdd12")
    n = rp.size - 1
    rows = np.sort(np.random.default_rng(cfg["qseed"]).choice(n, size=cfg["q"], replace=False))
    idx, d_rp, d_col, g_ids, g_cnt = _run(cfg, rp, col, rows)
    try:
        probe_rows = np.sort(np.random.default_rng(99).choice(n, size=5000, replace=False))
        _check_index_at_scale(idx, cfg, rp, col, d_rp, d_col, probe_rows)
        o_q = _oracle_addresses(cfg, rp, col, rows)
        g_q = flash.as_u32(idx.hash_addrs(*flash.to_device_csr(*_query_csr(rp, col, rows))))
        assert np.array_equal(g_q, o_q), "query addresses"
        _check_topk_structure(g_ids, g_cnt, rows, cfg["L"])
        _check_counts_bounded_by_coaddresses(cfg, rp, col, g_ids, g_cnt, o_q, np.arange(0, rows.size, 25))
        assert idx.errors() == 0
    finally:
        idx.close()
    del d_rp, d_col
    torch.cuda.empty_cache()
    # determinism: a second run gives identical bytes
    idx2, *_rest, ids2, cnt2 = _run(cfg, rp, col, rows)
    idx2.close()
    assert np.array_equal(ids2, g_ids) and np.array_equal(cnt2, g_cnt)


FRIENDSTER = dict(K=4, L=32, R=64, range=1 << 20, seed=0x5EED0005, k=20)


def test_friendster_full_graph_sampled_and_properties():
    """SURVEY §8(f) NEXT #4 at full size (65.6 M rows), in bench.py --workload
    friendster's launch configuration (flash_knn_graph over every row, k = 20): sampled
    addresses, every bucket's invariants, bottom-R membership, and for sampled graph rows
    the top-k structure and count bounds."""
    cfg = FRIENDSTER
    rp, col = synth.generate("friendster")
    n = rp.size - 1
    d_rp, d_col = flash.to_device_csr(rp, col)
    idx = flash.FlashIndex(cfg["K"], cfg["L"], cfg["R"], cfg["range"], cfg["seed"])
    try:
        g_ids, g_cnt = idx.knn_graph(d_rp, d_col, cfg["k"])
        rows = np.sort(np.random.default_rng(7).choice(n, size=3000, replace=False))
        sel = torch.from_numpy(rows.astype(np.int64)).cuda()
        s_ids, s_cnt = flash.as_u32(g_ids.index_select(0, sel)), flash.as_u32(g_cnt.index_select(0, sel))
        del g_ids, g_cnt
        o_q = _check_index_at_scale(idx, cfg, rp, col, d_rp, d_col, rows, n_members=1000)
        _check_topk_structure(s_ids, s_cnt, rows, cfg["L"])
        _check_counts_bounded_by_coaddresses(cfg, rp, col, s_ids, s_cnt, o_q, np.arange(0, rows.size, 10))
        assert idx.errors() == 0
    finally:
        idx.close()
