"""Reservoir sharing across tables (§3.2(4), §3.5; R#23) on the
GPU, bit-exact against the oracle's shared-pool build and query: the pool's arrivals,
offsets and kept ids, top-k ids and counts, the k-NN graph, incremental inserts, and F = 1
reducing to the unshared index."""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1709_01190_b200 import flash

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "these tests need a B200"
    torch.cuda.set_device(0)
    yield
    torch.cuda.synchronize()


def _shape(name, n, **kw):
    return synth.generate(synth.SHAPES[name].with_(N=n, **kw))


def _check_pool(idx, T):
    goff, ids, arr = idx.table_arrays()
    goff = goff.cpu().numpy()
    assert goff.size == T.P + 1
    assert np.array_equal(flash.as_u32(arr), T.arrivals), "arrivals"
    assert np.array_equal(goff - goff[0], T.off.astype(np.int64)), "offsets"
    assert np.array_equal(flash.as_u32(ids)[: int(goff[-1])], T.kept), "kept ids"


CASES = [
    ("tiny_F05", lambda: synth.generate("tiny"), 4, 16, 32, 1 << 15, 0.5, 10),
    ("tiny_F001", lambda: synth.generate("tiny"), 4, 16, 32, 1 << 15, 0.01, 10),
    ("webspam_F02", lambda: _shape("webspam", 2000), 4, 50, 128, 1 << 12, 0.2, 128),
    ("webspam_F005", lambda: _shape("webspam", 2000), 4, 50, 128, 1 << 12, 0.05, 64),
    ("url_F01", lambda: _shape("url", 6000), 4, 128, 32, 1 << 12, 0.1, 128),
    ("kdd12_F02", lambda: _shape("kdd12", 20000), 4, 32, 64, 1 << 12, 0.2, 32),
]


@pytest.mark.parametrize("name,make,K,L,R,rng,F,k", CASES, ids=[c[0] for c in CASES])
def test_pool_graph_tables_and_queries_bit_exact(name, make, K, L, R, rng, F, k):
    rp, col = make()
    n = rp.size - 1
    seed = 0x5EED0002
    P = oracle.pool_size(F, L, rng)
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    T = oracle.build_pool(L, R, rng, P, seed, addrs, np.arange(n, dtype=np.uint32))
    o_ids, o_cnt = oracle.query_pool(T, seed, addrs, k, exclude=np.arange(n, dtype=np.uint32))
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed, F=F) as idx:
        assert idx.pool == P
        g_ids, g_cnt = idx.knn_graph(d_rp, d_col, k)
        assert np.array_equal(flash.as_u32(g_ids), o_ids)
        assert np.array_equal(flash.as_u32(g_cnt), o_cnt)
        _check_pool(idx, T)
        # external queries (CSR path) with another exclusion
        excl = np.random.default_rng(5).integers(0, n, size=n).astype(np.uint32)
        q_ids, q_cnt = oracle.query_pool(T, seed, addrs, k, exclude=excl)
        g2_ids, g2_cnt = idx.query(d_rp, d_col, k, torch.from_numpy(excl.view(np.int32)).cuda())
        assert np.array_equal(flash.as_u32(g2_ids), q_ids)
        assert np.array_equal(flash.as_u32(g2_cnt), q_cnt)
        assert idx.errors() == 0


def test_pool_incremental_inserts_equal_one_build():
    rp, col = _shape("url", 5000)
    n = rp.size - 1
    K, L, R, rng, seed, F = 3, 20, 16, 1 << 9, 99, 0.3
    P = oracle.pool_size(F, L, rng)
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    T = oracle.build_pool(L, R, rng, P, seed, addrs, np.arange(n, dtype=np.uint32) + 1000)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed, F=F) as idx:
        for a, b in [(0, 1700), (1700, 1701), (1701, 5000)]:
            flash.flash_insert(idx.h, d_rp[a:b + 1].contiguous(), d_col, b - a, 1000 + a)
        _check_pool(idx, T)


def test_full_pool_is_the_unshared_index_and_errors():
    rp, col = _shape("webspam", 1500)
    K, L, R, rng, seed, k = 4, 50, 128, 1 << 12, 7, 64
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as a:
        ids_a, cnt_a = a.knn_graph(d_rp, d_col, k)
    h = flash.flash_create_pool(K, L, R, rng, L * rng, seed)  # pool = L*range: no sharing
    try:
        n = rp.size - 1
        ids_b = torch.empty((n, k), dtype=torch.int32, device="cuda")
        cnt_b = torch.empty_like(ids_b)
        flash.flash_knn_graph(h, d_rp, d_col, n, k, ids_b, cnt_b)
        assert torch.equal(ids_a, ids_b) and torch.equal(cnt_a, cnt_b)
    finally:
        flash.flash_destroy(h)
    with pytest.raises(flash.FlashError) as e:
        flash.flash_create_pool(K, L, R, rng, L * rng + 1, seed)
    assert e.value.status == flash.FLASH_EINVAL
    with flash.FlashIndex(K, L, R, rng, seed, F=0.25) as s:
        s.insert(d_rp, d_col)
        with pytest.raises(flash.FlashError) as e:
            s.table(0)
        assert e.value.status == flash.FLASH_ESTATE
        with pytest.raises(flash.FlashError) as e:
            s.insert_addrs_window(s.hash_addrs(d_rp, d_col), 0, 0, 10)
        assert e.value.status == flash.FLASH_EINVAL


@pytest.mark.parametrize("F", [1.0, 0.2])
def test_save_load_round_trip_then_further_inserts(tmp_path, F):
    """SPEC S:247 / S:478: load(save(index)) is bit-exact — same tables, same query answers —
    and inserting more rows into the loaded index equals one build over all rows."""
    rp, col = _shape("webspam", 3000)
    n = rp.size - 1
    K, L, R, rng, seed, k = 4, 50, 16, 1 << 10, 11, 32
    d_rp, d_col = flash.to_device_csr(rp, col)
    h = 1800
    with flash.FlashIndex(K, L, R, rng, seed, F=F) as a:
        flash.flash_insert(a.h, d_rp[: h + 1].contiguous(), d_col, h, 0)
        a.save(str(tmp_path / "idx.npz"))
        want = a.query(d_rp, d_col, k)
        g0, i0, r0 = a.table_arrays()
    # the anchor: the oracle's index over the first h rows answers the same
    P = oracle.pool_size(F, L, rng)
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    T = oracle.build_pool(L, R, rng, P, seed, addrs[:h], np.arange(h, dtype=np.uint32))
    o_ids, o_cnt = oracle.query_pool(T, seed, addrs, k)
    with flash.FlashIndex.load(str(tmp_path / "idx.npz")) as b:
        g1, i1, r1 = b.table_arrays()
        assert torch.equal(g0 - g0[0], g1 - g1[0]) and torch.equal(i0, i1) and torch.equal(r0, r1)
        _check_pool(b, T)
        got = b.query(d_rp, d_col, k)
        assert torch.equal(want[0], got[0]) and torch.equal(want[1], got[1])
        assert np.array_equal(flash.as_u32(got[0]), o_ids) and np.array_equal(flash.as_u32(got[1]), o_cnt)
        flash.flash_insert(b.h, d_rp[h:].contiguous(), d_col, n - h, h)
        with flash.FlashIndex(K, L, R, rng, seed, F=F) as c:
            c.insert(d_rp, d_col, 0)
            g2, i2, r2 = c.table_arrays()
            g3, i3, r3 = b.table_arrays()
            assert torch.equal(g2 - g2[0], g3 - g3[0]) and torch.equal(i2, i3) and torch.equal(r2, r3)
