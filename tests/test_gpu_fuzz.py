"""Randomised parity: many small seeded configurations (K, L, R, range, k, reservoir sharing,
row shapes, build schedule) drawn at random, each compared bit-exactly with the oracle —
tables, external queries with exclusions, and the k-NN graph.  Complements the hand-picked
cases in test_gpu_parity.py with combinations nobody chose."""
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


def _config(i):
    g = np.random.default_rng(1000 + i)
    shape = ["tiny", "webspam", "url", "kdd12"][int(g.integers(0, 4))]
    n = int(g.integers(20, 2500 if shape != "webspam" else 600))
    K = int(g.integers(1, 7))
    L = int(g.integers(1, min(64, 8192 // K) + 1))
    R = int(g.choice([1, 2, 5, 16, 32, 64, 128, 300]))
    while L * R > 32768:
        R //= 2
    rng = int(g.choice([1, 7, 64, 1000, 1 << 10, 1 << 15]))
    k = int(g.choice([1, 3, 10, 64, 128, 300]))
    F = 1.0 if g.random() < 0.6 else float(g.choice([0.5, 0.2, 0.05]))
    sched = str(g.choice(["default", "rowmajor", "tablemajor"]))
    seed = int(g.integers(0, 2**63))
    return shape, n, K, L, R, rng, k, F, sched, seed


@pytest.mark.parametrize("i", range(200))
def test_random_config_bit_exact(monkeypatch, i):
    shape, n, K, L, R, rng, k, F, sched, seed = _config(i)
    if sched == "rowmajor":
        monkeypatch.setenv("FLASH_BUILD_TM", "0")
        monkeypatch.setenv("FLASH_BUILD_SMEM", "0")
    elif sched == "tablemajor":
        monkeypatch.setenv("FLASH_BUILD_TM", "1")
    rp, col = synth.generate(synth.SHAPES[shape].with_(N=n, seed=7 + i))
    rows = [col[rp[j]:rp[j + 1]] for j in range(n)]
    if i % 5 == 0:  # a sprinkle of edge rows (empty, single index, duplicates)
        rows += synth.edge_case_rows()
    rp, col = synth.csr_from_rows(rows)
    n = rp.size - 1
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    ids = np.arange(n, dtype=np.uint32)
    excl = np.random.default_rng(i).integers(0, n + 3, size=n).astype(np.uint32)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed, F=F) as idx:
        if F < 1.0:
            T = oracle.build_pool(L, R, rng, idx.pool, seed, addrs, ids)
            o_q = oracle.query_pool(T, seed, addrs, k, exclude=excl)
            o_g = oracle.query_pool(T, seed, addrs, k, exclude=ids)
        else:
            T = oracle.build(L, R, rng, seed, addrs, ids)
            o_q = oracle.query(T, addrs, k, exclude=excl)
            o_g = oracle.query(T, addrs, k, exclude=ids)
        g_ids, g_cnt = idx.knn_graph(d_rp, d_col, k)
        assert np.array_equal(flash.as_u32(g_ids), o_g[0]), f"graph ids, config {_config(i)}"
        assert np.array_equal(flash.as_u32(g_cnt), o_g[1]), f"graph counts, config {_config(i)}"
        q_ids, q_cnt = idx.query(d_rp, d_col, k, torch.from_numpy(excl.view(np.int32)).cuda())
        assert np.array_equal(flash.as_u32(q_ids), o_q[0]), f"query ids, config {_config(i)}"
        assert np.array_equal(flash.as_u32(q_cnt), o_q[1]), f"query counts, config {_config(i)}"
        if F == 1.0:
            for t in sorted({0, L - 1, L // 2}):
                off, kept, arr = idx.table(t)
                o_off, o_kept, o_arr = T.table(t)
                assert np.array_equal(arr, o_arr) and np.array_equal(off, o_off) and np.array_equal(kept, o_kept)
        assert idx.errors() == 0
