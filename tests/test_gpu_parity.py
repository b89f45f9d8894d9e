"""Bit-exact parity of the CUDA path (through the C ABI) with the CPU oracle.

Integer work end to end, so the bar is bit-exactness (north_star): codes, addresses,
per-bucket arrivals / offsets / kept ids, top-k ids and counts.  Inputs are seeded
synthetic CSR (synth/) at sizes the oracle finishes in seconds, spanning many tiles
and ragged tails, plus the degenerate cases of SURVEY §4's edge matrix.
"""
import os

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


def shape_slice(name, n, **kw):
    s = synth.SHAPES[name].with_(N=n, **kw)
    return synth.generate(s)


def edge_csr():
    return synth.csr_from_rows(synth.edge_case_rows())


def skew_csr(n=3000, seed=5):
    """Half the rows identical (SURVEY §4 / S:219 heavy bucket), rest tiny-shaped."""
    rp, col = synth.generate(synth.SHAPES["tiny"].with_(N=n, seed=seed))
    rows = [col[rp[i]:rp[i + 1]] for i in range(n)]
    for i in range(0, n, 2):
        rows[i] = rows[0]
    return synth.csr_from_rows(rows)


HASH_CASES = [
    ("tiny", lambda: synth.generate("tiny"), 4, 16, 1 << 15),
    ("edge", edge_csr, 4, 16, 1000),
    ("edge_KL1", edge_csr, 1, 1, 1 << 15),
    ("edge_range1", edge_csr, 2, 8, 1),
    ("webspam_slice", lambda: shape_slice("webspam", 600), 4, 50, 1 << 15),
    ("webspam_B768", lambda: shape_slice("webspam", 200), 6, 128, 1 << 15),
    ("url_slice", lambda: shape_slice("url", 4000), 4, 128, 1 << 15),
    ("kdd12_slice", lambda: shape_slice("kdd12", 20000), 4, 32, 1 << 20),
    ("wide_K", lambda: shape_slice("url", 500), 64, 2, 12345),
    # the inverted-chain kernel (k_doph_mid: 256 < K*L <= 2047, rows with nnz <= K*L/2)
    ("kdd12_B512", lambda: shape_slice("kdd12", 6000), 4, 128, 1 << 20),
    ("url_B1024", lambda: shape_slice("url", 1500), 8, 128, 1 << 15),
    ("edge_B512", edge_csr, 4, 128, 1000),
    ("url_B2047", lambda: shape_slice("url", 600), 23, 89, 1 << 15),
    ("tiny_B260", lambda: synth.generate("tiny"), 2, 130, 1 << 15),
]


@pytest.mark.parametrize("name,make,K,L,rng", HASH_CASES, ids=[c[0] for c in HASH_CASES])
def test_hash_codes_and_addresses_bit_exact(name, make, K, L, rng):
    rp, col = make()
    seed = 0x5EED0000 + K * 131 + L
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, 8, rng, seed) as idx:
        codes, addrs = idx.hash(d_rp, d_col)
        o_codes = oracle.doph(K, L, seed, rp, col)
        o_addrs = oracle.addresses(K, L, rng, seed, o_codes)
        assert np.array_equal(flash.as_u32(codes), o_codes)
        assert np.array_equal(flash.as_u32(addrs), o_addrs)
        # addresses alone (the insert/graph kernel variant)
        _, a2 = idx.hash(d_rp, d_col, codes=False)
        assert np.array_equal(flash.as_u32(a2), o_addrs)


@pytest.mark.parametrize("cap", ["3", "100000"])
def test_hash_long_row_list_and_its_overflow(monkeypatch, cap):
    """K*L <= 256: k_doph_sparse lists the rows over 32 nonzeros for k_doph; with a list cap
    below their number (3) k_doph falls back to scanning every row's extent."""
    monkeypatch.setenv("FLASH_DOPH_LONGCAP", cap)
    rp, col = shape_slice("url", 3000)  # ~116 nnz per row, a few rows <= 32
    rows = [col[rp[i]:rp[i + 1]] for i in range(rp.size - 1)]
    rows = [r[:20] if i % 3 else r for i, r in enumerate(rows)]  # two thirds short
    rp, col = synth.csr_from_rows(rows)
    K, L, seed = 4, 32, 0x5EED0104
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, 8, 1 << 15, seed) as idx:
        codes, addrs = idx.hash(d_rp, d_col)
        o_codes = oracle.doph(K, L, seed, rp, col)
        assert np.array_equal(flash.as_u32(codes), o_codes)
        assert np.array_equal(flash.as_u32(addrs), oracle.addresses(K, L, 1 << 15, seed, o_codes))


@pytest.mark.parametrize("T1,mid_le", [("1", None), ("8", None), ("31", None), (None, "-1"), (None, "40")])
def test_hash_inverted_chain_kernel_settings(monkeypatch, T1, mid_le):
    """k_doph_mid under other inverted-chain depths T1 (T1 = 1 sends most empty bins to the
    parallel probes and the circular scan) and row-length cuts (-1 = every row probes in
    k_doph; 40 = a mix of both kernels), bit-exact vs the oracle."""
    if T1 is not None:
        monkeypatch.setenv("FLASH_DOPH_T1", T1)
    if mid_le is not None:
        monkeypatch.setenv("FLASH_DOPH_MID_LE", mid_le)
    for name, K, L, n in (("url", 4, 128, 1200), ("kdd12", 4, 128, 3000), ("tiny", 3, 100, 800)):
        rp, col = shape_slice(name, n)
        seed = 0x5EED0000 + K * 131 + L
        d_rp, d_col = flash.to_device_csr(rp, col)
        with flash.FlashIndex(K, L, 8, 1 << 15, seed) as idx:
            codes, addrs = idx.hash(d_rp, d_col)
            o_codes = oracle.doph(K, L, seed, rp, col)
            assert np.array_equal(flash.as_u32(codes), o_codes), name
            assert np.array_equal(flash.as_u32(addrs), oracle.addresses(K, L, 1 << 15, seed, o_codes)), name


def test_hash_row_slice_with_absolute_offsets_and_unaligned_col_idx():
    rp, col = shape_slice("webspam", 300)
    K, L, rng, seed = 4, 50, 1 << 15, 77
    o = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, 8, rng, seed) as idx:
        # rows 100..199 through a row_ptr slice (absolute offsets into the same col_idx)
        sub = d_rp[100:201].contiguous()
        a = torch.empty((100, L), dtype=torch.int32, device="cuda")
        flash.flash_hash(idx.h, sub, d_col, 100, None, a)
        assert np.array_equal(flash.as_u32(a), o[100:200])
        # col_idx starting 1 element past a 16-B boundary
        shifted = torch.empty(d_col.numel() + 1, dtype=torch.int32, device="cuda")
        shifted[1:] = d_col
        view = shifted[1:]
        a = torch.empty((300, L), dtype=torch.int32, device="cuda")
        flash.flash_hash(idx.h, d_rp, view, 300, None, a)
        assert np.array_equal(flash.as_u32(a), o)


def _check_tables(idx, T):
    for t in range(idx.L):
        off, ids, arr = idx.table(t)
        o_off, o_ids, o_arr = T.table(t)
        assert np.array_equal(arr, o_arr), f"arrivals t={t}"
        assert np.array_equal(off, o_off), f"off t={t}"
        assert np.array_equal(ids, o_ids), f"ids t={t}"


BUILD_CASES = [
    ("tiny", lambda: synth.generate("tiny"), 4, 16, 32, 1 << 15),
    ("edge", edge_csr, 4, 16, 3, 1000),
    ("skew_R8_range64", skew_csr, 2, 6, 8, 64),
    ("skew_R1", skew_csr, 2, 6, 1, 64),
    ("range1_R128", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=3000)), 1, 3, 128, 1),
    ("range1_R2000_big", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=3000)), 1, 2, 2000, 1),
    ("range1_R4096_m_le_R", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=3000)), 1, 2, 4096, 1),
    ("range1_R4096_m5000_overflow", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=5000)), 1, 2, 4096, 1),
    ("range2_R100_m2500_cta", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=5000)), 1, 2, 100, 2),
    ("webspam_slice", lambda: shape_slice("webspam", 1500), 4, 50, 128, 1 << 10),
    ("url_slice", lambda: shape_slice("url", 6000), 4, 128, 32, 1 << 12),
    # 33..256 members per bucket: the register-resident select (k_select_mid)
    ("mid_R16", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=20000, seed=9)), 2, 4, 16, 256),
    ("mid_R64", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=20000, seed=9)), 2, 4, 64, 256),
    ("mid_R200_all_kept", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=20000, seed=9)), 2, 4, 200, 256),
]


# (FLASH_BUILD_TM, FLASH_BUILD_SMEM, FLASH_BUILD_GROUPED): "tablemajor" takes the grouped
# table-major passes on fresh builds, "tm_plain" the plain table-major scatter
BUILD_SCHEDULES = {"rowmajor": ("0", "0", "1"), "tablemajor": ("1", "1", "1"), "smem": ("0", "1", "1"),
                   "tm_plain": ("1", "1", "0")}


@pytest.mark.parametrize("sched", list(BUILD_SCHEDULES))
@pytest.mark.parametrize("name,make,K,L,R,rng", BUILD_CASES, ids=[c[0] for c in BUILD_CASES])
def test_tables_bit_exact(monkeypatch, name, make, K, L, R, rng, sched):
    """Every build schedule: row-major global-atomic passes, the table-major passes
    (transposed addresses, table-ordered grid: large tables), and the shared-memory
    passes (a CTA per table slice: tables whose counters fit shared memory)."""
    monkeypatch.setenv("FLASH_BUILD_TM", BUILD_SCHEDULES[sched][0])
    monkeypatch.setenv("FLASH_BUILD_SMEM", BUILD_SCHEDULES[sched][1])
    monkeypatch.setenv("FLASH_BUILD_GROUPED", BUILD_SCHEDULES[sched][2])
    rp, col = make()
    n = rp.size - 1
    seed = 0xB0 + R
    d_rp, d_col = flash.to_device_csr(rp, col)
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    T = oracle.build(L, R, rng, seed, addrs, np.arange(n, dtype=np.uint32))
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        idx.insert(d_rp, d_col, 0)
        _check_tables(idx, T)
        assert idx.errors() == 0


@pytest.mark.parametrize("n,K,L,R,rng", [(300, 1, 300, 8, 64),    # more tables than SMs: one CTA per table
                                         (3, 1, 160, 4, 16),      # W*n = 480 units over 160 CTAs
                                         (1, 2, 160, 4, 16),      # one unit (row) per CTA
                                         (5000, 4, 3, 16, 64),    # 148 CTAs, segments span tables
                                         (2000, 2, 8, 64, 4)])    # > 512-member buckets: side stream
def test_smem_build_cta_mappings(monkeypatch, n, K, L, R, rng):
    """The shared-memory passes cut the W*n (table, row) units into equal CTA ranges whose
    segments may span tables; tables must not depend on where the cuts fall."""
    monkeypatch.setenv("FLASH_BUILD_TM", "0")
    monkeypatch.setenv("FLASH_BUILD_SMEM", "1")
    rp, col = synth.generate(synth.SHAPES["tiny"].with_(N=n, seed=n + L))
    seed = 0xC7A + L
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    T = oracle.build(L, R, rng, seed, addrs, np.arange(n, dtype=np.uint32))
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        idx.insert(d_rp, d_col, 0)
        _check_tables(idx, T)
        idx.insert(d_rp, d_col, n)  # a second batch: old kept ids first in every pool
        T2 = oracle.build(L, R, rng, seed, np.concatenate([addrs, addrs]), np.arange(2 * n, dtype=np.uint32))
        _check_tables(idx, T2)
        assert idx.errors() == 0


@pytest.mark.parametrize("mode", ["1", "2"])
def test_tables_bit_exact_on_the_exact_cta_path(monkeypatch, mode):
    """FLASH_DEBUG_FORCE_BIG=1 routes every bucket with > 32 members through the CTA
    kernel; =2 also skips its threshold filter so the exact radix select (normally only
    reached by rare threshold misses) decides every bucket."""
    monkeypatch.setenv("FLASH_DEBUG_FORCE_BIG", mode)
    for make, K, L, R, rng in [(skew_csr, 2, 6, 8, 64),
                               (lambda: shape_slice("webspam", 1500), 4, 50, 128, 256),
                               (lambda: synth.generate(synth.SHAPES["tiny"].with_(N=2000)), 1, 2, 300, 1)]:
        rp, col = make()
        n = rp.size - 1
        seed = 4242
        addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
        T = oracle.build(L, R, rng, seed, addrs, np.arange(n, dtype=np.uint32))
        d_rp, d_col = flash.to_device_csr(rp, col)
        with flash.FlashIndex(K, L, R, rng, seed) as idx:
            idx.insert(d_rp, d_col, 0)
            _check_tables(idx, T)


@pytest.mark.parametrize("sched", list(BUILD_SCHEDULES))
def test_incremental_inserts_equal_one_build(monkeypatch, sched):
    monkeypatch.setenv("FLASH_BUILD_TM", BUILD_SCHEDULES[sched][0])
    monkeypatch.setenv("FLASH_BUILD_SMEM", BUILD_SCHEDULES[sched][1])
    monkeypatch.setenv("FLASH_BUILD_GROUPED", BUILD_SCHEDULES[sched][2])
    rp, col = shape_slice("url", 5000)
    n = rp.size - 1
    K, L, R, rng, seed = 3, 20, 16, 1 << 9, 99
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    ids = np.arange(n, dtype=np.uint32) + 1000
    T = oracle.build(L, R, rng, seed, addrs, ids)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        for a, b in [(0, 1700), (1700, 1701), (1701, 5000)]:
            flash.flash_insert(idx.h, d_rp[a:b + 1].contiguous(), d_col, b - a, 1000 + a)
        _check_tables(idx, T)
    # precomputed-address insert in a different batch split, rows out of order
    d_addrs = torch.from_numpy(addrs.view(np.int32)).cuda()
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        idx.insert_addrs(d_addrs[3000:].contiguous(), 1000 + 3000)
        idx.insert_addrs(d_addrs[:3000].contiguous(), 1000)
        _check_tables(idx, T)


QUERY_CASES = [
    ("tiny_k10", lambda: synth.generate("tiny"), 4, 16, 32, 1 << 15, 10),
    ("tiny_k1", lambda: synth.generate("tiny"), 4, 16, 32, 1 << 15, 1),
    ("skew_k7", skew_csr, 2, 6, 8, 64, 7),
    ("skew_small_range_k1024", skew_csr, 1, 8, 64, 16, 1024),
    ("webspam_k128", lambda: shape_slice("webspam", 2500), 4, 50, 128, 1 << 15, 128),
    ("webspam_dense_buckets_k128", lambda: shape_slice("webspam", 2500), 4, 50, 128, 1 << 7, 128),
    ("url_k128", lambda: shape_slice("url", 6000), 4, 128, 32, 1 << 15, 128),
    ("edge_k5", edge_csr, 4, 16, 4, 1000, 5),
    # L*R = 10240 > 8192 with full buckets: M = 10240 candidates per query, the CTA sort class
    ("full_buckets_LR10240_k100", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=8000, seed=3)), 1, 40, 256, 16, 100),
    ("LR32768_k64", lambda: shape_slice("webspam", 1500), 4, 128, 256, 1 << 12, 64),
    ("LR16384_k1024", lambda: shape_slice("webspam", 1500), 4, 64, 256, 1 << 10, 1024),
    # L = 4096: the warp sort classes' per-warp slices (L*8 B of segment bases) do not fit, so
    # every class runs on the CTA sort kernel (classes that cannot launch)
    ("L4096_R8_k32", lambda: synth.generate(synth.SHAPES["tiny"].with_(N=500, seed=4)), 2, 4096, 8, 64, 32),
]


# query kernels: "default" (queries with more than 768 candidates on the occupancy-bitmap
# kernel when the ids fit its bitmap, the rest on the size-class sort kernels), "mark" /
# "split" = every query / those above 100 candidates on the bitmap kernel, "sort" =
# FLASH_QUERY_MARK=0 (sort kernels only), "fallback0" / "fallback3" = the bitmap kernel with
# at most 0 / 3 distinct repeated ids per query, so every / some queries go to its CTA-sort
# fallback list
QUERY_KERNELS = {"default": {}, "mark": {"FLASH_QUERY_MARK_MIN": "0"}, "split": {"FLASH_QUERY_MARK_MIN": "100"},
                 "sort": {"FLASH_QUERY_MARK": "0"},
                 "fallback0": {"FLASH_QUERY_MARK_MIN": "0", "FLASH_QUERY_MARK_REPMAX": "0"},
                 "fallback3": {"FLASH_QUERY_MARK_MIN": "0", "FLASH_QUERY_MARK_REPMAX": "3"}}


def _set_kernel(monkeypatch, kern):
    for key, val in QUERY_KERNELS[kern].items():
        monkeypatch.setenv(key, val)


@pytest.mark.parametrize("kern", list(QUERY_KERNELS))
@pytest.mark.parametrize("name,make,K,L,R,rng,k", QUERY_CASES, ids=[c[0] for c in QUERY_CASES])
def test_query_topk_bit_exact(monkeypatch, name, make, K, L, R, rng, k, kern):
    _set_kernel(monkeypatch, kern)
    rp, col = make()
    n = rp.size - 1
    seed = 0xC0DE + k
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    ids = np.arange(n, dtype=np.uint32)
    T = oracle.build(L, R, rng, seed, addrs, ids)
    g = np.random.default_rng(k)
    excl = g.integers(0, n + 5, size=n).astype(np.uint32)
    o_ids, o_cnt = oracle.query(T, addrs, k, exclude=excl)
    o_ids2, o_cnt2 = oracle.query(T, addrs, k)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        idx.insert(d_rp, d_col, 0)
        d_addrs = torch.from_numpy(addrs.view(np.int32)).cuda()
        d_ex = torch.from_numpy(excl.view(np.int32)).cuda()
        g_ids, g_cnt = idx.query_addrs(d_addrs, k, d_ex)
        assert np.array_equal(flash.as_u32(g_ids), o_ids)
        assert np.array_equal(flash.as_u32(g_cnt), o_cnt)
        g_ids, g_cnt = idx.query(d_rp, d_col, k)  # CSR query path, no exclusion
        assert np.array_equal(flash.as_u32(g_ids), o_ids2)
        assert np.array_equal(flash.as_u32(g_cnt), o_cnt2)


@pytest.mark.parametrize("name,make,K,L,R,rng,k", QUERY_CASES[:8], ids=[c[0] for c in QUERY_CASES[:8]])
def test_query_csort_kernel_every_class(monkeypatch, name, make, K, L, R, rng, k):
    """FLASH_QUERY_CSORT=1 routes every size class through the CTA sort kernel (the class of
    L*R > 8192 and the fallback of classes that do not fit): bit-exact on the same cases."""
    monkeypatch.setenv("FLASH_QUERY_CSORT", "1")
    test_query_topk_bit_exact(monkeypatch, name, make, K, L, R, rng, k, "sort")


@pytest.mark.parametrize("few", ["0", "1000000000"])
def test_query_4096_class_both_kernels(monkeypatch, few):
    """Queries with 3072 < M <= 4096 candidates run the warp-per-query sort class when there
    are many queries and the CTA-per-query kernel when there are few (FLASH_QUERY_FEW sets
    the cut; 0 forces the sort class, a huge value the CTA kernel): both bit-exact."""
    monkeypatch.setenv("FLASH_QUERY_FEW", few)
    monkeypatch.setenv("FLASH_QUERY_MARK", "0")
    rp, col = shape_slice("url", 6000)
    K, L, R, rng, k = 4, 128, 32, 1 << 6, 128  # 64 buckets: all saturate, M = L*R = 4096
    n = rp.size - 1
    seed = 0x4096
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    ids = np.arange(n, dtype=np.uint32)
    T = oracle.build(L, R, rng, seed, addrs, ids)
    o_ids, o_cnt = oracle.query(T, addrs, k, exclude=ids)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        g_ids, g_cnt = idx.knn_graph(d_rp, d_col, k)
        assert np.array_equal(flash.as_u32(g_ids), o_ids)
        assert np.array_equal(flash.as_u32(g_cnt), o_cnt)


GRAPH_CASES = [
    ("tiny", lambda: synth.generate("tiny"), 4, 16, 32, 1 << 15, 10),
    ("edge", edge_csr, 4, 16, 32, 1 << 15, 10),
    ("webspam_slice", lambda: shape_slice("webspam", 4000), 4, 50, 128, 1 << 15, 128),
    ("url_slice", lambda: shape_slice("url", 8000), 4, 128, 32, 1 << 15, 128),
    ("kdd12_slice", lambda: shape_slice("kdd12", 30000), 4, 32, 64, 1 << 20, 128),
]


@pytest.mark.parametrize("kern", list(QUERY_KERNELS))
@pytest.mark.parametrize("name,make,K,L,R,rng,k", GRAPH_CASES, ids=[c[0] for c in GRAPH_CASES])
def test_knn_graph_bit_exact(monkeypatch, name, make, K, L, R, rng, k, kern):
    _set_kernel(monkeypatch, kern)
    rp, col = make()
    seed = 0x5EED0002
    o_ids, o_cnt = oracle.knn_graph(K, L, R, rng, seed, rp, col, k)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        g_ids, g_cnt = idx.knn_graph(d_rp, d_col, k)
        assert np.array_equal(flash.as_u32(g_ids), o_ids)
        assert np.array_equal(flash.as_u32(g_cnt), o_cnt)
    # the host-buffer entry point (pageable and pinned inputs) gives the same graph
    n = rp.size - 1
    for pinned in (False, True):
        hrp = torch.from_numpy(rp.copy())
        hcol = torch.from_numpy(col.view(np.int32).copy())
        out_i = torch.empty((n, k), dtype=torch.int32)
        out_c = torch.empty((n, k), dtype=torch.int32)
        if pinned:
            hrp, hcol, out_i, out_c = (t.pin_memory() for t in (hrp, hcol, out_i, out_c))
        with flash.FlashIndex(K, L, R, rng, seed) as idx:
            flash.flash_knn_graph_host(idx.h, hrp, hcol, n, k, out_i, out_c)
        assert np.array_equal(out_i.numpy().view(np.uint32), o_ids)
        assert np.array_equal(out_c.numpy().view(np.uint32), o_cnt)


@pytest.mark.parametrize("grouped", ["1", "0"])
def test_table_major_build_over_several_row_chunks(monkeypatch, grouped):
    """2.3 M rows into 2^20-bucket tables: the grouped table-major passes span two 2^21-row
    chunks and 512-bucket groups (the kdd12 geometry at a small L), the plain scatter as the
    control; tables bit-exact against the oracle."""
    monkeypatch.setenv("FLASH_BUILD_TM", "1")
    monkeypatch.setenv("FLASH_BUILD_GROUPED", grouped)
    rp, col = shape_slice("kdd12", 2_300_000)
    n = rp.size - 1
    K, L, R, rng, seed = 4, 3, 8, 1 << 20, 0x5EED0004
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    T = oracle.build(L, R, rng, seed, addrs, np.arange(n, dtype=np.uint32) + 7)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        idx.insert(d_rp, d_col, 7)
        _check_tables(idx, T)


@pytest.mark.parametrize("rng,R,cap", [(1 << 14, 64, None), (1 << 14, 64, "3000"), (1 << 13, 200, None),
                                       (1 << 14, 16, None), (1 << 14, 64, "0")])
def test_grouped_build_fused_select(monkeypatch, rng, R, cap):
    """The grouped table-major passes with the fused placement + select (k_gplace_sel):
    ~140 / ~280 members per bucket (the register select in shared memory; buckets over 256
    listed for the warp select), heavy buckets from repeated rows (> 512: the CTA path), a
    small stage (FLASH_BUILD_GSEL_CAP: sub-ranges that overflow go through the pool and the
    select kernels), and FLASH_BUILD_GSEL=0 as the control; tables bit-exact vs the oracle."""
    monkeypatch.setenv("FLASH_BUILD_TM", "1")
    monkeypatch.setenv("FLASH_BUILD_SMEM", "0")
    monkeypatch.setenv("FLASH_BUILD_GROUPED", "1")
    monkeypatch.setenv("FLASH_BUILD_GSEL", "0" if cap == "0" else "1")
    if cap not in (None, "0"):
        monkeypatch.setenv("FLASH_BUILD_GSEL_CAP", cap)
    rp, col = shape_slice("kdd12", 2_300_000)
    rows = [col[rp[i]:rp[i + 1]] for i in range(0, 3000)]
    heavy = synth.csr_from_rows([rows[5]] * 1500 + rows)  # one row 1,500 times: a bucket per table
    rp = np.concatenate([heavy[0], heavy[0][-1] + rp[1:]])
    col = np.concatenate([heavy[1], col])
    n = rp.size - 1
    K, L, seed = 4, 3, 0x5EED0004
    addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    T = oracle.build(L, R, rng, seed, addrs, np.arange(n, dtype=np.uint32))
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        idx.insert(d_rp, d_col, 0)
        _check_tables(idx, T)
        assert idx.errors() == 0


def test_knn_graph_ids_beyond_the_bitmap_kernel():
    """800,000 rows: the ids no longer fit the bitmap kernel's shared-memory bitmap, so every
    query goes to the sort kernels — also in flash_knn_graph, whose size-class plan runs
    during the build (before the handle has counted the inserted ids)."""
    rp, col = shape_slice("kdd12", 800_000)
    K, L, R, rng, k, seed = 4, 32, 64, 1 << 18, 16, 0x5EED0004
    o_ids, o_cnt = oracle.knn_graph(K, L, R, rng, seed, rp, col, k)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        g_ids, g_cnt = idx.knn_graph(d_rp, d_col, k)
        assert np.array_equal(flash.as_u32(g_ids), o_ids)
        assert np.array_equal(flash.as_u32(g_cnt), o_cnt)


def test_graph_is_deterministic_across_runs_and_streams():
    rp, col = shape_slice("webspam", 3000)
    d_rp, d_col = flash.to_device_csr(rp, col)
    outs = []
    for i in range(3):
        s = torch.cuda.Stream() if i == 2 else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            with flash.FlashIndex(4, 50, 128, 1 << 12, 3) as idx:
                ids, cnt = idx.knn_graph(d_rp, d_col, 64)
                torch.cuda.synchronize()
                outs.append((flash.as_u32(ids), flash.as_u32(cnt)))
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])


def test_errors_and_states():
    rp, col = synth.generate("tiny")
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(4, 16, 32, 1 << 15, 1) as idx:
        # query before any insert: all pads
        ids, cnt = idx.query(d_rp, d_col, 5)
        assert (flash.as_u32(ids) == EMPTY).all() and (flash.as_u32(cnt) == 0).all()
        idx.insert(d_rp, d_col)
        with pytest.raises(flash.FlashError) as e:
            idx.knn_graph(d_rp, d_col, 5)
        assert e.value.status == flash.FLASH_ESTATE
        with pytest.raises(flash.FlashError) as e:
            idx.query(d_rp, d_col, 0)
        assert e.value.status == flash.FLASH_EINVAL
        with pytest.raises(flash.FlashError) as e:  # host pointer where a device one is required
            flash.flash_hash(idx.h, torch.from_numpy(rp), d_col, 3, None,
                             torch.empty((3, 16), dtype=torch.int32, device="cuda"))
        assert e.value.status == flash.FLASH_EINVAL
        bad = torch.full((4, 16), 1 << 20, dtype=torch.int32, device="cuda")  # >= range
        idx.insert_addrs(bad, 5000)
        assert idx.errors() == 64
    with flash.FlashIndex(4, 128, 512, 1 << 15, 1) as idx:  # L*R = 65536: beyond the count tables
        with pytest.raises(flash.FlashError) as e:
            idx.query(d_rp, d_col, 5)
        assert e.value.status == flash.FLASH_EINVAL


def test_full_webspam_graph_sampled_parity():
    """The bench's workload and launch configuration (350K x 3,728 nnz, K=4, L=50, R=128,
    range 2^15, k=128): addresses of sampled rows and the graph rows of sampled queries
    match the oracle (which builds the full tables on the host)."""
    rp, col = synth.generate("webspam")
    n = rp.size - 1
    K, L, R, rng, seed, k = 4, 50, 128, 1 << 15, 0x5EED0002, 128
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, seed) as idx:
        g_ids, g_cnt = idx.knn_graph(d_rp, d_col, k)
        _, g_addrs = idx.hash(d_rp, d_col, codes=False)
        torch.cuda.synchronize()
    o_addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
    assert np.array_equal(flash.as_u32(g_addrs), o_addrs)
    T = oracle.build(L, R, rng, seed, o_addrs, np.arange(n, dtype=np.uint32))
    sample = np.random.default_rng(0).choice(n, size=400, replace=False)
    o_ids, o_cnt = oracle.query(T, o_addrs[sample], k, exclude=sample.astype(np.uint32))
    assert np.array_equal(flash.as_u32(g_ids)[sample], o_ids)
    assert np.array_equal(flash.as_u32(g_cnt)[sample], o_cnt)


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer_clean(tool):
    """compute-sanitizer finds no memory errors / shared-memory races / barrier misuse on
    small runs of every kernel family (tools/sanitize_run.py: tiny, webspam, url, kdd12
    shapes plus the edge-case rows, both build schedules, the exchange steps)."""
    import shutil
    import subprocess
    import sys

    # opt-in: the GPU pool's compute-sanitizer wrapper refuses runs (it has left GPUs needing
    # a reset); the last clean pass is profiles/r01_sanitize.txt
    if os.environ.get("FLASH_SANITIZE") != "1":
        pytest.skip("compute-sanitizer runs are opt-in (FLASH_SANITIZE=1)")
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([exe, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(root, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=1500)
    if "closed on this pool" in r.stdout + r.stderr:
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def test_table_windows_assemble_to_the_full_index():
    """The multi-GPU build path on one GPU: G handles each build a table window
    (flash_insert_addrs_window), their windows are assembled like dist.py does, imported
    into a fresh handle (flash_import_tables), and the graph equals the oracle's."""
    rp, col = shape_slice("webspam", 2500)
    n = rp.size - 1
    K, L, R, rng, seed, k = 4, 50, 128, 1 << 12, 0x5EED0002, 64
    o_ids, o_cnt = oracle.knn_graph(K, L, R, rng, seed, rp, col, k)
    d_rp, d_col = flash.to_device_csr(rp, col)
    G = 3
    with flash.FlashIndex(K, L, R, rng, seed) as full:
        addrs = full.hash_addrs(d_rp, d_col)
        parts, ids_parts, arr_sum, base = [], [], None, 0
        for g in range(G):
            t0, t1 = (L * g) // G, (L * (g + 1)) // G
            with flash.FlashIndex(K, L, R, rng, seed) as w:
                w.insert_addrs_window(addrs, 0, t0, t1)
                goff, ids, arr = w.table_arrays()
                lo, hi = int(goff[t0 * rng]), int(goff[t1 * rng])
                parts.append(goff[t0 * rng: t1 * rng] - lo + base)
                ids_parts.append(ids[lo:hi])
                arr_sum = arr if arr_sum is None else arr_sum + arr
                base += hi - lo
        parts.append(torch.tensor([base], dtype=torch.int64, device="cuda"))
        with flash.FlashIndex(K, L, R, rng, seed) as imp:
            imp.import_tables(torch.cat(parts).contiguous(), torch.cat(ids_parts).contiguous(),
                              arr_sum.contiguous())
            excl = torch.arange(n, dtype=torch.int32, device="cuda")
            g_ids, g_cnt = imp.query_addrs(addrs, k, excl)
            assert np.array_equal(flash.as_u32(g_ids), o_ids)
            assert np.array_equal(flash.as_u32(g_cnt), o_cnt)
            o_addrs = oracle.addresses(K, L, rng, seed, oracle.doph(K, L, seed, rp, col))
            T = oracle.build(L, R, rng, seed, o_addrs, np.arange(n, dtype=np.uint32))
            for t in (0, 17, 49):
                off, ids_t, arr_t = imp.table(t)
                o_off, o_ids_t, o_arr = T.table(t)
                assert np.array_equal(off, o_off) and np.array_equal(ids_t, o_ids_t) and np.array_equal(arr_t, o_arr)


EXCHANGE_CASES = [(2, 50, "0", 128, 1 << 12, 64), (3, 50, "1", 128, 1 << 12, 64), (8, 50, "0", 128, 1 << 12, 64),
                  (5, 4, "1", 128, 1 << 12, 64), (7, 13, "0", 5, 300, 17), (4, 64, "0", 32, 1 << 10, 128),
                  (6, 6, "1", 2, 64, 9), (3, 1, "0", 64, 128, 20)]


@pytest.mark.parametrize("G,L,tm,R,rng,k", EXCHANGE_CASES)
def test_candidate_exchange_loopback_equals_oracle_graph(monkeypatch, G, L, tm, R, rng, k):
    """The table-partitioned multi-GPU path (north_star (d), dist.knn_graph_candidate_exchange)
    with G virtual ranks on one GPU: every C-ABI step runs for real (owner-blocked hash,
    window build from the address all-to-all's layout, window gather, count/top-k over
    the G received segments); the all-to-alls are done by slicing.  The graph must equal
    the oracle's single-process graph exactly (G = 5 > L = 4 leaves a rank tableless)."""
    from paper_1709_01190_b200 import dist as fdist

    monkeypatch.setenv("FLASH_BUILD_TM", tm)
    rp, col = shape_slice("webspam", 1500)
    n = rp.size - 1
    K, seed = 4, 0x5EED0002
    o_ids, o_cnt = oracle.knn_graph(K, L, R, rng, seed, rp, col, k)
    bounds = fdist.shard_bounds(np.diff(rp), G)
    wins = [fdist.table_window(L, G, g) for g in range(G)]
    cnts = [bounds[g + 1] - bounds[g] for g in range(G)]
    d_rp, d_col = flash.to_device_csr(rp, col)
    idx = [flash.FlashIndex(K, L, R, rng, seed) for _ in range(G)]
    try:
        # H1-H3 per rank (owner-blocked), X1 by slicing
        sends = [idx[g].hash_addrs_blocked(d_rp[bounds[g]: bounds[g + 1] + 1], d_col, G) for g in range(G)]
        recv = []
        for h in range(G):
            w = wins[h][1] - wins[h][0]
            recv.append(torch.cat([sends[s][cnts[s] * wins[h][0]: cnts[s] * wins[h][0] + cnts[s] * w]
                                   for s in range(G)]).view(n, w))
        sizes, offs, cands = [], [], []
        for h in range(G):
            t0, t1 = wins[h]
            if t1 > t0:
                idx[h].insert_addrs_cols(recv[h], 0, t0, t1)
            sz, off = idx[h].window_sizes(recv[h], t0, t1)
            sizes.append(sz)
            offs.append(off)
            cands.append(idx[h].window_gather(recv[h], t0, t1, off, int(off[-1].item())))
        for g in range(G):  # X2 by slicing, then Q2-Q3 on the owner
            q0, q1 = bounds[g], bounds[g + 1]
            seg = torch.stack([sizes[s][q0:q1] for s in range(G)])
            cand = torch.cat([cands[s][int(offs[s][q0].item()): int(offs[s][q1].item())] for s in range(G)])
            excl = torch.arange(q0, q1, dtype=torch.int32, device="cuda")
            g_ids, g_cnt = idx[g].count_topk(cand, seg, k, n - 1, excl)
            assert np.array_equal(flash.as_u32(g_ids), o_ids[q0:q1]), f"rank {g} ids"
            assert np.array_equal(flash.as_u32(g_cnt), o_cnt[q0:q1]), f"rank {g} counts"
        assert all(i.errors() == 0 for i in idx)
    finally:
        for i in idx:
            i.close()


def test_count_topk_on_raw_segments_matches_oracle_counting():
    """flash_count_topk on arbitrary candidate segments (each id at most once per
    segment, as in a table) equals the oracle's COUNTFREQUENCY + KSELECT on the same
    multisets, including empty queries, k above the distinct count and excluded ids."""
    rng_ = np.random.default_rng(7)
    n_seg, n_q, L, k = 6, 300, 6, 20
    segs = [[np.sort(rng_.choice(5000, size=int(rng_.integers(0, 120)), replace=False)).astype(np.uint32)
             if q % 17 else np.zeros(0, np.uint32) for q in range(n_q)] for _ in range(n_seg)]
    sizes = np.array([[segs[s][q].size for q in range(n_q)] for s in range(n_seg)], np.int32)
    cand = np.concatenate([segs[s][q] for s in range(n_seg) for q in range(n_q)])
    excl = rng_.integers(0, 5000, size=n_q).astype(np.uint32)
    # oracle: one stand-in table per segment, bucket q = segment (s, q)
    off = np.zeros((n_seg, n_q + 1), np.uint32)
    stride = int(sizes.sum(axis=1).max())
    kept = np.zeros(n_seg * stride, np.uint32)
    for s in range(n_seg):
        off[s, 1:] = np.cumsum(sizes[s])
        kept[s * stride: s * stride + off[s, -1]] = np.concatenate(segs[s])
    T = oracle.Tables(n_seg, 128, n_q, np.zeros((n_seg, n_q), np.uint32), off, kept, stride)
    o_ids, o_cnt = oracle.query(T, np.tile(np.arange(n_q, dtype=np.uint32)[:, None], (1, n_seg)), k, exclude=excl)
    with flash.FlashIndex(4, L, 128, 1 << 10, 1) as idx:
        g_ids, g_cnt = idx.count_topk(torch.from_numpy(cand.view(np.int32)).cuda(),
                                      torch.from_numpy(sizes).cuda(), k, 4999,
                                      torch.from_numpy(excl.view(np.int32)).cuda())
        assert np.array_equal(flash.as_u32(g_ids), o_ids)
        assert np.array_equal(flash.as_u32(g_cnt), o_cnt)
