"""Pins for the CPU oracle against what the paper (and mathematics) fix — no GPU.

Each test names the passage it pins.  None of them re-derives the oracle's own
formula: they check special cases that reduce to textbook routines (Eq. 1
minhash, OPH), closed forms (Eq. 2 calibration, App. B retrieval probability,
Vitter's R/m law), published reference vectors, SPEC worked examples, and
brute force on tiny inputs.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EMPTY = 0xFFFFFFFF


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def perm_values(orc, seed, cols):
    """pi(c) for many c via DOPH with K*L = 1 on single-element rows (Eq. 1 with |x| = 1)."""
    cols = np.asarray(cols, dtype=np.uint32)
    rp = np.arange(cols.size + 1, dtype=np.int64)
    return orc.doph(1, 1, seed, rp, cols)[:, 0]


def tables_from_buckets(orc, buckets):
    """Oracle Tables with L = len(buckets), range = 1, table t's bucket 0 = buckets[t]."""
    L = len(buckets)
    stride = max(1, max(len(b) for b in buckets))
    kept = np.zeros(L * stride, np.uint32)
    off = np.zeros((L, 2), np.uint32)
    for t, b in enumerate(buckets):
        kept[t * stride: t * stride + len(b)] = sorted(b)
        off[t, 1] = len(b)
    arr = off[:, 1:].copy()
    return orc.Tables(L, 1 << 16, 1, arr, off, kept, stride)


# --------------------------------------------------------------------------
# Hash primitives vs published reference vectors
# --------------------------------------------------------------------------

def test_fmix32_matches_murmurhash3_reference(orc):
    for x, want in _gold("hash_vectors.json")["fmix32"]["cases"]:
        assert orc.fmix32(x) == want


def test_mix64_matches_splitmix64_stream(orc):
    outs = _gold("hash_vectors.json")["splitmix64_seed0"]["outputs"]
    for i, want in enumerate(outs):
        assert orc.mix64(((i + 1) * 0x9E3779B97F4A7C15) % (1 << 64)) == int(want, 16)


def test_perm_is_a_permutation_on_a_large_sample(orc):
    # Eq. 1 needs pi to be a permutation: no two indices share a value.
    cols = np.arange(0, 1 << 21, dtype=np.uint32) * np.uint32(2047) + np.uint32(12345)
    v = perm_values(orc, 99, cols)
    assert np.unique(v).size == cols.size


# --------------------------------------------------------------------------
# H1 / H2 — DOPH (§2.3)
# --------------------------------------------------------------------------

def test_doph_with_one_bin_is_textbook_minhash(orc):
    # K*L = 1: DOPH degenerates to h_pi(x) = min_{x_i != 0} pi(i) (Eq. 1).
    rng = np.random.default_rng(1)
    rows = [rng.choice(1 << 28, size=int(rng.integers(1, 300)), replace=False).astype(np.uint32)
            for _ in range(200)]
    rp, col = synth.csr_from_rows(rows)
    for seed in (3, 0x5EED0001):
        got = orc.doph(1, 1, seed, rp, col)[:, 0]
        want = [perm_values(orc, seed, r).min() for r in rows]
        assert np.array_equal(got, np.array(want, np.uint32))


def test_doph_equals_oph_when_no_bin_is_empty(orc):
    # OPH: B equal ranges of the permuted index space; bin b keeps its minimum
    # (north_star "DOPH reduces to OPH when no bin is empty").
    rng = np.random.default_rng(2)
    K, L, seed = 4, 4, 77
    B = K * L
    rows = [rng.choice(1 << 30, size=800, replace=False).astype(np.uint32) for _ in range(50)]
    rp, col = synth.csr_from_rows(rows)
    got = orc.doph(K, L, seed, rp, col)
    for r, row in enumerate(rows):
        h = perm_values(orc, seed, row).astype(np.uint64)
        bins = (h * B) >> 32  # bin b = [b*2^32/B, (b+1)*2^32/B)
        want = np.full(B, EMPTY, np.uint64)
        for b in range(B):
            sel = h[bins == b]
            assert sel.size > 0, "test premise: every bin non-empty"
            want[b] = sel.min()
        assert np.array_equal(got[r].astype(np.uint64), want)


def test_densified_bins_copy_the_first_nonempty_bin_on_the_probe_chain(orc):
    # Reading R#4 (optimal densification, ref [36] via P:132): brute force on tiny rows.
    K, L, seed, B = 8, 8, 5, 64
    rng = np.random.default_rng(3)
    rows = [rng.choice(1 << 30, size=int(rng.integers(1, 6)), replace=False).astype(np.uint32)
            for _ in range(30)]
    rp, col = synth.csr_from_rows(rows)
    got = orc.doph(K, L, seed, rp, col)
    for r, row in enumerate(rows):
        h = perm_values(orc, seed, row).astype(np.uint64)
        native = {}
        for v in h:
            b = int((v * B) >> 32)
            native[b] = min(native.get(b, EMPTY), int(v))
        for i in range(B):
            if i in native:
                assert got[r, i] == native[i]
                continue
            donor = None
            for a in range(1, 65):
                j = orc.probe(seed, i, a, B)
                if j in native:
                    donor = native[j]
                    break
            if donor is None:
                for m in range(1, B + 1):
                    jj = (j + m) % B
                    if jj in native:
                        donor = native[jj]
                        break
            assert got[r, i] == donor
            assert donor in native.values()  # donors are original bins only


def test_doph_is_a_set_function(orc):
    rng = np.random.default_rng(4)
    base = rng.choice(1 << 24, size=400, replace=False).astype(np.uint32)
    rows = [base, base[::-1].copy(), np.concatenate([base, base[:100], base[5:9]]),
            rng.permutation(base)]
    rp, col = synth.csr_from_rows(rows)
    c = orc.doph(4, 50, 11, rp, col)
    for r in range(1, len(rows)):
        assert np.array_equal(c[0], c[r])


def test_empty_row_gets_empty_codes_and_no_address(orc):
    rp, col = synth.csr_from_rows([np.zeros(0, np.uint32), np.array([7], np.uint32)])
    c = orc.doph(4, 16, 1, rp, col)
    assert (c[0] == EMPTY).all() and (c[1] != EMPTY).all()
    a = orc.addresses(4, 16, 1 << 15, 1, c)
    assert (a[0] == EMPTY).all() and (a[1] < (1 << 15)).all()


def _planted_pair(rng, a, b):
    ids = rng.choice(1 << 30, size=a + 2 * b, replace=False).astype(np.uint32)
    return np.concatenate([ids[:a], ids[a:a + b]]), np.concatenate([ids[:a], ids[a + b:]])


@pytest.mark.parametrize("a,b,B", [(200, 100, 64), (100, 200, 64), (400, 50, 64),   # dense
                                    (6, 3, 64), (2, 4, 64), (8, 1, 64)])              # densified
def test_collision_rate_is_jaccard(orc, a, b, B):
    # Eq. 2: Pr[h(x) = h(y)] = J(x,y); per-bin, over >= 4000 seeds, within 0.02
    # (S:131/S:470).  The sparse rows (|x| <= 9, B = 64) make most bins densified,
    # which pins the densification rule (R#4).
    rng = np.random.default_rng(a * 1000 + b)
    x, y = _planted_pair(rng, a, b)
    J = a / (a + 2 * b)
    rp, col = synth.csr_from_rows([x, y])
    hits = tot = 0
    for s in range(4000):
        c = orc.doph(B, 1, 7919 * s + 13, rp, col)
        hits += int(np.sum(c[0] == c[1]))
        tot += B
    assert abs(hits / tot - J) < 0.02


def test_collision_rate_is_monotone_in_similarity(orc):
    # Definition 3 / S:145: J(q,x) > J(q,y) + 0.1 => higher collision rate.
    rng = np.random.default_rng(9)
    core = rng.choice(1 << 30, size=200, replace=False).astype(np.uint32)
    fresh = rng.choice(1 << 30, size=400, replace=False).astype(np.uint32) | np.uint32(1 << 30)
    q = core[:60]
    x = np.concatenate([core[:40], fresh[:20]])      # J = 40/80 = 0.5
    y = np.concatenate([core[:24], fresh[20:56]])    # J = 24/96 = 0.25
    rp, col = synth.csr_from_rows([q, x, y])
    hx = hy = 0
    for s in range(1500):
        c = orc.doph(4, 4, s + 1, rp, col)
        hx += int(np.sum(c[0] == c[1]))
        hy += int(np.sum(c[0] == c[2]))
    assert hx > hy
    assert abs(hx / 24000 - 0.5) < 0.03 and abs(hy / 24000 - 0.25) < 0.03


# --------------------------------------------------------------------------
# H3 — MapKHashesToAddress (Alg. 2 line 5)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("range_", [1 << 15, 1000, 1])
def test_addresses_in_range_and_uniform(orc, range_):
    rng = np.random.default_rng(range_)
    K, L = 4, 8
    codes = rng.integers(0, EMPTY, size=(100_000 // L, K * L), dtype=np.uint64).astype(np.uint32)
    a = orc.addresses(K, L, range_, 21, codes)
    assert (a < range_).all()
    if range_ > 1:
        # chi-square uniformity: p > 0.001
        from scipy.stats import chisquare
        cnt = np.bincount(a.ravel().astype(np.int64), minlength=range_)
        assert chisquare(cnt).pvalue > 1e-3


def test_equal_tuples_map_to_equal_addresses_and_tables_are_independent(orc):
    K, L = 3, 64
    row = np.arange(K * L, dtype=np.uint32) * 7 + 1
    codes = np.stack([row, row])
    a = orc.addresses(K, L, 1 << 20, 5, codes)
    assert np.array_equal(a[0], a[1])
    # the same K-tuple in every table maps independently per table
    same = np.tile(np.array([11, 22, 33], np.uint32), L)[None, :]
    b = orc.addresses(K, L, 1 << 20, 5, same)[0]
    assert np.unique(b).size > L - 3
    # changing one code of table t changes only a_t
    c2 = codes[:1].copy()
    c2[0, 5 * K + 1] ^= 1
    d = orc.addresses(K, L, 1 << 20, 5, c2)[0]
    assert (d != a[0]).sum() == 1 and d[5] != a[0][5]


# --------------------------------------------------------------------------
# B — bottom-R reservoirs (Alg. 2 ADD; Alg. 1's law)
# --------------------------------------------------------------------------

def _random_build_input(rng, n, L, range_):
    addrs = rng.integers(0, range_, size=(n, L), dtype=np.uint64).astype(np.uint32)
    ids = rng.permutation(np.arange(n, dtype=np.uint32) * 3 + 1000)
    return addrs, ids


def test_buckets_hold_min_arrivals_R_and_equal_bruteforce(orc):
    rng = np.random.default_rng(10)
    L, R, range_, seed = 3, 4, 16, 123
    addrs, ids = _random_build_input(rng, 300, L, range_)
    addrs[::7, 1] = EMPTY  # not inserted
    T = orc.build(L, R, range_, seed, addrs, ids)
    for t in range(L):
        off, kept, arr = T.table(t)
        for b in range(range_):
            S = [int(i) for i, a in zip(ids, addrs[:, t]) if a == b]
            assert arr[b] == len(S)
            got = list(kept[off[b]:off[b + 1]])
            assert len(got) == min(len(S), R)                    # north_star invariant
            want = sorted(sorted(S, key=lambda i: (orc.prio(seed, t, b, i), i))[:R])
            assert got == want                                    # brute force, ascending ids


def test_build_is_insert_order_invariant_and_composable(orc):
    rng = np.random.default_rng(11)
    L, R, range_, seed = 4, 5, 64, 9
    addrs, ids = _random_build_input(rng, 2000, L, range_)
    T = orc.build(L, R, range_, seed, addrs, ids)
    p = rng.permutation(ids.size)
    T2 = orc.build(L, R, range_, seed, addrs[p], ids[p])
    assert np.array_equal(T.off, T2.off) and np.array_equal(T.arrivals, T2.arrivals)
    for t in range(L):
        assert np.array_equal(T.table(t)[1], T2.table(t)[1])
    # composability: bottom-R(S_A ∪ S_B) = bottom-R(kept(A) ∪ S_B)
    A = slice(0, 1200)
    TA = orc.build(L, R, range_, seed, addrs[A], ids[A])
    for t in range(L):
        offA, keptA, _ = TA.table(t)
        kept_addr = np.repeat(np.arange(range_, dtype=np.uint32), np.diff(offA).astype(np.int64))
        addr_mix = np.concatenate([kept_addr, addrs[1200:, t]])
        id_mix = np.concatenate([keptA, ids[1200:]])
        got = {}
        for b in range(range_):
            members = [int(i) for i, a in zip(id_mix, addr_mix) if a == b]
            got[b] = sorted(sorted(members, key=lambda i: (orc.prio(seed, t, b, i), i))[:R])
        off, kept, _ = T.table(t)
        for b in range(range_):
            assert list(kept[off[b]:off[b + 1]]) == got[b]


def test_reservoir_inclusion_frequency_is_R_over_m(orc):
    # Vitter's guarantee: each of m streamed ids kept w.p. R/m.
    m, R, trials = 2000, 32, 1000
    addrs = np.zeros((m, 1), np.uint32)
    ids = np.arange(m, dtype=np.uint32)
    hits = np.zeros(m, np.int64)
    for s in range(trials):
        T = orc.build(1, R, 1, 1000 + s, addrs, ids)
        hits[T.kept[:R]] += 1
    p = R / m
    se = math.sqrt(p * (1 - p) / trials)
    freq = hits / trials
    assert abs(freq.mean() - p) < 1e-12  # exactly R kept every time
    assert np.mean(np.abs(freq - p) > 3 * se) < 0.01
    from scipy.stats import chisquare
    assert chisquare(hits).pvalue > 1e-3


def test_reservoir_subsets_are_uniform(orc):
    # Alg. 1 / Vitter: all C(6,2) = 15 subsets equally likely (chi-square).
    m, R, trials = 6, 2, 6000
    addrs = np.zeros((m, 1), np.uint32)
    ids = np.arange(m, dtype=np.uint32)
    subsets = {c: 0 for c in itertools.combinations(range(m), R)}
    for s in range(trials):
        T = orc.build(1, R, 1, 50_000 + s, addrs, ids)
        subsets[tuple(int(v) for v in T.kept[:R])] += 1
    from scipy.stats import chisquare
    assert chisquare(list(subsets.values())).pvalue > 1e-3


def test_vitter_algorithm1_has_the_same_law(orc):
    # Literal Alg. 1 (inclusive RANDOM([0,i]), j < R; reading R#8) simulated
    # directly: its inclusion law matches the bottom-R oracle's (both R/m).
    rng = np.random.default_rng(12)
    m, R, trials = 40, 4, 4000
    vit = np.zeros(m, np.int64)
    for _ in range(trials):
        res = list(range(R))
        for i in range(R, m):
            j = int(rng.integers(0, i + 1))
            if j < R:
                res[j] = i
        vit[res] += 1
    bot = np.zeros(m, np.int64)
    addrs = np.zeros((m, 1), np.uint32)
    ids = np.arange(m, dtype=np.uint32)
    for s in range(trials):
        bot[orc.build(1, R, 1, 7 + s, addrs, ids).kept[:R]] += 1
    from scipy.stats import chi2_contingency
    assert chi2_contingency(np.stack([vit, bot])).pvalue > 1e-3


# --------------------------------------------------------------------------
# Q — count-based k-selection (Alg. 3)
# --------------------------------------------------------------------------

def test_spec_worked_examples_count_and_kselect(orc):
    g = _gold("spec_examples.json")
    A = g["count_frequencies"]["A"]
    # represent A as buckets whose concatenation is A (each table holds distinct ids)
    buckets = [[5, 3], [5, 3, 2], [5]]
    assert sorted(sum(buckets, [])) == sorted(A)
    T = tables_from_buckets(orc, buckets)
    ids, cnt = orc.query(T, np.zeros((1, 3), np.uint32), 3)
    assert {int(i): int(c) for i, c in zip(ids[0], cnt[0])} == {int(k): v for k, v in g["count_frequencies"]["counts"].items()}
    for ex in g["k_select"]:
        vals = ex["A"]
        bks = [[v] for v in vals] if len(set(vals)) == len(vals) else buckets
        T = tables_from_buckets(orc, bks)
        ids, cnt = orc.query(T, np.zeros((1, len(bks)), np.uint32), ex["k"])
        assert [[int(i), int(c)] for i, c in zip(ids[0], cnt[0])] == ex["out"]


def test_kselect_pads_when_fewer_than_k_and_excludes_before_truncation(orc):
    T = tables_from_buckets(orc, [[1, 2], [2, 3], [2]])
    ids, cnt = orc.query(T, np.zeros((1, 3), np.uint32), 5, exclude=np.array([2], np.uint32))
    assert list(ids[0]) == [1, 3, EMPTY, EMPTY, EMPTY] and list(cnt[0]) == [1, 1, 0, 0, 0]
    ids, cnt = orc.query(T, np.full((1, 3), EMPTY, np.uint32), 2)  # empty query row
    assert list(ids[0]) == [EMPTY, EMPTY] and list(cnt[0]) == [0, 0]


def test_count_without_eviction_is_number_of_shared_addresses(orc):
    # With R >= N nothing is evicted, so count(q, x) = #{t : addr_t(q) = addr_t(x)}
    # (the collision count of §3.3.2) — a definition that uses no tables.
    rp, col = synth.generate(synth.SHAPES["tiny"].with_(N=300))
    K, L, range_, seed = 2, 12, 64, 31
    addrs = orc.addresses(K, L, range_, seed, orc.doph(K, L, seed, rp, col))
    n = addrs.shape[0]
    ids = np.arange(n, dtype=np.uint32)
    T = orc.build(L, n, range_, seed, addrs, ids)
    got_ids, got_cnt = orc.query(T, addrs, n, exclude=ids)
    shared = (addrs[:, None, :] == addrs[None, :, :]).sum(-1)
    for q in range(0, n, 7):
        want = sorted(((int(shared[q, x]), x) for x in range(n) if x != q and shared[q, x] > 0),
                      key=lambda p: (-p[0], p[1]))
        m = len(want)
        assert [int(v) for v in got_ids[q, :m]] == [x for _, x in want]
        assert [int(v) for v in got_cnt[q, :m]] == [c for c, _ in want]
        assert (got_ids[q, m:] == EMPTY).all()


def test_mean_count_estimates_L_times_jaccard_for_K1(orc):
    # §3.3.2: the count is a binomial estimator of L * CP(q,x); with K = 1 and
    # a huge range CP = J.  Averaged over seeds, within 0.05 * L.
    rng = np.random.default_rng(13)
    q, x = _planted_pair(rng, 60, 20)  # J = 0.6
    rp, col = synth.csr_from_rows([q, x])
    L, counts = 32, []
    for s in range(200):
        a = orc.addresses(1, L, 1 << 12, s, orc.doph(1, L, s, rp, col))
        T = orc.build(L, 4, 1 << 12, s, a, np.arange(2, dtype=np.uint32))
        ids, cnt = orc.query(T, a[:1], 2, exclude=np.array([0], np.uint32))
        counts.append(int(cnt[0, 0]) if ids[0, 0] == 1 else 0)
    assert abs(np.mean(counts) / L - 0.6) < 0.05


def test_retrieval_probability_matches_appendix_b(orc):
    # App. B: Pr[x retrieved] = 1 - (1 - J^K)^L without eviction.
    rng = np.random.default_rng(14)
    K, L = 3, 4
    q, x = _planted_pair(rng, 70, 15)  # J = 0.7
    J = 70 / 100
    want = 1 - (1 - J ** K) ** L
    rp, col = synth.csr_from_rows([q, x])
    hit, trials = 0, 3000
    for s in range(trials):
        a = orc.addresses(K, L, 1 << 30, s, orc.doph(K, L, s, rp, col))
        hit += int((a[0] == a[1]).any())
    assert abs(hit / trials - want) < 0.03


def test_knn_graph_self_exclusion_and_identical_pair(orc):
    rows = [np.arange(50, dtype=np.uint32) + 1000, np.arange(50, dtype=np.uint32) + 1000,
            np.arange(30, dtype=np.uint32) + 9000]
    rp, col = synth.csr_from_rows(rows)
    K, L, R = 2, 10, 8
    ids, cnt = orc.knn_graph(K, L, R, 1 << 15, 1, rp, col, 2)
    assert ids[0, 0] == 1 and cnt[0, 0] == L and ids[1, 0] == 0 and cnt[1, 0] == L
    for r in range(3):
        assert r not in set(int(v) for v in ids[r])


def test_counts_never_exceed_L_and_rows_are_sorted(orc):
    rp, col = synth.generate("tiny")
    ids, cnt = orc.knn_graph(4, 16, 32, 1 << 15, 0x5EED0001, rp, col, 10)
    assert cnt.max() <= 16
    valid = ids != EMPTY
    for r in range(ids.shape[0]):
        v = valid[r]
        assert (cnt[r][~v] == 0).all() and v[:v.sum()].all()
        pairs = list(zip(-cnt[r][v].astype(np.int64), ids[r][v]))
        assert pairs == sorted(pairs) and len(set(ids[r][v])) == v.sum()


# --------------------------------------------------------------------------
# O-2 brute force (Eq. 2, Eq. 3)
# --------------------------------------------------------------------------

def test_similarity_worked_examples(orc):
    g = _gold("spec_examples.json")
    rp, col = synth.csr_from_rows([g["jaccard"]["x"], g["jaccard"]["y"]])
    assert orc.pair_similarity(rp, col, [[0, 1]], "jaccard")[0] == g["jaccard"]["value"]
    assert abs(orc.pair_similarity(rp, col, [[0, 1]], "cosine")[0] - g["cosine"]["value"]) < 1e-15


def test_bruteforce_matches_independent_dense_computation(orc):
    # agreement with an independent O(N^2) pairwise scan on 100 points.
    rng = np.random.default_rng(15)
    n, D = 100, 400
    M = rng.random((n, D)) < 0.05
    M[3] = M[7]  # an exact duplicate pair
    rows = [np.flatnonzero(M[i]).astype(np.uint32) for i in range(n)]
    rp, col = synth.csr_from_rows(rows)
    inter = M.astype(np.int64) @ M.T.astype(np.int64)
    sz = M.sum(1)
    union = sz[:, None] + sz[None, :] - inter
    Jm = np.where(union > 0, inter / np.maximum(union, 1), 0.0)
    Cm = np.where((sz[:, None] * sz[None, :]) > 0, inter / np.sqrt(np.maximum(sz[:, None] * sz[None, :], 1)), 0.0)
    for metric, S in (("jaccard", Jm), ("cosine", Cm)):
        ids, sim = orc.bruteforce_topk(rp, col, np.arange(n), 5, metric)
        for q in range(n):
            order = sorted((x for x in range(n) if x != q), key=lambda x: (-S[q, x], x))[:5]
            assert list(ids[q]) == order
            assert np.allclose(sim[q], S[q, order], rtol=0, atol=1e-12)


def test_app_a_reservoir_bound_first_holds_at_R5():
    g = _gold("spec_examples.json")["app_a_reservoir_bound"]
    ok = [R for R in range(1, 50) if (1 - 1 / math.e) * (1 - 1 / R) > 0.5]
    assert ok[0] == g["first_R"]


def test_oracle_graph_recall_on_planted_tiny(orc):
    # Sanity: the oracle graph recovers planted near-duplicates (P:393 R@k definition).
    rp, col = synth.generate("tiny")
    ids, cnt = orc.knn_graph(4, 16, 32, 1 << 15, 0x5EED0001, rp, col, 10)
    q = np.arange(0, 1000, 5)
    bf, sim = orc.bruteforce_topk(rp, col, q, 1, "jaccard")
    hit = [bf[i, 0] in set(ids[qq]) for i, qq in enumerate(q) if sim[i, 0] > 0.3]
    assert np.mean(hit) > 0.9


def test_exclusion_happens_before_truncation(orc):
    # R#14 / S:338: the excluded id is removed before the top-k cut.
    T = tables_from_buckets(orc, [[1, 2], [2, 3], [2]])
    ids, cnt = orc.query(T, np.zeros((1, 3), np.uint32), 1, exclude=np.array([2], np.uint32))
    assert list(ids[0]) == [1] and list(cnt[0]) == [1]


def test_reservoirs_of_different_tables_sample_independently(orc):
    # R#9: the priority must depend on the table (and bucket), otherwise the same ids
    # would win in every table and counts would be biased.  Two tables receive the
    # same m ids in one bucket: the kept sets overlap ~ R^2/m, not R.
    m, R = 4000, 64
    addrs = np.zeros((m, 2), np.uint32)
    ids = np.arange(m, dtype=np.uint32)
    overlaps = []
    for s in range(50):
        T = orc.build(2, R, 1, 300 + s, addrs, ids)
        a, b = T.table(0)[1], T.table(1)[1]
        overlaps.append(np.intersect1d(a, b).size)
    assert abs(np.mean(overlaps) - R * R / m) < 1.0


# --------------------------------------------------------------------------
# Reservoir sharing across tables (§3.2(4); §3.5, Fig. 3/4; R#23)
# --------------------------------------------------------------------------

def test_pool_with_full_allocation_is_the_unshared_index(orc):
    """F = 1 (P = L*range): every reservoir is one table's bucket, exactly the unshared
    build and query ("Allocated Range = F * Actual Range")."""
    rng = np.random.default_rng(40)
    L, R, range_, seed = 5, 6, 32, 9
    addrs, ids = _random_build_input(rng, 500, L, range_)
    addrs[::5, 2] = EMPTY
    T = orc.build(L, R, range_, seed, addrs, ids)
    P = orc.build_pool(L, R, range_, L * range_, seed, addrs, ids)
    assert P.arrivals.tolist() == T.arrivals.reshape(-1).tolist()
    flat = np.concatenate([T.table(t)[1] for t in range(L)])
    assert np.array_equal(P.kept, flat)
    q = addrs[:60]
    want = orc.query(T, q, 7, exclude=ids[:60])
    got = orc.query_pool(P, seed, q, 7, exclude=ids[:60])
    assert np.array_equal(want[0], got[0]) and np.array_equal(want[1], got[1])


def test_pool_reservoirs_equal_bruteforce(orc):
    """Brute force with Python sets: a reservoir holds the distinct rows pointing to it
    through any of their tables (a row enters a shared reservoir once), keeps the
    min(arrivals, R) with smallest (prio, id), ascending."""
    rng = np.random.default_rng(41)
    L, R, range_, seed = 4, 3, 16, 77
    addrs, ids = _random_build_input(rng, 200, L, range_)
    addrs[::9, 0] = EMPTY
    P = orc.pool_size(0.25, L, range_)
    T = orc.build_pool(L, R, range_, P, seed, addrs, ids)
    members = [set() for _ in range(P)]
    for row, i in zip(addrs, ids):
        for t in range(L):
            if row[t] != EMPTY:
                members[orc.reservoir(seed, t, int(row[t]), L, range_, P)].add(int(i))
    for r in range(P):
        S = members[r]
        assert T.arrivals[r] == len(S)
        want = sorted(sorted(S, key=lambda i: (orc.prio(seed, r // range_, r % range_, i), i))[:R])
        assert T.reservoir(r).tolist() == want
    assert T.off[-1] == sum(min(len(S), R) for S in members)  # memory <= P reservoirs of R


def test_pool_binding_is_uniform(orc):
    """Each table bucket points to a uniformly random shared reservoir: chi-square
    over the pool for every (t, b) cell, p > 0.001."""
    from scipy.stats import chisquare

    L, range_, seed = 8, 4096, 5
    P = orc.pool_size(0.125, L, range_)
    hits = np.zeros(P, np.int64)
    for t in range(L):
        for b in range(range_):
            hits[orc.reservoir(seed, t, b, L, range_, P)] += 1
    assert chisquare(hits).pvalue > 1e-3


def test_pool_queries_return_only_inserted_ids_and_counts_le_L(orc):
    """SPEC S:234 sharing correctness: every reported id was inserted into one of the
    query's reservoirs, and its count (each distinct reservoir aggregated once) is at most
    the number of those reservoirs <= L."""
    rng = np.random.default_rng(42)
    L, R, range_, seed, k = 6, 8, 16, 3, 12
    addrs, ids = _random_build_input(rng, 400, L, range_)
    P = orc.pool_size(0.1, L, range_)
    T = orc.build_pool(L, R, range_, P, seed, addrs, ids)
    got_ids, got_cnt = orc.query_pool(T, seed, addrs[:80], k)
    for q in range(80):
        res = {orc.reservoir(seed, t, int(addrs[q, t]), L, range_, P) for t in range(L)}
        for i, c in zip(got_ids[q], got_cnt[q]):
            if i == EMPTY:
                continue
            holders = [r for r in res if int(i) in set(T.reservoir(r).tolist())]
            assert c == len(holders) and 1 <= c <= len(res) <= L


def test_pool_quality_degrades_only_for_small_F(orc):
    """Fig. 4: search quality is essentially unchanged down to F = 0.2 and
    degrades for very small F.  R@10 of the exact cosine 1-NN on planted tiny data."""
    rp, col = synth.generate(synth.SHAPES["tiny"].with_(N=3000, seed=21))
    n = rp.size - 1
    K, L, R, range_, seed, k = 4, 32, 16, 1 << 12, 77, 10
    nn, _ = orc.bruteforce_topk(rp, col, np.arange(n), 1, metric="cosine")

    def recall(F):
        ids, cnt = orc.knn_graph_pool(K, L, R, range_, orc.pool_size(F, L, range_), seed, rp, col, k)
        assert cnt.max() <= L
        return np.mean([nn[q, 0] in set(ids[q].tolist()) for q in range(n)])

    full = recall(1.0)
    assert recall(0.2) >= full - 0.01
    assert recall(0.002) < full - 0.3
