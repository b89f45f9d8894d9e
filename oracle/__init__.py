"""CPU oracle for FLASH's hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1709_01190_b200`` never imports it, and it never imports the product.

Thin ctypes marshalling over ``oracle/flash_oracle.c`` (plain C + OpenMP); every
function there cites the PAPER.md passage it follows.  Parity status: the hash
constants are HASHSPEC choices that the paper does not print ("parity unpinned"
against the paper for the raw hash values); they are pinned by the MurmurHash3 /
SplitMix64 reference vectors and statistically (Eq. 2 calibration, Vitter's
reservoir law) in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

EMPTY = 0xFFFFFFFF
_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "flash_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")


def build_lib(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = ctypes.CDLL(_SO)
        u32, u64, i32, vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        L.oracle_fmix32.argtypes, L.oracle_fmix32.restype = [u32], u32
        L.oracle_mix64.argtypes, L.oracle_mix64.restype = [u64], u64
        L.oracle_perm.argtypes, L.oracle_perm.restype = [u64, u32], u32
        L.oracle_probe.argtypes, L.oracle_probe.restype = [u64, u32, u32, u32], u32
        L.oracle_prio.argtypes, L.oracle_prio.restype = [u64, u32, u32, u32], u32
        L.oracle_reservoir.argtypes, L.oracle_reservoir.restype = [u64, u32, u32, u32, u32, u64], u32
        L.oracle_build_pool.argtypes = [u32, u32, u32, u64, u64, vp, vp, u64, vp, vp, vp]
        L.oracle_query_pool.argtypes = [u32, u32, u64, u64, vp, vp, vp, u64, u32, vp, vp, vp]
        L.oracle_build_pool.restype = i32
        L.oracle_query_pool.restype = i32
        L.oracle_prio_batch.argtypes = [u64, vp, vp, vp, u64, vp]
        L.oracle_prio_batch.restype = None
        L.oracle_doph.argtypes = [u32, u32, u64, vp, vp, u64, vp]
        L.oracle_addresses.argtypes = [u32, u32, u32, u64, vp, u64, vp]
        L.oracle_build.argtypes = [u32, u32, u32, u64, vp, vp, u64, vp, vp, vp]
        L.oracle_query.argtypes = [u32, u32, vp, vp, u64, vp, u64, u32, vp, vp, vp]
        L.oracle_knn_graph.argtypes = [u32, u32, u32, u32, u64, vp, vp, u64, u32, vp, vp]
        L.oracle_pair_similarity.argtypes = [vp, vp, u64, vp, u64, i32, vp]
        L.oracle_bruteforce_topk.argtypes = [vp, vp, u64, vp, u64, u32, i32, i32, vp, vp]
        for f in ("oracle_doph", "oracle_addresses", "oracle_build", "oracle_query",
                  "oracle_knn_graph", "oracle_pair_similarity", "oracle_bruteforce_topk"):
            getattr(L, f).restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _csr(row_ptr, col_idx):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.uint32)
    if ci.size == 0:
        ci = np.zeros(1, np.uint32)
    return rp, ci


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"{what} failed (rc={rc})")


# ---- primitives -----------------------------------------------------------

def fmix32(h: int) -> int:
    return lib().oracle_fmix32(h & 0xFFFFFFFF)


def mix64(z: int) -> int:
    return lib().oracle_mix64(z & 0xFFFFFFFFFFFFFFFF)


def perm(seed: int, c: int) -> int:
    return lib().oracle_perm(seed, c)


def probe(seed: int, i: int, a: int, B: int) -> int:
    return lib().oracle_probe(seed, i, a, B)


def prio(seed: int, t: int, b: int, id_: int) -> int:
    return lib().oracle_prio(seed, t, b, id_)


def prio_batch(seed: int, t, b, ids) -> np.ndarray:
    """prio(t[i], b[i], ids[i]) for arrays of equal length (HASHSPEC B; R#9)."""
    t = np.ascontiguousarray(t, dtype=np.uint32)
    b = np.ascontiguousarray(b, dtype=np.uint32)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    out = np.empty(max(t.size, 1), dtype=np.uint32)
    if t.size:
        lib().oracle_prio_batch(seed & 0xFFFFFFFFFFFFFFFF, _p(t), _p(b), _p(ids), t.size, _p(out))
    return out[:t.size]


# ---- the path -------------------------------------------------------------

def doph(K: int, L: int, seed: int, row_ptr, col_idx) -> np.ndarray:
    """codes uint32 [n][K*L] (§2.3; DESIGN.md HASHSPEC H1-H2)."""
    rp, ci = _csr(row_ptr, col_idx)
    n = rp.size - 1
    codes = np.empty((max(n, 1), K * L), dtype=np.uint32)
    _check(lib().oracle_doph(K, L, seed, _p(rp), _p(ci), n, _p(codes)), "oracle_doph")
    return codes[:n]


def addresses(K: int, L: int, range_: int, seed: int, codes: np.ndarray) -> np.ndarray:
    """addrs uint32 [n][L] (Alg. 2 line 5; HASHSPEC H3)."""
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    n = codes.shape[0]
    out = np.empty((max(n, 1), L), dtype=np.uint32)
    _check(lib().oracle_addresses(K, L, range_, seed, _p(codes if n else np.zeros((1, K * L), np.uint32)), n, _p(out)),
           "oracle_addresses")
    return out[:n]


class Tables:
    """Oracle index: arrivals [L][range], off [L][range+1], kept ids per table."""

    def __init__(self, L, R, range_, arrivals, off, kept, stride):
        self.L, self.R, self.range = L, R, range_
        self.arrivals, self.off, self.kept, self.stride = arrivals, off, kept, stride

    def table(self, t: int):
        o = self.off[t]
        return o, self.kept[t * self.stride: t * self.stride + int(o[-1])], self.arrivals[t]


def build(L: int, R: int, range_: int, seed: int, addrs: np.ndarray, ids: np.ndarray) -> Tables:
    """Adding phase (Alg. 2) with bottom-R reservoirs over ALL ids given (HASHSPEC B)."""
    addrs = np.ascontiguousarray(addrs, dtype=np.uint32).reshape(-1, L)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    n = addrs.shape[0]
    arrivals = np.empty((L, range_), dtype=np.uint32)
    off = np.empty((L, range_ + 1), dtype=np.uint32)
    kept = np.empty(max(n * L, 1), dtype=np.uint32)
    a = addrs if n else np.full((1, L), EMPTY, np.uint32)
    i = ids if n else np.zeros(1, np.uint32)
    _check(lib().oracle_build(L, R, range_, seed, _p(a), _p(i), n, _p(arrivals), _p(off), _p(kept)),
           "oracle_build")
    return Tables(L, R, range_, arrivals, off, kept, n)


def query(tables: Tables, q_addrs: np.ndarray, k: int, exclude=None):
    """Querying phase (Alg. 3): top-k (ids, counts), each uint32 [n_q][k]."""
    L = tables.L
    q = np.ascontiguousarray(q_addrs, dtype=np.uint32).reshape(-1, L)
    nq = q.shape[0]
    ids = np.empty((max(nq, 1), k), dtype=np.uint32)
    cnt = np.empty((max(nq, 1), k), dtype=np.uint32)
    ex = None if exclude is None else np.ascontiguousarray(exclude, dtype=np.uint32)
    kept = tables.kept if tables.kept.size else np.zeros(1, np.uint32)
    _check(lib().oracle_query(L, tables.range, _p(tables.off), _p(kept), tables.stride,
                              _p(q if nq else np.full((1, L), EMPTY, np.uint32)), nq, k,
                              _p(ex), _p(ids), _p(cnt)), "oracle_query")
    return ids[:nq], cnt[:nq]


# ---- reservoir sharing (§3.2(4), §3.5; R#23) ---------------------

def pool_size(F: float, L: int, range_: int) -> int:
    """P = ceil(F * L * range) shared reservoirs ("Allocated Range = F * Actual Range")."""
    import math
    return max(1, min(L * range_, int(math.ceil(F * L * range_))))


def reservoir(seed: int, t: int, b: int, L: int, range_: int, P: int) -> int:
    return lib().oracle_reservoir(seed, t, b, L, range_, P)


class PoolTables:
    """Oracle index over a shared pool: arrivals [P], off [P+1], kept ids (flat)."""

    def __init__(self, L, R, range_, P, arrivals, off, kept):
        self.L, self.R, self.range, self.P = L, R, range_, P
        self.arrivals, self.off, self.kept = arrivals, off, kept

    def reservoir(self, r: int):
        return self.kept[self.off[r]: self.off[r + 1]]


def build_pool(L: int, R: int, range_: int, P: int, seed: int, addrs: np.ndarray, ids: np.ndarray) -> PoolTables:
    """Adding phase over P shared reservoirs (oracle_build_pool)."""
    addrs = np.ascontiguousarray(addrs, dtype=np.uint32).reshape(-1, L)
    ids = np.ascontiguousarray(ids, dtype=np.uint32)
    n = addrs.shape[0]
    arrivals = np.empty(P, dtype=np.uint32)
    off = np.empty(P + 1, dtype=np.uint32)
    kept = np.empty(max(n * L, 1), dtype=np.uint32)
    a = addrs if n else np.full((1, L), EMPTY, np.uint32)
    i = ids if n else np.zeros(1, np.uint32)
    _check(lib().oracle_build_pool(L, R, range_, P, seed, _p(a), _p(i), n, _p(arrivals), _p(off), _p(kept)),
           "oracle_build_pool")
    return PoolTables(L, R, range_, P, arrivals, off, kept[: int(off[-1])].copy())


def query_pool(T: PoolTables, seed: int, q_addrs: np.ndarray, k: int, exclude=None):
    """Querying phase over the shared pool (oracle_query_pool): top-k (ids, counts)."""
    L = T.L
    q = np.ascontiguousarray(q_addrs, dtype=np.uint32).reshape(-1, L)
    nq = q.shape[0]
    ids = np.empty((max(nq, 1), k), dtype=np.uint32)
    cnt = np.empty((max(nq, 1), k), dtype=np.uint32)
    ex = None if exclude is None else np.ascontiguousarray(exclude, dtype=np.uint32)
    kept = T.kept if T.kept.size else np.zeros(1, np.uint32)
    _check(lib().oracle_query_pool(L, T.range, T.P, seed, _p(T.off), _p(kept),
                                   _p(q if nq else np.full((1, L), EMPTY, np.uint32)), nq, k, _p(ex),
                                   _p(ids), _p(cnt)), "oracle_query_pool")
    return ids[:nq], cnt[:nq]


def knn_graph_pool(K, L, R, range_, P, seed, row_ptr, col_idx, k):
    """k-NN graph over a shared pool: insert ids 0..n-1, query every row excluding itself."""
    rp, ci = _csr(row_ptr, col_idx)
    n = rp.size - 1
    a = addresses(K, L, range_, seed, doph(K, L, seed, rp, ci))
    T = build_pool(L, R, range_, P, seed, a, np.arange(n, dtype=np.uint32))
    return query_pool(T, seed, a, k, exclude=np.arange(n, dtype=np.uint32))


def knn_graph(K, L, R, range_, seed, row_ptr, col_idx, k):
    rp, ci = _csr(row_ptr, col_idx)
    n = rp.size - 1
    ids = np.empty((max(n, 1), k), dtype=np.uint32)
    cnt = np.empty((max(n, 1), k), dtype=np.uint32)
    _check(lib().oracle_knn_graph(K, L, R, range_, seed, _p(rp), _p(ci), n, k, _p(ids), _p(cnt)),
           "oracle_knn_graph")
    return ids[:n], cnt[:n]


# ---- O-2: exact similarities ---------------------------------------------

def pair_similarity(row_ptr, col_idx, pairs, metric: str = "jaccard") -> np.ndarray:
    rp, ci = _csr(row_ptr, col_idx)
    pr = np.ascontiguousarray(pairs, dtype=np.uint64).reshape(-1, 2)
    out = np.empty(max(pr.shape[0], 1), dtype=np.float64)
    _check(lib().oracle_pair_similarity(_p(rp), _p(ci), rp.size - 1, _p(pr), pr.shape[0],
                                        0 if metric == "jaccard" else 1, _p(out)), "pair_similarity")
    return out[:pr.shape[0]]


def bruteforce_topk(row_ptr, col_idx, queries, k: int, metric: str = "jaccard", exclude_self=True):
    rp, ci = _csr(row_ptr, col_idx)
    q = np.ascontiguousarray(queries, dtype=np.uint64)
    ids = np.empty((max(q.size, 1), k), dtype=np.uint32)
    sim = np.empty((max(q.size, 1), k), dtype=np.float64)
    _check(lib().oracle_bruteforce_topk(_p(rp), _p(ci), rp.size - 1, _p(q), q.size, k,
                                        0 if metric == "jaccard" else 1, 1 if exclude_self else 0,
                                        _p(ids), _p(sim)), "bruteforce_topk")
    return ids[:q.size], sim[:q.size]
