"""Seeded synthetic CSR inputs shared by the oracle tests and the CUDA path.

This module holds none of FLASH's arithmetic (no DOPH, no address map, no
priority hash): it only produces sparse binary rows.  The bulk generator is
``synth/gen.c`` (PCG32 streams, OpenMP over rows, deterministic per row);
small edge-case builders are plain numpy.  Recipe and per-shape parameters:
DESIGN.md "Inputs" (after SURVEY.md §8(d), shapes from PAPER.md Table 1,
P:413-419).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")


class _Params(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_uint64),
        ("D", ctypes.c_uint64),
        ("mean_nnz", ctypes.c_double),
        ("sigma", ctypes.c_double),
        ("f_core", ctypes.c_double),
        ("V_c", ctypes.c_uint64),
        ("fam_min", ctypes.c_uint32),
        ("fam_extra", ctypes.c_double),
        ("mu_f", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("shuffle", ctypes.c_int32),
    ]


@dataclass(frozen=True)
class Shape:
    """Generator parameters (Table 1 P:413-419 for N, D, nnz)."""

    name: str
    N: int
    D: int
    mean_nnz: float
    sigma: float
    f_core: float
    V_c: int
    fam_min: int
    fam_extra: float
    mu_f: float
    seed: int
    shuffle: bool = True

    def with_(self, **kw) -> "Shape":
        return replace(self, **kw)


SHAPES = {
    # tiny: planted families, 1-NN cos ~0.8, background ~0.01
    "tiny": Shape("tiny", 1_000, 1 << 20, 100.0, 0.3, 0.1, 100, 1, 4.0, 0.1, 1),
    # webspam: 350K x 16.6M dims, 3,728 nnz/row, pairwise cos 0.33 (Table 1), 1-NN
    # 0.972: f_core / V_c calibrated by tools/calibrate_webspam.py (0.331 over 2e4 pairs),
    # mu_f = 1 - 0.972 (a row's 1-NN is its family root or member at cosine ~1 - mu_f)
    "webspam": Shape("webspam", 350_000, 16_609_143, 3728.0, 0.6, 0.58, 2600, 2, 1.0, 0.028, 2),
    # url: 2.39M x 3.23M dims, 116 nnz/row
    "url": Shape("url", 2_386_130, 3_231_961, 116.0, 0.4, 0.85, 129, 2, 1.0, 0.015, 3),
    # kdd12: 149.6M x 54.7M dims, 11 nnz/row
    "kdd12": Shape("kdd12", 149_629_105, 54_686_452, 11.0, 0.3, 0.5, 18, 1, 1.0, 0.1, 4),
    # friendster: 65.6M users x 65.6M dims (friend lists), 27.5 nnz/row, pairwise cos ~0;
    # heavy-tailed degrees (sigma 1.0), families of users with similar friend sets (mu_f 0.3)
    "friendster": Shape("friendster", 65_608_366, 65_608_366, 27.5, 1.0, 0.05, 1000, 1, 1.0, 0.3, 5),
}


def build_lib(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"]
        )
    return _SO


_lib = None


def _load():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_SO)
        P = ctypes.POINTER(_Params)
        u64 = ctypes.c_uint64
        vp = ctypes.c_void_p
        lib.synth_row_lengths.argtypes = [P, u64, u64, vp]
        lib.synth_fill.argtypes = [P, u64, u64, vp, vp]
        lib.synth_family_of.argtypes = [P, u64, u64, vp]
        for f in (lib.synth_row_lengths, lib.synth_fill, lib.synth_family_of):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _cparams(s: Shape) -> _Params:
    return _Params(s.N, s.D, s.mean_nnz, s.sigma, s.f_core, s.V_c, s.fam_min,
                   s.fam_extra, s.mu_f, s.seed, 1 if s.shuffle else 0)


def generate(shape: Shape | str, rows: tuple[int, int] | None = None,
             row_ptr_out: np.ndarray | None = None, col_out: np.ndarray | None = None):
    """CSR (row_ptr int64[n+1] starting at 0, col_idx uint32[nnz]) for final rows
    [r0, r1) of `shape` (all rows by default).  Optional preallocated (e.g. pinned)
    output arrays may be passed; col_out must hold at least nnz entries."""
    s = SHAPES[shape] if isinstance(shape, str) else shape
    r0, r1 = rows if rows is not None else (0, s.N)
    n = r1 - r0
    lib = _load()
    p = _cparams(s)
    lens = np.empty(n, dtype=np.int64)
    if lib.synth_row_lengths(ctypes.byref(p), r0, r1, lens.ctypes.data) != 0:
        raise ValueError("synth_row_lengths: bad parameters")
    row_ptr = row_ptr_out if row_ptr_out is not None else np.empty(n + 1, dtype=np.int64)
    row_ptr[0] = 0
    np.cumsum(lens, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = col_out if col_out is not None else np.empty(nnz, dtype=np.uint32)
    assert col.dtype == np.uint32 and col.size >= nnz
    if lib.synth_fill(ctypes.byref(p), r0, r1, row_ptr.ctypes.data, col.ctypes.data) != 0:
        raise ValueError("synth_fill: bad parameters")
    return row_ptr, col[:nnz]


def family_of(shape: Shape | str, rows: tuple[int, int] | None = None) -> np.ndarray:
    s = SHAPES[shape] if isinstance(shape, str) else shape
    r0, r1 = rows if rows is not None else (0, s.N)
    out = np.empty(r1 - r0, dtype=np.uint64)
    if _load().synth_family_of(ctypes.byref(_cparams(s)), r0, r1, out.ctypes.data) != 0:
        raise ValueError("synth_family_of: bad parameters")
    return out


# ---------------------------------------------------------------------------
# Small hand-built edge cases (numpy only)
# ---------------------------------------------------------------------------

def csr_from_rows(rows) -> tuple[np.ndarray, np.ndarray]:
    lens = np.array([len(r) for r in rows], dtype=np.int64)
    row_ptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    col = np.concatenate([np.asarray(r, dtype=np.uint32) for r in rows]) if rows and lens.sum() else np.zeros(0, np.uint32)
    return row_ptr, col.astype(np.uint32)


def edge_case_rows(seed: int = 7) -> list[np.ndarray]:
    """Rows exercising the hot path's degenerate cases (SURVEY §4 edge matrix):
    empty rows, 1-nnz rows, duplicate and permuted col indices, col ids near
    2^32-1, identical rows, a row longer than one warp tile, 2-nnz rows."""
    rng = np.random.default_rng(seed)
    rows: list[np.ndarray] = []
    rows.append(np.zeros(0, np.uint32))                                   # empty
    rows.append(np.array([5], np.uint32))                                 # 1 nnz
    rows.append(np.array([0xFFFFFFFE], np.uint32))                        # max legal col
    rows.append(np.array([0xFFFFFFFE, 0xFFFFFFF0, 3, 3, 3], np.uint32))   # dupes + high ids
    base = rng.choice(1 << 20, size=300, replace=False).astype(np.uint32)
    rows.append(base.copy())
    rows.append(base[::-1].copy())                                        # permuted copy
    rows.append(np.concatenate([base, base[:50]]))                        # duplicated entries
    rows.append(rng.integers(0, 1 << 32 - 1, size=1_000_000, dtype=np.uint64).astype(np.uint32))  # 10^6-nnz row
    rows.append(np.zeros(0, np.uint32))                                   # another empty
    for _ in range(6):
        rows.append(base.copy())                                          # identical rows
    for _ in range(20):
        rows.append(rng.choice(1 << 20, size=int(rng.integers(1, 40)), replace=False).astype(np.uint32))
    rows.append(np.array([1, 2], np.uint32))
    return rows
