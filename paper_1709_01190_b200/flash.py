"""ctypes binding for libflash.so (include/flash.h) — argument marshalling only.

Every function here has the same name as the C-ABI entry point it wraps and only
converts torch tensors / numpy arrays to pointers and sizes; all steps of FLASH's
hot path run in the library's sm_100a kernels.  There is no CPU fallback: if
``libflash.so`` is missing or no CUDA device is visible, calls raise.

Tensors: CSR ``row_ptr`` int64 [n+1], ``col_idx`` int32 [nnz] (reinterpreted as
uint32; col ids >= 2^31 are stored as their two's-complement int32 bit pattern),
addresses / ids / counts int32 [n, L] / [n, k] holding uint32 bit patterns
(``as_u32`` converts to numpy uint32).  ``stream`` defaults to torch's current
stream on the tensors' device.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libflash.so")
EMPTY = 0xFFFFFFFF

FLASH_OK, FLASH_EINVAL, FLASH_ENOMEM, FLASH_ECUDA, FLASH_ENCCL, FLASH_ESTATE = range(6)
_NAMES = {1: "FLASH_EINVAL", 2: "FLASH_ENOMEM", 3: "FLASH_ECUDA", 4: "FLASH_ENCCL", 5: "FLASH_ESTATE"}

# Every symbol include/flash.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "flash_create", "flash_destroy", "flash_hash", "flash_insert", "flash_insert_addrs",
    "flash_query_topk", "flash_query_addrs", "flash_knn_graph", "flash_knn_graph_host",
    "flash_get_table", "flash_clear", "flash_check", "flash_insert_addrs_window",
    "flash_table_arrays", "flash_import_tables", "flash_set_profiling", "flash_phase_ms",
    "flash_launch_count", "flash_reset_counters", "flash_last_error",
    "flash_hash_blocked", "flash_insert_addrs_cols", "flash_window_sizes", "flash_window_gather",
    "flash_count_topk", "flash_create_pool", "flash_get_unique_id", "flash_create_dist",
    "flash_create_dist_local", "flash_dist_info",
)
UNIQUE_ID_BYTES = 128


class FlashError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libflash.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run __graft_entry__.build() (no CPU fallback exists)")
    L = ctypes.CDLL(path)
    vp, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    L.flash_create.argtypes = [u32, u32, u32, u32, u64, ctypes.POINTER(vp)]
    L.flash_create_pool.argtypes = [u32, u32, u32, u32, u64, u64, ctypes.POINTER(vp)]
    L.flash_destroy.argtypes = [vp]
    L.flash_destroy.restype = None
    L.flash_hash.argtypes = [vp, vp, vp, u64, vp, vp, vp]
    L.flash_insert.argtypes = [vp, vp, vp, u64, u32, vp]
    L.flash_insert_addrs.argtypes = [vp, vp, u64, u32, vp]
    L.flash_query_topk.argtypes = [vp, vp, vp, u64, u32, vp, vp, vp, vp]
    L.flash_query_addrs.argtypes = [vp, vp, u64, u32, vp, vp, vp, vp]
    L.flash_knn_graph.argtypes = [vp, vp, vp, u64, u32, vp, vp, vp]
    L.flash_knn_graph_host.argtypes = [vp, vp, vp, u64, u32, vp, vp, vp]
    L.flash_get_table.argtypes = [vp, u32, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                  ctypes.POINTER(u64)]
    L.flash_check.argtypes = [vp, ctypes.POINTER(u64)]
    L.flash_clear.argtypes = [vp, vp]
    L.flash_insert_addrs_window.argtypes = [vp, vp, u64, u32, u32, u32, vp]
    L.flash_table_arrays.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                     ctypes.POINTER(u64)]
    L.flash_import_tables.argtypes = [vp, vp, vp, u64, vp, vp]
    L.flash_set_profiling.argtypes = [vp, i32]
    L.flash_phase_ms.argtypes = [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(u64)]
    L.flash_launch_count.argtypes = [vp]
    L.flash_launch_count.restype = u64
    L.flash_reset_counters.argtypes = [vp]
    L.flash_hash_blocked.argtypes = [vp, vp, vp, u64, u32, vp, vp]
    L.flash_insert_addrs_cols.argtypes = [vp, vp, u64, u32, u32, u32, vp]
    L.flash_window_sizes.argtypes = [vp, vp, u64, u32, u32, vp, vp, vp]
    L.flash_window_gather.argtypes = [vp, vp, u64, u32, u32, vp, vp, vp]
    L.flash_count_topk.argtypes = [vp, vp, vp, u32, u64, u32, vp, u32, vp, vp, vp]
    L.flash_get_unique_id.argtypes = [vp]
    L.flash_create_dist.argtypes = [u32, u32, u32, u32, u64, i32, i32, vp, ctypes.POINTER(vp)]
    L.flash_create_dist_local.argtypes = [u32, u32, u32, u32, u64, i32, vp, vp]
    L.flash_dist_info.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(u32),
                                  ctypes.POINTER(u32)]
    L.flash_last_error.argtypes = []
    L.flash_last_error.restype = ctypes.c_char_p
    for name in EXPORTS:
        f = getattr(L, name)
        if name not in ("flash_destroy", "flash_launch_count", "flash_last_error"):
            f.restype = i32
    _lib = L
    return L


def _check(st: int):
    if st != FLASH_OK:
        raise FlashError(st, load_library().flash_last_error().decode())


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return t.ctypes.data
    return int(t)


def _stream(stream, ref: torch.Tensor | None = None) -> int | None:
    if stream is None:
        dev = ref.device if isinstance(ref, torch.Tensor) and ref.is_cuda else torch.device("cuda", torch.cuda.current_device())
        return torch.cuda.current_stream(dev).cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def as_u32(t) -> np.ndarray:
    """int32 tensor/array holding uint32 bit patterns -> numpy uint32."""
    if isinstance(t, torch.Tensor):
        t = t.detach().cpu().numpy()
    return np.ascontiguousarray(t).view(np.uint32)


def to_device_csr(row_ptr, col_idx, device="cuda"):
    """numpy CSR (int64, uint32) -> torch CUDA tensors (int64, int32 bit patterns)."""
    rp = torch.from_numpy(np.ascontiguousarray(row_ptr, dtype=np.int64)).to(device)
    ci_np = np.ascontiguousarray(col_idx, dtype=np.uint32)
    if ci_np.size == 0:
        ci_np = np.zeros(1, np.uint32)
    ci = torch.from_numpy(ci_np.view(np.int32)).to(device)
    return rp, ci


# ---------------------------------------------------------------------------
# C-ABI wrappers (same names)
# ---------------------------------------------------------------------------

def flash_create(K: int, L: int, R: int, range_: int, seed: int) -> int:
    torch.cuda.current_device()  # make sure the CUDA context exists
    h = ctypes.c_void_p()
    _check(load_library().flash_create(K, L, R, range_, seed & 0xFFFFFFFFFFFFFFFF, ctypes.byref(h)))
    return h.value


def flash_create_pool(K: int, L: int, R: int, range_: int, pool: int, seed: int) -> int:
    torch.cuda.current_device()
    h = ctypes.c_void_p()
    _check(load_library().flash_create_pool(K, L, R, range_, pool, seed & 0xFFFFFFFFFFFFFFFF, ctypes.byref(h)))
    return h.value


def pool_size(F: float, L: int, range_: int) -> int:
    """P = ceil(F * L * range) shared reservoirs ("Allocated Range = F * Actual Range")."""
    import math
    return max(1, min(L * range_, int(math.ceil(F * L * range_))))


def flash_destroy(h: int) -> None:
    load_library().flash_destroy(h)


def flash_hash(h, row_ptr, col_idx, n_rows, codes=None, addrs=None, stream=None):
    _check(load_library().flash_hash(h, _ptr(row_ptr), _ptr(col_idx), n_rows, _ptr(codes), _ptr(addrs),
                                     _stream(stream, row_ptr)))


def flash_insert(h, row_ptr, col_idx, n_rows, id_base=0, stream=None):
    _check(load_library().flash_insert(h, _ptr(row_ptr), _ptr(col_idx), n_rows, id_base, _stream(stream, row_ptr)))


def flash_insert_addrs(h, addrs, n_rows, id_base=0, stream=None):
    _check(load_library().flash_insert_addrs(h, _ptr(addrs), n_rows, id_base, _stream(stream, addrs)))


def flash_query_topk(h, row_ptr, col_idx, n_q, k, exclude, out_ids, out_counts, stream=None):
    _check(load_library().flash_query_topk(h, _ptr(row_ptr), _ptr(col_idx), n_q, k, _ptr(exclude),
                                           _ptr(out_ids), _ptr(out_counts), _stream(stream, row_ptr)))


def flash_query_addrs(h, addrs, n_q, k, exclude, out_ids, out_counts, stream=None):
    _check(load_library().flash_query_addrs(h, _ptr(addrs), n_q, k, _ptr(exclude), _ptr(out_ids),
                                            _ptr(out_counts), _stream(stream, addrs)))


def flash_knn_graph(h, row_ptr, col_idx, n_rows, k, out_ids, out_counts, stream=None):
    _check(load_library().flash_knn_graph(h, _ptr(row_ptr), _ptr(col_idx), n_rows, k, _ptr(out_ids),
                                          _ptr(out_counts), _stream(stream, row_ptr)))


def flash_knn_graph_host(h, row_ptr, col_idx, n_rows, k, out_ids, out_counts, stream=None):
    """Host buffers in and out (numpy or pinned CPU tensors); synchronizes."""
    _check(load_library().flash_knn_graph_host(h, _ptr(row_ptr), _ptr(col_idx), n_rows, k, _ptr(out_ids),
                                               _ptr(out_counts), _stream(stream)))


def flash_get_table(h, t: int):
    """(off, ids, arrivals) device pointers and n_ids for table t."""
    off, ids, arr = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    n = ctypes.c_uint64()
    _check(load_library().flash_get_table(h, t, ctypes.byref(off), ctypes.byref(ids), ctypes.byref(arr),
                                          ctypes.byref(n)))
    return off.value, ids.value, arr.value, n.value


def flash_insert_addrs_window(h, addrs, n_rows, id_base, t_begin, t_end, stream=None):
    _check(load_library().flash_insert_addrs_window(h, _ptr(addrs), n_rows, id_base, t_begin, t_end,
                                                    _stream(stream, addrs)))


def flash_table_arrays(h):
    """(goff, ids, arrivals) device pointers and the total number of kept ids."""
    g, i, a = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    n = ctypes.c_uint64()
    _check(load_library().flash_table_arrays(h, ctypes.byref(g), ctypes.byref(i), ctypes.byref(a), ctypes.byref(n)))
    return g.value, i.value, a.value, n.value


def flash_import_tables(h, goff, ids, n_ids, arrivals, stream=None):
    _check(load_library().flash_import_tables(h, _ptr(goff), _ptr(ids), n_ids, _ptr(arrivals),
                                              _stream(stream, goff)))


def flash_get_unique_id() -> bytes:
    """NCCL bootstrap id (FLASH_UNIQUE_ID_BYTES) for flash_create_dist; rank 0 makes it."""
    buf = ctypes.create_string_buffer(UNIQUE_ID_BYTES)
    _check(load_library().flash_get_unique_id(buf))
    return buf.raw


def flash_create_dist(K: int, L: int, R: int, range_: int, seed: int, rank: int, world: int,
                      unique_id: bytes) -> int:
    """Collective: rank `rank` of a multi-GPU handle on the current device (NCCL)."""
    torch.cuda.current_device()
    if len(unique_id) != UNIQUE_ID_BYTES:
        raise ValueError(f"unique_id must be {UNIQUE_ID_BYTES} bytes")
    buf = ctypes.create_string_buffer(bytes(unique_id), UNIQUE_ID_BYTES)
    h = ctypes.c_void_p()
    _check(load_library().flash_create_dist(K, L, R, range_, seed & 0xFFFFFFFFFFFFFFFF, rank, world, buf,
                                            ctypes.byref(h)))
    return h.value


def flash_create_dist_local(K: int, L: int, R: int, range_: int, seed: int, world: int,
                            devices=None) -> list[int]:
    """`world` virtual ranks in this process (devices: list of device indices, or None = the
    current device for every rank).  Each rank's collective calls come from its own thread."""
    torch.cuda.current_device()
    hs = (ctypes.c_void_p * world)()
    dev = (ctypes.c_int * world)(*devices) if devices is not None else None
    _check(load_library().flash_create_dist_local(K, L, R, range_, seed & 0xFFFFFFFFFFFFFFFF, world,
                                                  dev, hs))
    return [hs[g] for g in range(world)]


def flash_dist_info(h):
    """(rank, world, t_begin, t_end) of a handle."""
    r, w = ctypes.c_int(), ctypes.c_int()
    t0, t1 = ctypes.c_uint32(), ctypes.c_uint32()
    _check(load_library().flash_dist_info(h, ctypes.byref(r), ctypes.byref(w), ctypes.byref(t0), ctypes.byref(t1)))
    return r.value, w.value, t0.value, t1.value


def flash_hash_blocked(h, row_ptr, col_idx, n_rows, world, addrs, stream=None):
    _check(load_library().flash_hash_blocked(h, _ptr(row_ptr), _ptr(col_idx), n_rows, world, _ptr(addrs),
                                             _stream(stream, row_ptr)))


def flash_insert_addrs_cols(h, addrs, n_rows, id_base, t_begin, t_end, stream=None):
    _check(load_library().flash_insert_addrs_cols(h, _ptr(addrs), n_rows, id_base, t_begin, t_end,
                                                  _stream(stream, addrs)))


def flash_window_sizes(h, addrs, n_q, t_begin, t_end, sizes, offsets, stream=None):
    _check(load_library().flash_window_sizes(h, _ptr(addrs), n_q, t_begin, t_end, _ptr(sizes), _ptr(offsets),
                                             _stream(stream, offsets)))


def flash_window_gather(h, addrs, n_q, t_begin, t_end, offsets, out_ids, stream=None):
    _check(load_library().flash_window_gather(h, _ptr(addrs), n_q, t_begin, t_end, _ptr(offsets), _ptr(out_ids),
                                              _stream(stream, offsets)))


def flash_count_topk(h, cand, seg_sizes, n_seg, n_q, k, exclude, max_id, out_ids, out_counts, stream=None):
    _check(load_library().flash_count_topk(h, _ptr(cand), _ptr(seg_sizes), n_seg, n_q, k, _ptr(exclude), max_id,
                                           _ptr(out_ids), _ptr(out_counts), _stream(stream, seg_sizes)))


def flash_clear(h, stream=None):
    _check(load_library().flash_clear(h, _stream(stream)))


def flash_check(h) -> int:
    n = ctypes.c_uint64()
    _check(load_library().flash_check(h, ctypes.byref(n)))
    return n.value


def flash_set_profiling(h, enable: bool):
    _check(load_library().flash_set_profiling(h, 1 if enable else 0))


def flash_phase_ms(h):
    ms = (ctypes.c_double * 4)()
    calls = (ctypes.c_uint64 * 4)()
    _check(load_library().flash_phase_ms(h, ms, calls))
    return list(ms), list(calls)


def flash_launch_count(h) -> int:
    return int(load_library().flash_launch_count(h))


def flash_reset_counters(h):
    _check(load_library().flash_reset_counters(h))


def flash_last_error() -> str:
    return load_library().flash_last_error().decode()


# ---------------------------------------------------------------------------
# Convenience object
# ---------------------------------------------------------------------------

class _DeviceArray:
    """Zero-copy view of library-owned device memory (CUDA array interface)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<i4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 2, "strides": None}


def _copy_device(ptr: int, n: int, device, typestr: str = "<i4") -> torch.Tensor:
    dt = torch.int64 if typestr == "<i8" else torch.int32
    if n == 0:
        return torch.empty(0, dtype=dt, device=device)
    return torch.as_tensor(_DeviceArray(ptr, n, typestr), device=device).clone()


class FlashIndex:
    """Owns one flash_index handle (device = the current CUDA device)."""

    def __init__(self, K: int, L: int, R: int, range_: int, seed: int, F: float = 1.0, pool: int | None = None,
                 handle: int | None = None):
        """F < 1 (or an explicit pool < L*range): reservoir sharing over a pool of
        ceil(F*L*range) reservoirs (R#23).  handle: adopt an existing handle (e.g. a
        multi-GPU rank from flash_create_dist / dist.create_dist_index)."""
        self.K, self.L, self.R, self.range, self.seed = K, L, R, range_, seed
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.pool = int(pool) if pool is not None else (pool_size(F, L, range_) if F < 1.0 else L * range_)
        if handle is not None:
            self.h = handle
        else:
            self.h = (flash_create_pool(K, L, R, range_, self.pool, seed) if self.pool < L * range_
                      else flash_create(K, L, R, range_, seed))

    def dist_info(self):
        """(rank, world, t_begin, t_end): this handle's rank and table window."""
        return flash_dist_info(self.h)

    def close(self):
        if getattr(self, "h", None):
            flash_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def hash(self, row_ptr, col_idx, codes=True, addrs=True):
        n = row_ptr.numel() - 1
        c = torch.empty((n, self.K * self.L), dtype=torch.int32, device=self.device) if codes else None
        a = torch.empty((n, self.L), dtype=torch.int32, device=self.device) if addrs else None
        flash_hash(self.h, row_ptr, col_idx, n, c, a)
        return c, a

    def hash_addrs(self, row_ptr, col_idx):
        return self.hash(row_ptr, col_idx, codes=False)[1]

    def insert(self, row_ptr, col_idx, id_base=0, stream=None):
        flash_insert(self.h, row_ptr, col_idx, row_ptr.numel() - 1, id_base, stream)

    def insert_addrs(self, addrs, id_base=0):
        flash_insert_addrs(self.h, addrs, addrs.shape[0], id_base)

    def query(self, row_ptr, col_idx, k, exclude=None, stream=None):
        n = row_ptr.numel() - 1
        ids = torch.empty((max(n, 1), k), dtype=torch.int32, device=self.device)[:n]
        cnt = torch.empty((max(n, 1), k), dtype=torch.int32, device=self.device)[:n]
        flash_query_topk(self.h, row_ptr, col_idx, n, k, exclude, ids, cnt, stream)
        return ids, cnt

    def query_addrs(self, addrs, k, exclude=None):
        n = addrs.shape[0]
        ids = torch.empty((n, k), dtype=torch.int32, device=self.device)
        cnt = torch.empty((n, k), dtype=torch.int32, device=self.device)
        flash_query_addrs(self.h, addrs, n, k, exclude, ids, cnt)
        return ids, cnt

    def knn_graph(self, row_ptr, col_idx, k, stream=None):
        n = row_ptr.numel() - 1
        ids = torch.empty((max(n, 1), k), dtype=torch.int32, device=self.device)[:n]
        cnt = torch.empty((max(n, 1), k), dtype=torch.int32, device=self.device)[:n]
        flash_knn_graph(self.h, row_ptr, col_idx, n, k, ids, cnt, stream)
        return ids, cnt

    def table(self, t: int):
        """(off, ids, arrivals) of table t as numpy uint32 (synchronizes)."""
        off_p, ids_p, arr_p, n = flash_get_table(self.h, t)
        off = _copy_device(off_p, self.range + 1, self.device)
        ids = _copy_device(ids_p, n, self.device)
        arr = _copy_device(arr_p, self.range, self.device)
        return as_u32(off), as_u32(ids), as_u32(arr)

    def clear(self):
        flash_clear(self.h)

    def insert_addrs_window(self, addrs, id_base, t_begin, t_end):
        flash_insert_addrs_window(self.h, addrs, addrs.shape[0], id_base, t_begin, t_end)

    def table_arrays(self, ids: bool = True):
        """Copies of (goff int64 [L*range+1], ids int32 [n] (None unless ids), arrivals int32
        [L*range])."""
        g, i, a, n = flash_table_arrays(self.h)
        nb = self.pool
        return (_copy_device(g, nb + 1, self.device, "<i8"), _copy_device(i, n, self.device) if ids else None,
                _copy_device(a, nb, self.device))

    def import_tables(self, goff, ids, arrivals):
        flash_import_tables(self.h, goff, ids if ids.numel() else None, ids.numel(), arrivals)

    def errors(self) -> int:
        return flash_check(self.h)

    # ---- serialization ----
    FORMAT = "flash-b200-index-v1"

    def save(self, path: str):
        """Write the index (config + bucket offsets + kept ids + arrivals) to an .npz file."""
        goff, ids, arr = self.table_arrays()
        np.savez(path, format=self.FORMAT, K=self.K, L=self.L, R=self.R, range=self.range, seed=self.seed,
                 pool=self.pool, goff=goff.cpu().numpy(), ids=as_u32(ids), arrivals=as_u32(arr))

    @classmethod
    def load(cls, path: str) -> "FlashIndex":
        """Rebuild an index from save(): load(save(x)) answers queries and takes further
        inserts exactly like x (bottom-R is composable)."""
        z = np.load(path)
        if str(z["format"]) != cls.FORMAT:
            raise ValueError(f"{path}: not a {cls.FORMAT} file")
        K, L, R, rng, seed, pool = (int(z[k]) for k in ("K", "L", "R", "range", "seed", "pool"))
        idx = cls(K, L, R, rng, seed, pool=pool)
        dev = idx.device
        goff = torch.from_numpy(z["goff"].astype(np.int64)).to(dev)
        ids = torch.from_numpy(np.ascontiguousarray(z["ids"]).view(np.int32)).to(dev)
        arr = torch.from_numpy(np.ascontiguousarray(z["arrivals"]).view(np.int32)).to(dev)
        idx.import_tables(goff, ids, arr)
        return idx

    # ---- candidate exchange (dist.knn_graph_candidate_exchange) ----
    def hash_addrs_blocked(self, row_ptr, col_idx, world: int):
        """Addresses of the rows, owner-blocked for `world` table windows (flat int32 [n*L])."""
        n = row_ptr.numel() - 1
        a = torch.empty(n * self.L, dtype=torch.int32, device=self.device)
        flash_hash_blocked(self.h, row_ptr, col_idx, n, world, a)
        return a

    def insert_addrs_cols(self, addrs, id_base, t_begin, t_end):
        flash_insert_addrs_cols(self.h, addrs, addrs.shape[0], id_base, t_begin, t_end)

    def window_sizes(self, addrs, t_begin, t_end):
        """(sizes int32 [n], offsets int64 [n+1]) of the window's candidates per query."""
        n = addrs.shape[0]
        sizes = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)[:n]
        off = torch.empty(n + 1, dtype=torch.int64, device=self.device)
        flash_window_sizes(self.h, addrs, n, t_begin, t_end, sizes, off)
        return sizes, off

    def window_gather(self, addrs, t_begin, t_end, offsets, total: int):
        out = torch.empty(max(total, 1), dtype=torch.int32, device=self.device)
        flash_window_gather(self.h, addrs, addrs.shape[0], t_begin, t_end, offsets, out)
        return out[:total]

    def count_topk(self, cand, seg_sizes, k, max_id: int, exclude=None):
        """seg_sizes int32 [n_seg, n_q]; cand int32 in (segment, query) order; max_id bounds
        the candidate ids (it sets the sort's digit range: pass the real bound)."""
        n_seg, n_q = seg_sizes.shape
        ids = torch.empty((n_q, k), dtype=torch.int32, device=self.device)
        cnt = torch.empty((n_q, k), dtype=torch.int32, device=self.device)
        flash_count_topk(self.h, cand if cand.numel() else None, seg_sizes.contiguous(), n_seg, n_q, k,
                         exclude, int(max_id), ids, cnt)
        return ids, cnt
