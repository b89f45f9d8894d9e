"""Per-phase cycle breakdown of the warp-per-query kernel (diagnostic build libflash_qprof.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

lib = flash.load_library(os.path.join(os.path.dirname(flash.LIB_PATH), "libflash_qprof.so"))
shape = synth.SHAPES["webspam"]
K, L, R, rng, seed, k = 4, 50, 128, 1 << 15, 0x5EED0002, 128
rp, col = synth.generate(shape)
d_rp, d_col = flash.to_device_csr(rp, col)
idx = flash.FlashIndex(K, L, R, rng, seed)
ids = torch.empty((shape.N, k), dtype=torch.int32, device="cuda")
cnt = torch.empty_like(ids)
buf = (ctypes.c_ulonglong * 8)()
for rep in range(2):
    lib.flash_debug_qprof(buf, 1)
    idx.clear()
    flash.flash_knn_graph(idx.h, d_rp, d_col, shape.N, k, ids, cnt)
    torch.cuda.synchronize()
lib.flash_debug_qprof(buf, 0)
names = ["Q1 segments", "Q2 insert", "Q3a threshold", "Q3b collect", "Q3c radix+append", "clear", "sort+write"]
tot = sum(buf[i] for i in range(7))
for i, nm in enumerate(names):
    print(f"{nm:18s} {buf[i] / shape.N:10.0f} cycles/query  {100 * buf[i] / tot:5.1f}%")
print(f"total {tot / shape.N:.0f} cycles/query (per warp, summed over phases)")
