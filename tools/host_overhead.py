"""Host enqueue time vs device time of each API call (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

shape = synth.SHAPES["webspam"]
K, L, R, rng, seed, k = 4, 50, 128, 1 << 15, 0x5EED0002, 128
rp, col = synth.generate(shape)
d_rp, d_col = flash.to_device_csr(rp, col)
n = shape.N
idx = flash.FlashIndex(K, L, R, rng, seed)
ids = torch.empty((n, k), dtype=torch.int32, device="cuda")
cnt = torch.empty_like(ids)
addrs = torch.empty((n, L), dtype=torch.int32, device="cuda")
for rep in range(4):
    idx.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    flash.flash_hash(idx.h, d_rp, d_col, n, None, addrs)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    flash.flash_insert_addrs(idx.h, addrs, n, 0)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    flash.flash_query_addrs(idx.h, addrs, n, k, None, ids, cnt)
    t5 = time.perf_counter()
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    print(f"hash enq {1e3*(t1-t0):.3f} tot {1e3*(t2-t0):.3f} | insert enq {1e3*(t3-t2):.3f} tot {1e3*(t4-t2):.3f}"
          f" | query enq {1e3*(t5-t4):.3f} tot {1e3*(t6-t4):.3f} ms")
