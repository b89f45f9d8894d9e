"""Per-phase cycle breakdown of the warp-per-query sort kernel (diagnostic build
libflash_qprof.so from `python -m paper_1709_01190_b200.build --qprof`)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

VARIANT = sys.argv[1] if len(sys.argv) > 1 else "qprof"  # "product" = libflash.so (timing only)
lib = flash.load_library(flash.LIB_PATH if VARIANT == "product" else
                         os.path.join(os.path.dirname(flash.LIB_PATH), f"libflash_{VARIANT}.so"))
shape = synth.SHAPES["webspam"]
K, L, R, rng, seed, k = 4, 50, 128, 1 << 15, 0x5EED0002, 128
rp, col = synth.generate(shape)
d_rp, d_col = flash.to_device_csr(rp, col)
idx = flash.FlashIndex(K, L, R, rng, seed)
ids = torch.empty((shape.N, k), dtype=torch.int32, device="cuda")
cnt = torch.empty_like(ids)
buf = (ctypes.c_ulonglong * 8)()
prof = hasattr(lib, "flash_debug_qprof")
mbuf = (ctypes.c_ulonglong * 8)()
lib.flash_set_profiling(idx.h, 1)
for rep in range(3):
    if prof:
        lib.flash_debug_qprof(buf, 1)
        lib.flash_debug_mprof(mbuf, 1)
    idx.clear()
    flash.flash_knn_graph(idx.h, d_rp, d_col, shape.N, k, ids, cnt)
    torch.cuda.synchronize()
    if rep == 0:
        lib.flash_reset_counters(idx.h)
ph = (ctypes.c_double * 4)()
nc = (ctypes.c_uint64 * 4)()
lib.flash_phase_ms(idx.h, ph, nc)
print(VARIANT, "phase ms (mean of 2): " + " ".join(f"{n} {ph[i] / max(nc[i], 1):.3f}"
                                                  for i, n in enumerate(["hash", "build", "query"])))
if not prof:
    sys.exit(0)
lib.flash_debug_qprof(buf, 0)
lib.flash_debug_mprof(mbuf, 0)
# the bitmap kernel (query_mark.cu), consumer thread 0 of each CTA: cycles between its barriers
mnames = ["wait for Q1 (full barrier)", "Q2 gather+mark", "Q3a compact", "Q3c scan", "Q3b rank + pads",
          "reset"]
mtot = sum(mbuf[i] for i in range(6))
for i, nm in enumerate(mnames):
    print(f"mark {nm:22s} {mbuf[i] / shape.N:10.0f} cycles/query  {100 * mbuf[i] / max(mtot, 1):5.1f}%")
print(f"mark total {mtot / shape.N:.0f} cycles/query (per CTA; queries not on the bitmap path count 0)")
names = ["Q1 buckets", "Q2a count", "scan", "Q2b scatter", "bin sort", "Q3a runs", "Q3b/c select+write"]
tot = sum(buf[i] for i in range(7))
for i, nm in enumerate(names):
    print(f"{nm:20s} {buf[i] / shape.N:10.0f} cycles/query  {100 * buf[i] / tot:5.1f}%")
print(f"total {tot / shape.N:.0f} cycles/query (per warp)")
print(f"bin-sort passes per query {buf[7] / shape.N:.2f}")
