"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck): every
kernel family — dense and sparse DOPH, row-major and table-major builds, the small /
register / warp / CTA selects, the size-classed query kernels, and the multi-GPU
exchange steps (window gather, direct-segment count/top-k) on one GPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

CASES = [("tiny", 1000, (4, 16, 32, 1 << 15, 10), "0"),
         ("webspam", 300, (4, 50, 128, 1 << 12, 128), "0"),
         ("url", 3000, (4, 128, 32, 1 << 10, 128), "0"),
         ("url", 3000, (4, 64, 128, 1 << 6, 300), "1"),
         ("kdd12", 6000, (4, 32, 64, 1 << 7, 64), "1"),   # sparse DOPH, 33..256-member buckets
         ("tiny", 4000, (2, 4, 16, 64, 20), "0"),          # register-path select, m > R
         ("tiny", 3000, (4, 8, 64, 4, 10), "0")]           # > 512 members: early list, side stream

for ci, (name, n, (K, L, R, rng, k), tm) in enumerate(CASES):
    os.environ["FLASH_BUILD_TM"] = tm
    # query kernels: alternate the occupancy-bitmap kernel (with a forced fallback list on
    # every third case) and the size-class sort kernels
    os.environ["FLASH_QUERY_MARK"] = "1" if ci % 2 == 0 else "0"
    os.environ["FLASH_QUERY_MARK_MIN"] = "0" if ci % 4 == 0 else "64"
    os.environ["FLASH_QUERY_MARK_REPMAX"] = "2" if ci % 3 == 0 else "224"
    rp, col = synth.generate(synth.SHAPES[name].with_(N=n))
    rows = [col[rp[i]:rp[i + 1]] for i in range(n)] + synth.edge_case_rows()
    rp, col = synth.csr_from_rows(rows)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, 7) as idx:
        ids, cnt = idx.knn_graph(d_rp, d_col, k)
        idx.table(0)
        torch.cuda.synchronize()
    print(name, n, "mark" if ci % 2 == 0 else "sort", "ok", int(flash.as_u32(cnt).max()), flush=True)

# the exchange steps: 2 virtual ranks, each owning half of the tables
os.environ["FLASH_BUILD_TM"] = "0"
rp, col = synth.generate(synth.SHAPES["webspam"].with_(N=400))
d_rp, d_col = flash.to_device_csr(rp, col)
n, K, L, R, rng, k = 400, 4, 8, 16, 1 << 8, 32
parts = []
for t0, t1 in ((0, 4), (4, 8)):
    with flash.FlashIndex(K, L, R, rng, 7) as idx:
        blocked = idx.hash_addrs_blocked(d_rp, d_col, 2).view(-1)
        cols = blocked[n * t0: n * t1].view(n, t1 - t0).contiguous()
        idx.insert_addrs_cols(cols, 0, t0, t1)
        sz, off = idx.window_sizes(cols, t0, t1)
        parts.append((sz, idx.window_gather(cols, t0, t1, off, int(off[-1].item()))))
with flash.FlashIndex(K, L, R, rng, 7) as idx:
    seg = torch.stack([p[0] for p in parts])
    cand = torch.cat([p[1] for p in parts])
    excl = torch.arange(n, dtype=torch.int32, device="cuda")
    ids, cnt = idx.count_topk(cand, seg, k, n - 1, excl)
    torch.cuda.synchronize()
print("exchange ok", int(flash.as_u32(cnt).max()), flush=True)
