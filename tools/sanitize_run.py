"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1709_01190_b200 import flash  # noqa: E402

CASES = [("tiny", 1000, (4, 16, 32, 1 << 15, 10)),
         ("webspam", 300, (4, 50, 128, 1 << 12, 128)),
         ("url", 3000, (4, 128, 32, 1 << 10, 128)),
         ("url", 3000, (4, 64, 128, 1 << 6, 300))]

for name, n, (K, L, R, rng, k) in CASES:
    rp, col = synth.generate(synth.SHAPES[name].with_(N=n))
    rows = [col[rp[i]:rp[i + 1]] for i in range(n)] + synth.edge_case_rows()
    rp, col = synth.csr_from_rows(rows)
    d_rp, d_col = flash.to_device_csr(rp, col)
    with flash.FlashIndex(K, L, R, rng, 7) as idx:
        ids, cnt = idx.knn_graph(d_rp, d_col, k)
        idx.table(0)
        torch.cuda.synchronize()
    print(name, n, "ok", int(flash.as_u32(cnt).max()), flush=True)
