"""bench.py's data / quality statistics (pairwise cosine, 1-NN cosine, R@k,
S@k of P:391-395) against a brute force written out with Python sets (CPU, small)."""
import numpy as np
import torch

import bench
import synth


def _cos(rows, a, b):
    return len(rows[a] & rows[b]) / np.sqrt(len(rows[a]) * len(rows[b]))


def test_quality_stats_match_brute_force():
    shape = synth.SHAPES["tiny"].with_(N=300)
    rp, col = synth.generate(shape)
    n = rp.size - 1
    rows = [set(col[rp[i]:rp[i + 1]].tolist()) for i in range(n)]
    rng = np.random.default_rng(1)
    k = 10
    out = rng.integers(0, n, size=(n, k)).astype(np.int32)
    out[:, -2:] = -1  # pads
    for q in range(0, n, 3):  # plant the true 1-NN first for a third of the rows
        c = [(_cos(rows, q, j), -j) for j in range(n) if j != q]
        out[q, 0] = -max(c)[1]
    res = bench.data_quality_stats(torch.from_numpy(rp), torch.from_numpy(col.view(np.int32)),
                                   torch.from_numpy(out), n_q=60, n_pairs=1500)
    r2 = np.random.default_rng(13)
    pa, pb = r2.integers(0, n, 1500), r2.integers(0, n, 1500)
    ok = pa != pb
    want_pair = np.mean([_cos(rows, a, b) for a, b in zip(pa[ok], pb[ok])])
    assert abs(res["pairwise_cosine_mean"] - want_pair) < 1e-9
    qs = r2.choice(n, size=60, replace=False)
    r_at, s_at, best_sum = {1: 0, 10: 0}, {1: 0.0, 10: 0.0}, 0.0
    for q in qs:
        c = np.array([_cos(rows, q, j) if j != q else -1.0 for j in range(n)])
        best = c.max()
        best_sum += best
        for kk in (1, 10):
            ids = [i for i in out[q, :kk] if i >= 0]
            r_at[kk] += any(c[i] >= best - 1e-9 for i in ids)
            s_at[kk] += np.mean([c[i] for i in ids]) if ids else 0.0
    assert abs(res["one_nn_cosine_mean"] - best_sum / 60) < 1e-9
    for kk in (1, 10):
        assert abs(res["quality"]["R@k"][str(kk)] - r_at[kk] / 60) < 1e-12
        assert abs(res["quality"]["S@k"][str(kk)] - s_at[kk] / 60) < 1e-9
    assert res["quality"]["R@k"]["1"] > 0.2  # the planted neighbours are found


def test_bench_entry_points_exist():
    """bench.py's driver contract: every arm main() dispatches to is defined."""
    for fn in ("run_ours", "run_shape", "run_reference", "cpu_baseline", "main", "data_quality_stats",
               "exact_cosine", "recall_at_k", "shape_stats"):
        assert callable(getattr(bench, fn)), fn
