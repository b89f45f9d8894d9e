"""Calibrate the webspam generator to Table 1's mean pairwise cosine (0.33) and the
1-NN cosine (0.972): mean binary cosine over random row pairs of a row sample, for
candidate core-vocabulary sizes V_c (evaluation only; prints a table)."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402


def pairwise_cos(shape, n_rows=20000, pairs=20000, seed=0):
    rp, col = synth.generate(shape, rows=(0, n_rows))
    rows = [np.unique(col[rp[i]:rp[i + 1]]) for i in range(n_rows)]
    rng = np.random.default_rng(seed)
    a, b = rng.integers(0, n_rows, pairs), rng.integers(0, n_rows, pairs)
    cs = []
    for i, j in zip(a, b):
        if i == j:
            continue
        x, y = rows[i], rows[j]
        inter = np.intersect1d(x, y, assume_unique=True).size
        cs.append(inter / np.sqrt(x.size * y.size))
    return float(np.mean(cs))


if __name__ == "__main__":
    base = synth.SHAPES["webspam"]
    for vc in [int(v) for v in sys.argv[1:]] or [2824, 2400, 2200, 2000]:
        print(vc, round(pairwise_cos(base.with_(V_c=vc)), 4), flush=True)


def grid(cands):
    base = synth.SHAPES["webspam"]
    for f, vc in cands:
        print(f, vc, round(pairwise_cos(base.with_(f_core=f, V_c=vc), n_rows=8000, pairs=8000), 4), flush=True)
