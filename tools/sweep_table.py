"""Format a tools/sweep.py JSON result as the text table kept under profiles/.

    python tools/sweep_table.py profiles/r01_sweep.json > profiles/r01_sweep.txt
"""
import json
import sys

d = json.load(open(sys.argv[1]))
print("# webspam-shaped sweep (tools/sweep.py): full k-NN graph on 1 B200, k=128, range 2^15; "
      "R@k/S@k over 1000 sampled rows vs exact cosine")
print("# K  L    R    graph_ms  hash_ms build_ms query_ms  R@1    R@10   S@10   cand/q  cand/LR  q_frac_hbm")
for p in d["points"]:
    c = p.get("candidates_per_query", {})
    rf = p.get("query_roofline", {})
    print(f"{p['K']:2d} {p['L']:4d} {p['R']:4d} {p['graph_ms']:9.2f} {p['hash_ms']:8.2f} {p['build_ms']:8.2f} "
          f"{p['query_ms']:8.2f}  {p['R@k']['1']:.3f}  {p['R@k']['10']:.3f}  {p['S@k']['10']:.3f}  "
          f"{c.get('mean', float('nan')):7.0f}  {c.get('of_LR', float('nan')):6.3f}  {rf.get('frac', float('nan')):.4f}")
