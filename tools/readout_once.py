"""A few read-outs of a config-2-like small window, for ncu: tools/readout_once.py [n_scanners]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11449_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
cand, opp = O.distinct_pairs(3_000_000, 14)
parts = [(cand, opp)] + [O.plant_pairs(2_000_000 + 7 * t, 2048 + 100 * (t % 50), 600 + t) for t in range(n)]
cand, opp = np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])
sk = P.Dhla(P.DhgParams())
sk.update_batch(cand, opp)
for rep in range(4):
    got = sk.restore_superpoints(1024)
print(len(got), sk.small_tail_used, sk.last_info["stage_counts"], sk.last_info["hot_counts"])
