"""One scan launch of a synthetic trace, for ncu: tools/one_launch.py <all_distinct|config2> <scan mode> [packets]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11449_b200 as P  # noqa: E402

kind, mode = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 64_000_000
if kind == "all_distinct":
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    cand = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
    opp = torch.randint(-2 ** 31, 2 ** 31 - 1, (n,), device="cuda", generator=g, dtype=torch.int64).to(torch.int32)
else:
    import bench
    c_np, o_np, *_ = bench.make_window(100, n, 0)
    cand, opp = torch.from_numpy(c_np.view(np.int32)).cuda(), torch.from_numpy(o_np.view(np.int32)).cuda()
sk = P.Dhla(P.DhgParams())
sk.set_scan_mode(mode)
for rep in range(2):
    sk.reset()
    sk.update_batch(cand, opp)
    sk.seal()
print(kind, mode, n, sk.scan_mode_used, sk.flow_cache_stats())
