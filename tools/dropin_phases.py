"""Phase times of the drop-in path (reference WindowSession holding the CUDA sketch, pageable numpy, 65,536-pair batches):
python tools/dropin_phases.py [windows]  ->  one line per window: create / feed / seal / restore ms."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1803_11449_b200 as P  # noqa: E402

dhsa = bench.load_reference()
from dhsa.engine import WindowConfig, WindowSession  # noqa: E402
import dhsa.engine as ref_engine  # noqa: E402

n = 100_000_000
cand, opp, *_ = bench.make_window(100, n, 0)
cand, opp = cand.copy(), opp.copy()
ref_engine.Dhla = lambda params, backend="auto", window_id=0: P.Dhla(params, backend="cuda", window_id=window_id)
for w in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    t = [time.perf_counter()]
    s = WindowSession(WindowConfig(workers=1, theta=1024), w, "auto", None); t.append(time.perf_counter())
    s.feed_batch(cand, opp); t.append(time.perf_counter())
    s.seal(); t.append(time.perf_counter())
    got = s.restore(); t.append(time.perf_counter())
    del s; t.append(time.perf_counter())
    ms = [round((b - a) * 1e3, 2) for a, b in zip(t[:-1], t[1:])]
    if w < 8 or w % 50 == 0:
        import psutil
        import torch
        free, total = torch.cuda.mem_get_info()
        print(dict(zip(("create", "feed", "seal", "restore", "destroy"), ms)), "Gpps", round(n / (t[4] - t[0]) / 1e9, 2), len(got),
              "RSS MiB", psutil.Process().memory_info().rss >> 20, "device MiB", (total - free) >> 20, flush=True)
