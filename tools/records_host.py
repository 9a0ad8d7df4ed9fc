"""DetectionEngine.run on HOST record arrays (row N1 end to end): pageable numpy vs pinned."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1803_11449_b200 as P  # noqa: E402

cfg = P.GeneratorConfig(background_hosts=150_000, superpoints=50, duplicate_factor=26, window_seconds=600, start_ts=2100)
got = P.generate_trace_device(cfg, seed=100, fmt="records")
n = got["total"]
pinned = torch.empty(n * 12, dtype=torch.uint8, pin_memory=True)
pinned.copy_(got["records"])
torch.cuda.synchronize()
pageable = pinned.numpy().copy()
eng = P.DetectionEngine(P.WindowConfig(theta=1024, window_seconds=300))
want = eng.run(got["records"])
out = {"records": n}
for name, arr in (("pageable", pageable), ("pinned", pinned.numpy())):
    eng.run(arr)
    t0 = time.perf_counter()
    for _ in range(3):
        res = eng.run(arr)
    dt = (time.perf_counter() - t0) / 3
    same = [(r.window_id, r.pairs, r.dropped, [(x.host, x.estimate) for x in r.reports]) for r in res] == \
           [(r.window_id, r.pairs, r.dropped, [(x.host, x.estimate) for x in r.reports]) for r in want]
    out[name] = {"ms_per_run": dt * 1e3, "mpps": n / dt / 1e6, "equal_device_resident_run": bool(same)}
print(json.dumps(out))
