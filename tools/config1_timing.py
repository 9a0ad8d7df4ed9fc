"""BASELINE config 1 (the reference's own CPU-runnable case: 978,703 records, 37k background hosts +
20 super points, theta 1024) on the GPU: device-resident and from host arrays, next to the CPU arm."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1803_11449_b200 as P  # noqa: E402
from helpers import config1_pairs, load_json  # noqa: E402

src, dst = config1_pairs()
exp = load_json("config1_expected.json")
n = len(src)
sk = P.Dhla(P.DhgParams())
stream = torch.cuda.Stream()
out = {"packets": n}
with torch.cuda.stream(stream):
    sk.use_stream(stream.cuda_stream)
    cd, od = torch.from_numpy(src.view(np.int32)).cuda(), torch.from_numpy(dst.view(np.int32)).cuda()
    for name, (c, o) in (("device_resident", (cd, od)), ("host_arrays", (src, dst))):
        for _ in range(3):
            sk.reset(); sk.update_batch(c, o); reports = sk.restore_superpoints(1024)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            sk.reset(); sk.update_batch(c, o); reports = sk.restore_superpoints(1024)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / reps * 1e3
        out[name] = {"ms_per_window": ms, "mpps": n / ms / 1e3, "reports": len(reports)}
out["reports_equal_reference_fixture"] = [(r.host, r.saturated) for r in reports] == [(h, s) for h, _, s in exp["reports"]]
out["reference_cpu_ms_per_window"] = {"value": 58.9, "source": "SURVEY.md section 6: compiled backend, 1 worker (update 54.8 + zero counts 3.0 + candidates 0.8 + re-estimate 0.3)"}
print(json.dumps(out))
