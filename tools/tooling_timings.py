"""One-off timings of the evaluation tooling rows (N3 exact oracle, N4 generator) for DESIGN.md."""
import json
import time

import torch

import paper_1803_11449_b200 as P

cfg = P.GeneratorConfig(background_hosts=150_000, superpoints=50, duplicate_factor=26)
torch.cuda.synchronize()
out = {}
for fmt in ("pairs", "records"):
    got = P.generate_trace_device(cfg, seed=100, fmt=fmt)   # warm-up + data
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    got = P.generate_trace_device(cfg, seed=100, fmt=fmt)
    e1.record()
    torch.cuda.synchronize()
    out[f"generate_{fmt}"] = {"packets": got["total"], "flows": got["flows"], "gpu_ms": e0.elapsed_time(e1),
                              "wall_ms": 1e3 * (time.perf_counter() - t0)}
got = P.generate_trace_device(cfg, seed=100, fmt="pairs")
for rep in range(2):
    c = P.ExactCounter(expected_pairs=got["flows"])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    c.add_pairs(got["cand"], got["opp"])
    hosts, counts, n_pairs, n_hosts = c.result(min_count=1024)
    e1.record()
    torch.cuda.synchronize()
out["exact_oracle"] = {"packets": got["total"], "distinct_pairs": n_pairs, "hosts": n_hosts,
                       "superpoints": len(hosts), "gpu_ms": e0.elapsed_time(e1)}
sk = P.Dhla(P.DhgParams())
sk.update_batch(got["cand"], got["opp"])
m = P.evaluate(sk.restore_superpoints(1024), dict(zip(hosts.tolist(), counts.tolist())), 1024)
out["accuracy_config2"] = m.as_dict()
print(json.dumps(out))
