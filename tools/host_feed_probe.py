"""Where the time of a 65,536-pair host batch goes (run on the GPU box):
python tools/host_feed_probe.py  ->  one JSON document on stdout."""
import ctypes as C
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11449_b200 as P  # noqa: E402
from paper_1803_11449_b200 import _cabi  # noqa: E402

N = 50_000_000
B = 65536
rng = np.random.default_rng(1)
flows_c = rng.integers(0, 2 ** 32, size=2_000_000, dtype=np.uint64).astype(np.uint32)
flows_o = rng.integers(0, 2 ** 32, size=2_000_000, dtype=np.uint64).astype(np.uint32)
pick = rng.integers(0, len(flows_c), size=N)
cand, opp = flows_c[pick].copy(), flows_o[pick].copy()
out = {"packets": N, "batch": B, "cpus": os.cpu_count()}

# 1. single-thread copy bandwidth, pageable -> pageable, in 256 KB pieces (what one batch array is)
dst = np.empty(B, dtype=np.uint32)
t0 = time.perf_counter()
for lo in range(0, N, B):
    np.copyto(dst[: len(cand[lo:lo + B])], cand[lo:lo + B])
dt = time.perf_counter() - t0
out["numpy_copy_256k_pieces_gbs"] = 4 * N / dt / 1e9

sk = P.Dhla(P.DhgParams())
lib = _cabi.lib()
sk.update_batch(cand[:B], opp[:B])
sk.seal()

# 2. python + ctypes overhead: the same loop, zero-length calls
t0 = time.perf_counter()
for lo in range(0, N, B):
    c, o = cand[lo:lo + B], opp[lo:lo + B]
    lib.dhsa_update_host(sk._h, c.ctypes.data, o.ctypes.data, 0)
out["python_loop_us_per_call_raw_ctypes"] = (time.perf_counter() - t0) / (N / B) * 1e6
t0 = time.perf_counter()
for lo in range(0, N, B):
    sk.update_batch(cand[lo:lo + 0], opp[lo:lo + 0])
out["python_loop_us_per_call_update_batch_empty"] = (time.perf_counter() - t0) / (N / B) * 1e6


def feed(workers, batch):
    sk.reset()
    sk.seal()
    t0 = time.perf_counter()
    if workers == 1:
        for lo in range(0, N, batch):
            sk.update_batch(cand[lo:lo + batch], opp[lo:lo + batch])
    else:
        with ThreadPoolExecutor(workers) as pool:
            futs = [pool.submit(sk.update_batch, cand[lo:lo + batch], opp[lo:lo + batch]) for lo in range(0, N, batch)]
            for f in futs:
                f.result()
    t1 = time.perf_counter()
    sk.seal()
    t2 = time.perf_counter()
    return {"workers": workers, "batch": batch, "feed_ms": (t1 - t0) * 1e3, "seal_ms": (t2 - t1) * 1e3,
            "mpps": N / (t2 - t0) / 1e6, "us_per_call": (t1 - t0) / (N / batch) * 1e6}


out["runs"] = []
for workers in (1, 2, 4, 8):
    for batch in (B, 1 << 20):
        feed(workers, batch)
        out["runs"].append(feed(workers, batch))
        print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))

# fresh sketch per window, as the reference engine does (engine.py:63): phase timings
import torch  # noqa: E402

phases = []
for rep in range(4):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    s2 = P.Dhla(P.DhgParams()); t.append(time.perf_counter())
    s2.update_batch(cand[:B], opp[:B]); t.append(time.perf_counter())
    for lo in range(B, N, B):
        s2.update_batch(cand[lo:lo + B], opp[lo:lo + B])
    t.append(time.perf_counter())
    s2.seal(); t.append(time.perf_counter())
    s2.restore_superpoints(1024); t.append(time.perf_counter())
    s2.restore_superpoints(1024); t.append(time.perf_counter())
    del s2; t.append(time.perf_counter())
    phases.append(dict(zip(("create", "first_update", "feed_rest", "seal", "restore_1", "restore_2", "destroy"),
                           [round((b - a) * 1e3, 3) for a, b in zip(t[:-1], t[1:])])))
    print(json.dumps(phases[-1]), file=sys.stderr, flush=True)
print(json.dumps({"fresh_sketch_per_window_ms": phases}))
