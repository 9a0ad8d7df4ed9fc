"""Every API family in a loop with the cyclic collector off: host RSS and device memory before / after.
python tools/leak_probe.py [iterations]  (run on the GPU box)"""
import gc
import io
import os
import sys

import numpy as np
import psutil
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11449_b200 as P  # noqa: E402
from paper_1803_11449_b200 import dhg  # noqa: E402
from oracle import oracle as O  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 150
cand, opp = O.distinct_pairs(200_000, 5)
pc, po = O.plant_pairs(777_777, 3000, 2)
cand, opp = np.concatenate([cand, pc]), np.concatenate([opp, po])
cd, od = torch.from_numpy(cand.view(np.int32)).cuda(), torch.from_numpy(opp.view(np.int32)).cuda()
trace = O.engine_trace(11)
cfg = P.GeneratorConfig(background_hosts=2_000, superpoints=4, duplicate_factor=3)


def mem():
    free, total = torch.cuda.mem_get_info()
    return psutil.Process().memory_info().rss >> 20, (total - free) >> 20


def sketch_per_window():
    sk = P.Dhla(P.DhgParams())
    sk.update_batch(cand, opp)
    sk.update_batch(cd, od)
    assert sk.bits.any()
    sk.bits[0, 0, 0] = 1
    sk.restore_superpoints(1024)
    sk.zero_counts(), sk.hot_sets(1024), sk.estimate(1024), sk.shared_zero_counts(np.array([777_777], dtype=np.uint64))
    sk._candidate_hosts(1024)


def other_params():
    sk = P.Dhla(P.DhgParams(r=3, g=256, k=12, alpha=10, key_width=22))
    sk.update_batch(cand & 0x3FFFFF, opp)
    sk.restore_superpoints(256)


def snapshot_and_merge():
    a, b = P.Dhla(P.DhgParams()), P.Dhla(P.DhgParams())
    a.update_batch(cand[::2], opp[::2]), b.update_batch(cand[1::2], opp[1::2])
    buf = io.BytesIO()
    P.write_snapshot(a, buf)
    buf.seek(0)
    c = P.read_snapshot(buf)
    P.merge(c, b).restore_superpoints(1024)


def engine_run():
    P.DetectionEngine(P.WindowConfig(theta=1024)).run(trace)


def exact_and_generator():
    got = P.generate_trace_device(cfg, seed=5, fmt="both")
    c = P.ExactCounter(expected_pairs=got["flows"])
    c.add_pairs(got["cand"], got["opp"])
    c.result(min_count=1024)


def hash_group():
    keys = np.arange(20_000, dtype=np.uint64) * 977
    dhg.reconstruct_many(P.DhgParams(), dhg.forward_many(P.DhgParams(), keys))


def pipelined():
    sk = P.Dhla(P.DhgParams())
    for w in range(3):
        sk.reset()
        sk.update_batch(cd, od)
        if w:
            sk.restore_superpoints_end()
        sk.restore_superpoints_begin(1024)
    sk.restore_superpoints_end()


gc.collect()
gc.disable()
for fn in (sketch_per_window, other_params, snapshot_and_merge, engine_run, exact_and_generator, hash_group, pipelined):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    r0, d0 = mem()
    for _ in range(N):
        fn()
    torch.cuda.synchronize()
    r1, d1 = mem()
    print(f"{fn.__name__:22s} x{N}: host RSS {r0} -> {r1} MiB, device {d0} -> {d1} MiB", flush=True)
