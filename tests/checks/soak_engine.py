"""Randomised soak of the record engine (row N1) against the oracle's restatement of the reference
engine: random traces with out-of-order and far-future timestamps, window lengths, directions,
chunk sizes, host and device inputs.  python tests/checks/soak_engine.py [seconds]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1803_11449_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only)

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(77)
t0 = time.perf_counter()
runs = records_total = windows_total = 0
while time.perf_counter() - t0 < budget:
    n = int(rng.integers(1, 600_000))
    wsec = int(rng.choice([1, 7, 60, 300, 3600]))
    n_windows = int(rng.integers(1, 6))
    start = int(rng.integers(0, 2 ** 31))
    ts = np.sort(rng.integers(start, start + n_windows * wsec, size=n, dtype=np.int64))
    jitter = rng.random(n)
    ts = np.where(jitter < 0.02, ts - rng.integers(0, 2 * wsec + 1, size=n), ts)          # late arrivals
    ts = np.where(jitter > 0.999, ts + rng.integers(0, 3 * wsec + 1, size=n), ts)          # clocks running ahead
    ts = np.clip(ts, 0, 2 ** 32 - 1)
    flows = int(rng.integers(1, 50_000))
    fc, fo = O.distinct_pairs(flows, int(rng.integers(1 << 20)))
    for host, fan in ((0x0A000001, 1500), (0xC0A80001, 3000)):
        c2, o2 = O.plant_pairs(host, fan, int(rng.integers(1 << 16)))
        fc, fo = np.concatenate([fc, c2]), np.concatenate([fo, o2])
    pick = rng.integers(0, len(fc), size=n)
    rec = np.zeros(n, dtype=P.TRACE_DTYPE)
    rec["ts"], rec["src"], rec["dst"] = ts.astype(np.uint32), fc[pick], fo[pick]
    direction = ["src", "dst", "both"][rng.integers(3)]
    theta = int(rng.choice([256, 1024]))
    chunk = int(rng.choice([1 << 24, 65_536, 4_099, 1_000]))
    want = O.run_windows(rec, wsec, theta, direction)
    eng = P.DetectionEngine(P.WindowConfig(theta=theta, window_seconds=wsec, direction=direction), chunk_records=chunk)
    src = rec
    if rng.random() < 0.5:                                   # raw records already on the device
        src = torch.from_numpy(P.engine._as_record_bytes(rec).copy()).cuda()
    got = eng.run(src)
    a = [(r.window_id, r.pairs, r.dropped, [(x.host, x.saturated) for x in r.reports]) for r in got]
    b = [(w, p, d, [(x.host, x.saturated) for x in reps]) for w, p, d, reps in want]
    if a != b:
        print(f"MISMATCH run {runs}: n={n} wsec={wsec} direction={direction} chunk={chunk} theta={theta}")
        print([x[:3] for x in a][:8], [x[:3] for x in b][:8])
        sys.exit(1)
    runs += 1
    records_total += n
    windows_total += len(got)
print(f"engine soak ok: {runs} random traces, {records_total} records, {windows_total} windows, "
      f"{time.perf_counter() - t0:.0f} s")
