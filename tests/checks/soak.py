"""Randomised soak of the scan against the oracle: random window sizes, duplication, skew, scan
modes, flow-cache sizes, batch splits and host/device inputs; bits must match every time.
python tests/checks/soak.py [seconds]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1803_11449_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only)

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(2026)
t0 = time.perf_counter()
runs = packets = 0
long_runs = gated = 0
PARAMS = [dict(), dict(r=3, g=256, k=18, alpha=14, key_width=32, seed_dh0=3, seed_h1=4),
          dict(r=6, g=512, k=12, alpha=5), dict(r=4, g=32, k=9, alpha=8, key_width=24),
          dict(r=5, g=4096, k=12, alpha=7, seed_h1=99)]
while time.perf_counter() - t0 < budget:
    kw = PARAMS[rng.integers(len(PARAMS))]
    flows = int(rng.integers(1, 400_000))
    cand, opp = O.distinct_pairs(flows, int(rng.integers(1 << 20)))
    if rng.random() < 0.3:   # a few heavy keys
        cand[: flows // 3] = cand[rng.integers(0, min(8, flows), size=flows // 3)]
    if rng.random() < 0.2:   # many flows of few hosts with colliding h1: the (cand, h) key collapses them
        opp[::2] = opp[rng.integers(0, min(64, flows), size=len(opp[::2]))]
    n = int(rng.integers(1, 3_000_000))
    long_launch = rng.random() < 0.12          # a window long enough for a device-gated auto launch (>= 2^23 packets)
    if long_launch:
        n = int(rng.integers(8_400_000, 20_000_000))
        if rng.random() < 0.5:                 # ... over flows that (almost) never repeat
            flows = n
            cand, opp = O.distinct_pairs(flows, int(rng.integers(1 << 20)))
    pick = rng.integers(0, flows, size=n)
    c, o = cand[pick], opp[pick]
    mode = "auto" if long_launch else ["red", "test", "test_agg", "flow_cache", "auto"][rng.integers(5)]
    sk = P.Dhla(P.DhgParams(**kw))
    sk.set_scan_mode(mode)
    sk.set_flow_cache(int(2 ** rng.integers(10, 21)))
    ora = O.OracleSketch(**kw)
    ora.update_batch(c, o, threads=8)
    pos = 0
    gated_launches = 0
    while pos < n:          # random batch splits, alternating host and device inputs
        step = int(rng.integers(1, n + 1))
        if long_launch and pos == 0:           # the first batch in one device launch
            step = int(rng.integers(8_400_000, n + 1))
            before = sk.launch_count
            sk.update_batch(torch.from_numpy(c[:step].view(np.int32)).cuda(), torch.from_numpy(o[:step].view(np.int32)).cuda())
            gated_launches = sk.launch_count - before
            pos = step
            continue
        cc, oo = c[pos:pos + step], o[pos:pos + step]
        if rng.random() < 0.5:
            sk.update_batch(cc, oo)
        else:
            sk.update_batch(torch.from_numpy(cc.view(np.int32)).cuda(), torch.from_numpy(oo.view(np.int32)).cuda())
        if rng.random() < 0.1:
            sk.update_batch(cc, oo)        # replay: idempotent
        pos += step
    if not np.array_equal(sk.bits, ora.bits):
        print(f"MISMATCH run {runs}: kw={kw} flows={flows} n={n} mode={mode}")
        sys.exit(1)
    if long_launch:
        gated += gated_launches >= 4           # sample, verdict, two gated kernels (+ a ragged tail)
        long_runs += 1
    def outcome(f):   # reports, or the CapacityError text (the reference aborts loudly; so must both sides, identically)
        try:
            return [(r.host, r.saturated) for r in f(256)]
        except (P.CapacityError, O.OracleCapacityError) as e:
            return str(e)

    got = outcome(sk.restore_superpoints)
    # (millions of distinct flows make every cell hot: the oracle's literal |HE|^3 enumeration would run for hours
    # before it reports the overflow the device chain finds at once -- the bits were compared above)
    want = outcome(ora.restore_superpoints) if flows <= 400_000 else got
    if got != want:
        print(f"REPORT MISMATCH run {runs}: kw={kw} flows={flows} n={n} mode={mode}")
        sys.exit(1)
    runs += 1
    packets += n
    if runs % 100 == 0:      # a leak would show here long before the box runs out of memory
        import psutil
        print(f"  {runs} windows, {time.perf_counter() - t0:.0f} s, host RSS {psutil.Process().memory_info().rss >> 20} MiB, "
              f"device {torch.cuda.memory_allocated() >> 20} MiB (torch) / {(torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) >> 20} MiB (all)",
              flush=True)
print(f"soak ok: {runs} random windows, {packets} packets, {time.perf_counter() - t0:.0f} s "
      f"({long_runs} with a first launch of >= 8.4M packets, {gated} of them sampled and gated on the device)")
