#!/bin/bash
# compute-sanitizer over a small end-to-end run of every kernel family (memcheck, then racecheck and synccheck on the scan)
mkdir -p gpurun_out
cat > /tmp/san_small.py <<'PY'
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1803_11449_b200 as P
from oracle import oracle as O

cand, opp = O.distinct_pairs(40_000, 14)
for host, fan, seed in [(2_000_000 + 7 * n, 2048, 600 + n) for n in range(4)]:
    c, o = O.plant_pairs(host, fan, seed)
    cand, opp = np.concatenate([cand, c]), np.concatenate([opp, o])
pick = np.random.default_rng(0).integers(0, len(cand), size=4 * len(cand))
cand, opp = cand[pick], opp[pick]
ora = O.OracleSketch()
ora.update_batch(cand, opp)
want = ora.restore_superpoints(1024)
for mode in ("red", "test", "test_agg", "flow_cache", "auto"):
    sk = P.Dhla(P.DhgParams())
    sk.set_scan_mode(mode)
    sk.update_batch(cand, opp)
    sk.update_batch(cand[:1001], opp[:1001])
    assert np.array_equal(sk.bits, ora.bits), mode
    got = sk.restore_superpoints(1024)
    assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want], mode
# records through the engine (plan kernels, RecordSource scan), exact counter, generator
cfg = P.GeneratorConfig(background_hosts=2_000, superpoints=4, duplicate_factor=3, window_seconds=600, start_ts=2100)
got = P.generate_trace_device(cfg, seed=5, fmt="both")
eng = P.DetectionEngine(P.WindowConfig(theta=1024, window_seconds=300))
res = eng.run(got["records"])
c = P.ExactCounter(expected_pairs=got["flows"])
c.add_pairs(got["cand"], got["opp"])
hosts, counts, n_pairs, n_hosts = c.result(min_count=1024)
# round 2 kernels and paths: hash group forward/inverse, the re-filter, host batches through the slots from threads,
# workspace growth, range download/upload (snapshot), zero_counts hand-in, a parked sketch handed out again
from paper_1803_11449_b200 import dhg
from concurrent.futures import ThreadPoolExecutor
import io
keys = np.arange(5000, dtype=np.uint64) * 977
t = dhg.forward_many(P.DhgParams(), keys)
k2, ok = dhg.reconstruct_many(P.DhgParams(), t)
assert ok.all() and np.array_equal(k2, keys)
sk = P.Dhla(P.DhgParams())
with ThreadPoolExecutor(4) as pool:
    for f in [pool.submit(sk.update_batch, cand[lo:lo + 3001], opp[lo:lo + 3001]) for lo in range(0, len(cand), 3001)]:
        f.result()
assert np.array_equal(sk.bits, ora.bits)
assert len(sk.restore_superpoints(1024, max_candidates=1 << 40)) == len(want)
zc = sk.zero_counts()
assert [len(h) for h in sk.hot_sets(1024, zero_counts=zc)] == [len(h) for h in sk.hot_sets(1024)]
buf = io.BytesIO()
P.write_snapshot(sk, buf)
buf.seek(0)
assert np.array_equal(P.read_snapshot(buf).bits, ora.bits)
del sk
sk = P.Dhla(P.DhgParams())          # the parked one
assert not sk.bits.any()
# round 2, later: one long launch in auto mode is sampled and gated on the device (k_auto_decide + the gated instantiations
# of the test-first and the cache kernel), once with flows that repeat and once with all-distinct pairs; the counter
# snapshot travels on its side stream and the reset waits for it
import torch
big = np.random.default_rng(1).integers(0, len(cand), size=8_600_000)
bc, bo = torch.from_numpy(cand[big].view(np.int32)).cuda(), torch.from_numpy(opp[big].view(np.int32)).cuda()
sk = P.Dhla(P.DhgParams())
n0 = sk.launch_count
sk.update_batch(bc, bo)
assert sk.launch_count - n0 == 4 and np.array_equal(sk.bits, ora.bits)
sk.reset()                                      # waits (stream-ordered) for the snapshot on the side stream
sk.update_batch(bc, bo)                         # the counters have shown repeats: one plain launch now
assert sk.launch_count - n0 == 5 and np.array_equal(sk.bits, ora.bits)
sk = P.Dhla(P.DhgParams(k=15, alpha=6))         # a sketch without that prior
dc, do = O.distinct_pairs(8_600_000, 77)
ora2 = O.OracleSketch(k=15, alpha=6)
ora2.update_batch(dc, do, threads=8)
sk.update_batch(torch.from_numpy(dc.view(np.int32)).cuda(), torch.from_numpy(do.view(np.int32)).cuda())
assert np.array_equal(sk.bits, ora2.bits) and sk.flow_cache_stats()[0] == 1 << 20
# ... and the same through the record form (gated RecordSource instantiations): one window of 8.6M all-distinct records
rec = np.empty(len(dc), dtype=P.TRACE_DTYPE)
rec["ts"], rec["src"], rec["dst"] = 900 + (np.arange(len(dc)) % 300), dc, do
seen = []
try:
    P.DetectionEngine(P.WindowConfig(theta=1024, dhg=P.DhgParams(k=15, alpha=6)), chunk_records=1 << 24).run(
        torch.from_numpy(rec.view(np.uint8).reshape(-1).copy()).cuda(),
        on_sealed=lambda q: seen.append((q.flow_cache_stats()[0], bool(np.array_equal(q.bits, ora2.bits)))))
except P.CapacityError:
    pass
assert seen == [(1 << 20, True)], seen
print("sanitizer run ok:", [len(r.reports) for r in res], n_pairs, n_hosts)
PY
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?"; tail -4 gpurun_out/sanitize_$tool.log
done
