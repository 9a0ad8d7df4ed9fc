"""Row N1 on the GPU: record decode + windowing + direction split fused into the scan,
behind the reference engine's API (pkg/src/dhsa/engine.py), against the reference
engine's own results (tests/golden/engine_cases.json) and the oracle's restatement."""
import numpy as np
import pytest

import paper_1803_11449_b200 as P
from oracle import oracle as O

from helpers import load_json

pytestmark = pytest.mark.gpu

REL_TOL = 1e-6
ENGINE_CASES = load_json("engine_cases.json")


def _same(results, windows):
    assert [(r.window_id, r.pairs, r.dropped) for r in results] == \
        [(w["window_id"], w["pairs"], w["dropped"]) for w in windows]
    for r, w in zip(results, windows):
        assert [(x.host, x.saturated) for x in r.reports] == [(h, s) for h, _, s in w["reports"]]
        for x, (_, e, _) in zip(r.reports, w["reports"]):
            assert x.estimate == pytest.approx(e, rel=REL_TOL)


@pytest.mark.parametrize("chunk", [1 << 24, 4096, 1000])
@pytest.mark.parametrize("case", ENGINE_CASES, ids=[f"{c['seed']}-{c['direction']}" for c in ENGINE_CASES])
def test_engine_matches_reference_engine(case, chunk):
    """Windows, pair counts, late-record drops and reports equal the reference engine's,
    whatever the staging chunk size (window boundaries inside and across chunks)."""
    trace = O.engine_trace(case["seed"])
    cfg = P.WindowConfig(direction=case["direction"], window_seconds=case["window_seconds"], theta=case["theta"])
    results = P.DetectionEngine(cfg, chunk_records=chunk).run(trace)
    _same(results, case["windows"])


def test_engine_accepts_device_tensors_tuples_and_bytes():
    import torch

    case = ENGINE_CASES[0]
    trace = O.engine_trace(case["seed"])
    cfg = P.WindowConfig(direction=case["direction"])
    raw = trace.view(np.uint8).reshape(-1)
    dev = torch.from_numpy(raw.copy()).cuda()
    _same(P.DetectionEngine(cfg).run(dev), case["windows"])
    _same(P.DetectionEngine(cfg).run(raw.tobytes()), case["windows"])
    small = trace[:2000]
    tuples = [(int(t), int(s), int(d)) for t, s, d in zip(small["ts"], small["src"], small["dst"])]
    a = P.DetectionEngine(cfg).run(tuples)
    b = O.run_windows(small, 300, 1024, case["direction"])
    assert [(r.window_id, r.pairs, r.dropped) for r in a] == [(w, p, d) for w, p, d, _ in b]


def test_engine_empty_stream_and_on_sealed_hook():
    cfg = P.WindowConfig()
    assert P.DetectionEngine(cfg).run(np.empty(0, dtype=P.TRACE_DTYPE)) == []
    trace = O.engine_trace(9)
    seen = []
    res = P.DetectionEngine(cfg).run(trace, on_sealed=lambda sk: seen.append((sk.window_id, int(sk.bits.any()))))
    assert [w for w, _ in seen] == [r.window_id for r in res] and all(b for _, b in seen)


@pytest.mark.parametrize("kw", [dict(r=4, g=64, k=8, alpha=4, key_width=16), dict(r=3, g=8, k=8, alpha=8, key_width=16),
                                dict(r=7, g=128, k=10, alpha=4, key_width=30)])
def test_engine_general_path_parameters(kw):
    """Parameter sets outside the vectorised kernels go through the one-record-per-lane path."""
    trace = O.engine_trace(10, n_noise=6_000)
    if kw["key_width"] < 32:   # keep candidate keys inside the key width so planted hosts restore
        for f in ("src", "dst"):
            trace[f] = trace[f] & np.uint32((1 << kw["key_width"]) - 1)
    theta = kw["g"] // 2
    cfg = P.WindowConfig(dhg=P.DhgParams(**kw), theta=theta, direction="both", max_candidates=1 << 22)
    try:
        want = O.run_windows(trace, 300, theta, "both", max_candidates=1 << 22, **kw)
    except O.OracleCapacityError as exc:
        with pytest.raises(P.CapacityError) as err:
            P.DetectionEngine(cfg, chunk_records=5000).run(trace)
        assert str(err.value) == str(exc)
        return
    got = P.DetectionEngine(cfg, chunk_records=5000).run(trace)
    assert [(r.window_id, r.pairs, r.dropped) for r in got] == [(w, p, d) for w, p, d, _ in want]
    for r, (_, _, _, reps) in zip(got, want):
        assert [(x.host, x.saturated) for x in r.reports] == [(x.host, x.saturated) for x in reps]


def test_window_session_contract():
    # pkg/tests/test_engine.py: seal contract and feed/restore ordering
    cfg = P.WindowConfig()
    s = P.WindowSession(cfg, window_id=3)
    cand, opp = O.plant_pairs(0xC63A1B02, 2048, 10)
    with pytest.raises(P.SealedWindowError):
        s.restore()
    with pytest.raises(ValueError):
        s.feed_batch(cand, opp[:-1])
    s.feed_batch(cand, opp)
    s.seal()
    assert s.pairs == 2048
    with pytest.raises(P.SealedWindowError):
        s.feed_batch(cand, opp)
    (rep,) = s.restore()
    assert rep.host == 0xC63A1B02
    with pytest.raises(P.ConfigError):
        P.WindowConfig(direction="sideways")
    with pytest.raises(P.ConfigError):
        P.WindowConfig(theta=0)


def test_records_scan_bits_equal_pair_scan_for_unaligned_segments():
    """dhsa_update_records_device over ragged [lo, hi) ranges equals update_batch on the
    decoded pairs (bit-exact), for every direction."""
    import ctypes as C

    import torch

    from paper_1803_11449_b200 import _cabi

    rec = O.engine_trace(9, n_noise=30_000)
    rec["ts"] = 1000  # one window
    dev = torch.from_numpy(rec.view(np.uint8).reshape(-1).copy()).cuda()
    n = len(rec)
    for direction, (lo, hi) in zip((0, 1, 2, 0, 2), ((0, n), (1, n - 1), (3, 10_001), (5, 6), (7, 9))):
        sk = P.Dhla(P.DhgParams())
        _cabi.check(_cabi.lib().dhsa_update_records_device(sk._h, C.c_void_p(dev.data_ptr()), n, lo, hi, 300, 3, direction))
        src, dst = rec["src"][lo:hi].astype(np.uint32), rec["dst"][lo:hi].astype(np.uint32)
        ora = O.OracleSketch()
        if direction in (0, 2):
            ora.update_batch(src, dst)
        if direction in (1, 2):
            ora.update_batch(dst, src)
        assert np.array_equal(sk.bits, ora.bits), (direction, lo, hi)


def test_auto_mode_decides_on_the_device_for_a_long_record_segment():
    """One window of 9M all-distinct records handed over in one device buffer: the segment's scan is sampled and gated
    on the device like a long pair launch (k_auto_decide + the gated RecordSource instantiations) -- only the sample
    consults the flow cache -- and the sealed sketch equals the oracle's."""
    import torch

    n = 9_000_000
    cand, opp = O.distinct_pairs(n, 95)
    rec = np.empty(n, dtype=P.TRACE_DTYPE)
    rec["ts"] = 3 * 300 + (np.arange(n) % 300)
    rec["src"], rec["dst"] = cand, opp
    ora = O.OracleSketch()
    ora.update_batch(cand, opp, threads=8)
    dev = torch.from_numpy(rec.view(np.uint8).reshape(-1).copy()).cuda()
    seen = []

    def sealed(sk):
        seen.append((sk.window_id, sk.flow_cache_stats(), bool(np.array_equal(sk.bits, ora.bits))))

    try:
        res = P.DetectionEngine(P.WindowConfig(theta=1024), chunk_records=1 << 24).run(dev, on_sealed=sealed)
    except P.CapacityError:
        res = None                                   # 9M distinct flows make every cell hot, as in the reference
    assert len(seen) == 1
    window_id, (lookups, hits), same = seen[0]
    assert window_id == 3 and same
    assert lookups == 1 << 20 and hits * 10 < lookups
