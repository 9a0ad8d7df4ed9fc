"""GPU parity: the CUDA path, called through the C ABI, against the CPU oracle,
against the committed golden fixtures (recorded from the live reference), and
-- at BASELINE.json's full sizes -- through properties that do not need a CPU
run of the same size (the sketch is a pure function of the distinct pair set,
/root/reference/SPEC.md:356).

Bar: bit-exact on the DDH bit array, zero counts, hot sets, candidate hosts,
per-stage survivor counts, CapacityError text and the reported host list and
order; cardinality estimates within REL_TOL = 1e-6 relative (the north star's
tolerance; observed agreement is ~1e-15, device fp64 log vs numpy's).
"""
import concurrent.futures
import hashlib

import numpy as np
import pytest

import paper_1803_11449_b200 as P
from oracle import oracle as O

from helpers import (case_batches, case_params, config1_pairs, load_json, oracle_for_case,
                     restore_cases)

pytestmark = pytest.mark.gpu

REL_TOL = 1e-6
CASES = restore_cases()
PARAM_SETS = {
    "default": dict(),
    "toy": dict(r=4, g=64, k=8, alpha=4, key_width=16),
    "small": dict(r=5, g=256, k=10, alpha=8, key_width=32, seed_dh0=1, seed_h1=2),
    "min_r3": dict(r=3, g=256, k=18, alpha=14, key_width=32, seed_dh0=3, seed_h1=4),
    "six": dict(r=6, g=512, k=12, alpha=5),
    "g8": dict(r=3, g=8, k=8, alpha=8, key_width=16),
    "g16": dict(r=4, g=16, k=10, alpha=8, key_width=24, seed_dh0=11, seed_h1=12),
    "g32": dict(r=4, g=32, k=9, alpha=8, key_width=24),
    "r7_generic": dict(r=7, g=128, k=10, alpha=4, key_width=30),
    "big_g": dict(r=3, g=8192, k=11, alpha=11, key_width=22),
}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gpu_for_case(case, mode="test_agg"):
    sk = P.Dhla(P.DhgParams(**case["params"]))
    sk.set_scan_mode(mode)
    for c, o in case_batches(case):
        sk.update_batch(c, o)
    return sk


# ------------------------------------------------------------------------ scan --


MODES = ["red", "test", "test_agg", "flow_cache", "auto"]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", list(PARAM_SETS))
def test_update_batch_bits_equal_oracle(name, mode):
    # pkg/tests/test_kernels.py:37-48 (compiled == numpy), here CUDA == oracle
    kw = PARAM_SETS[name]
    cand, opp = O.distinct_pairs(50_000, 3)
    ora = O.OracleSketch(**kw)
    ora.update_batch(cand, opp)
    sk = P.Dhla(P.DhgParams(**kw))
    sk.set_scan_mode(mode)
    sk.update_batch(cand, opp)
    assert np.array_equal(sk.bits, ora.bits)
    assert np.array_equal(sk.zero_counts(), ora.zero_counts())
    if name == "default":
        assert sha(sk.bits) == "38d4cac25b1922468b09d87d40a536699a03d0a58ac44cdc776a8ed1995dd136"


def test_single_update_sets_exactly_r_bits():
    # pkg/tests/test_dhla.py:49-52 and the byte/mask constants of SURVEY 8(c)
    const = load_json("constants.json")
    sk = P.Dhla(P.DhgParams())
    sk.update(0xC0A80101, 0x08080808)
    bits = sk.bits
    got = [[int(i), int(j), int(b), int(bits[i, j, b])] for i, j, b in np.argwhere(bits)]
    assert got == const["single_update"]
    assert sk.memory_bytes == 10_485_760


@pytest.mark.parametrize("n", [0, 1, 2, 3, 4, 5, 31, 33, 1023, 4097])
def test_ragged_lengths_and_empty_batches(n):
    cand, opp = O.distinct_pairs(max(n, 1), 8)
    cand, opp = cand[:n], opp[:n]
    ora = O.OracleSketch()
    ora.update_batch(cand, opp)
    sk = P.Dhla(P.DhgParams())
    sk.update_batch(cand, opp)
    assert np.array_equal(sk.bits, ora.bits)


def test_length_mismatch_raises_value_error():
    # pkg/src/dhsa/_core.pyx:73-74
    sk = P.Dhla(P.DhgParams())
    with pytest.raises(ValueError):
        sk.update_batch(np.zeros(4, np.uint32), np.zeros(5, np.uint32))


def test_update_is_idempotent_and_permutation_invariant():
    # pkg/tests/test_dhla.py:55-78
    cand, opp = O.distinct_pairs(10_000, 3)
    order = np.random.default_rng(4).permutation(len(cand))
    a, b, c = (P.Dhla(P.DhgParams()) for _ in range(3))
    a.update_batch(cand, opp)
    b.update_batch(cand[order], opp[order])
    c.update_batch(cand, opp)
    c.update_batch(cand, opp)
    ref = a.bits
    assert np.array_equal(ref, b.bits) and np.array_equal(ref, c.bits)


def test_device_tensor_inputs_including_unaligned_views():
    import torch

    cand, opp = O.distinct_pairs(100_003, 9)
    ora = O.OracleSketch()
    ora.update_batch(cand[1:], opp[1:])
    ct = torch.from_numpy(cand.view(np.int32)).cuda()
    ot = torch.from_numpy(opp.view(np.int32)).cuda()
    sk = P.Dhla(P.DhgParams())
    sk.update_batch(ct[1:], ot[1:])  # 4-byte aligned only: takes the general kernel
    assert np.array_equal(sk.bits, ora.bits)
    sk2 = P.Dhla(P.DhgParams())
    sk2.update_batch(ct[4:], ot[4:])  # 16-byte aligned: vector kernel + scalar tail
    sk2.update_batch(ct[1:4], ot[1:4])
    assert np.array_equal(sk2.bits, ora.bits)


def test_concurrent_updates_from_threads_are_lossless():
    # pkg/tests/test_kernels.py:62-74
    cand, opp = O.distinct_pairs(400_000, 5)
    ora = O.OracleSketch()
    ora.update_batch(cand, opp, threads=4)
    shared = P.Dhla(P.DhgParams())
    chunks = [(cand[s::8], opp[s::8]) for s in range(8)]
    with concurrent.futures.ThreadPoolExecutor(max_workers=8) as pool:
        list(pool.map(lambda co: shared.update_batch(*co), chunks))
    assert np.array_equal(shared.bits, ora.bits)


@pytest.mark.parametrize("mode", MODES)
def test_ddos_contention_all_packets_hit_the_same_cells(mode):
    # BASELINE config 4 shape: many sources -> few victims, victims as candidates
    rng = np.random.default_rng(44)
    victims = rng.integers(0, 2 ** 32, size=4, dtype=np.uint64).astype(np.uint32)
    n = 2_000_000
    cand = victims[rng.zipf(1.2, size=n) % 4]
    opp = rng.integers(0, 2 ** 32, size=n, dtype=np.uint64).astype(np.uint32)
    ora = O.OracleSketch()
    ora.update_batch(cand, opp, threads=4)
    sk = P.Dhla(P.DhgParams())
    sk.set_scan_mode(mode)
    sk.update_batch(cand, opp)
    assert np.array_equal(sk.bits, ora.bits)
    got, want = sk.restore_superpoints(1024), ora.restore_superpoints(1024)
    assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
    assert all(r.saturated for r in got) and len(got) == 4


@pytest.mark.parametrize("n_sets", [1024, 50_000, 1 << 21])
def test_flow_cache_is_exact_across_batches_resets_and_uploads(n_sets):
    """The cache may only skip pairs whose bits are already in the sketch: heavy
    duplication over several batches, tiny tables that evict constantly, the
    all-ones pair (never cached), then reset and load_bits, which must empty it."""
    rng = np.random.default_rng(5)
    base_c, base_o = O.distinct_pairs(60_000, 31)
    base_c = np.concatenate([base_c, np.array([0xFFFFFFFF, 0, 0xFFFFFFFF], np.uint32)])
    base_o = np.concatenate([base_o, np.array([0xFFFFFFFF, 0, 0], np.uint32)])
    sk = P.Dhla(P.DhgParams())
    sk.set_scan_mode("flow_cache")
    sk.set_flow_cache(n_sets)
    ora = O.OracleSketch()
    for _ in range(3):
        pick = rng.integers(0, len(base_c), size=400_000)
        sk.update_batch(base_c[pick], base_o[pick])
        ora.update_batch(base_c[pick], base_o[pick], threads=4)
        assert np.array_equal(sk.bits, ora.bits)
    lookups, hits = sk.flow_cache_stats()
    assert lookups == 1_200_000 and 0 < hits < lookups
    # reset: same pairs again must set their bits again
    sk.reset()
    pick = rng.integers(0, len(base_c), size=100_000)
    sk.update_batch(base_c[pick], base_o[pick])
    fresh = O.OracleSketch()
    fresh.update_batch(base_c[pick], base_o[pick])
    assert np.array_equal(sk.bits, fresh.bits)
    # load_bits with cleared cells: cached pairs must not be trusted afterwards
    sk.load_bits(np.zeros_like(fresh.bits))
    sk.update_batch(base_c[pick], base_o[pick])
    assert np.array_equal(sk.bits, fresh.bits)
    # merge only adds bits: the cache stays valid and the result is still exact
    other = P.Dhla(P.DhgParams())
    oc, oo = O.distinct_pairs(10_000, 32)
    other.update_batch(oc, oo)
    sk.merge_from(other)
    sk.update_batch(base_c[pick], base_o[pick])
    fresh.update_batch(oc, oo)
    assert np.array_equal(sk.bits, fresh.bits)
    # a reset bumps the table's epoch instead of clearing it; go around the epoch counter
    # (31 epochs at 32768 sets, 1 at 2048) so stale entries of a recycled epoch would show
    small_c, small_o = base_c[:5000], base_o[:5000]
    want = O.OracleSketch()
    want.update_batch(small_c, small_o)
    for _ in range(40):
        sk.reset()
        sk.update_batch(small_c, small_o)
        sk.seal()            # host batches are coalesced into one scan per slot: the barrier makes it two scans
        sk.update_batch(small_c, small_o)
    assert np.array_equal(sk.bits, want.bits)
    lookups, hits = sk.flow_cache_stats()
    assert lookups == 10_000 and 2_500 <= hits <= 5_100       # the second pass of the last window hits (lost insert races aside)


def test_restore_begin_end_overlaps_the_next_window():
    """dhsa_restore_begin/_end: window k's read-out is enqueued, window k + 1 is reset and fed on
    the same sketch, and only then are window k's reports collected -- they must be window k's."""
    windows = []
    for w in range(3):
        cand, opp = O.distinct_pairs(100_000, 200 + w)
        for host, fan, seed in [(3_000_000 + 11 * w + n, 2048 + 100 * n, 700 + 10 * w + n) for n in range(4 + w)]:
            c, o = O.plant_pairs(host, fan, seed)
            cand, opp = np.concatenate([cand, c]), np.concatenate([opp, o])
        ora = O.OracleSketch()
        ora.update_batch(cand, opp, threads=4)
        windows.append((cand, opp, ora.restore_superpoints(1024)))
    sk = P.Dhla(P.DhgParams())
    with pytest.raises(P.ConfigError):
        sk.restore_superpoints_end()                       # nothing begun
    got = []
    for w, (cand, opp, _) in enumerate(windows):
        sk.reset()
        sk.update_batch(cand, opp)
        if w:
            got.append(sk.restore_superpoints_end())       # window w - 1, collected after window w was fed
        sk.restore_superpoints_begin(1024)
        with pytest.raises(P.ConfigError):
            sk.estimate(1024)                              # the pinned mirrors belong to the pending read-out
        with pytest.raises(P.ConfigError):
            sk.restore_superpoints_begin(1024)
    got.append(sk.restore_superpoints_end())
    for reports, (_, _, want) in zip(got, windows):
        assert [(r.host, r.saturated) for r in reports] == [(r.host, r.saturated) for r in want]
        assert len(reports) >= 4
        for a, b in zip(reports, want):
            assert a.estimate == pytest.approx(b.estimate, rel=REL_TOL)
    assert sk.estimate(1024)["flow_count"] > 0              # collected: read-out calls work again


def test_auto_mode_falls_back_when_flows_do_not_repeat():
    """All-distinct pairs: the hit rate stays ~0, auto switches kernels mid-window; bits stay exact."""
    cand, opp = O.distinct_pairs(12_000_000, 90)
    ora = O.OracleSketch(r=5, g=1024, k=16, alpha=6)
    ora.update_batch(cand, opp, threads=8)
    sk = P.Dhla(P.DhgParams(r=5, g=1024, k=16, alpha=6))
    for s in range(0, len(cand), 2_000_000):   # several launches so the policy sees the statistics
        sk.update_batch(cand[s:s + 2_000_000], opp[s:s + 2_000_000])
        sk.seal()
    assert sha(sk.bits) == sha(ora.bits)
    assert sk.scan_mode_used == "test"                       # what auto resolved to for the last batches
    lookups, hits = sk.flow_cache_stats()
    assert 0 < lookups < len(cand) and hits * 10 < lookups   # later batches bypassed the cache
    sk.reset()                                               # next window starts behind the cache again
    sk.update_batch(cand[:1_000_000], opp[:1_000_000])
    assert sk.flow_cache_stats()[0] == 1_000_000 and sk.scan_mode_used == "flow_cache"


def test_auto_mode_decides_on_the_device_inside_one_long_launch():
    """One 24M-packet launch of all-distinct pairs: the host cannot read the counters mid-launch, so the
    launch is sampled and gated on the device -- the first 2^20 packets go through the flow cache, the hit
    rate projected from them (~0) sends the rest to the test-first kernel.  Then a window whose flows
    repeat (a cold table: few hits in the sample, many projected): the cache kernel takes the rest, and
    from the next window on the launch is not split at all.  Bits exact throughout."""
    import torch

    n = 24_000_000
    cand, opp = O.distinct_pairs(n, 91)
    ora = O.OracleSketch()
    ora.update_batch(cand, opp, threads=8)
    cd, od = torch.from_numpy(cand.view(np.int32)).cuda(), torch.from_numpy(opp.view(np.int32)).cuda()
    sk = P.Dhla(P.DhgParams())
    before = sk.launch_count
    sk.update_batch(cd, od)
    assert sk.launch_count - before == 4                      # sample, verdict, gated test-first, gated cache
    assert sha(sk.bits) == sha(ora.bits)
    lookups, hits = sk.flow_cache_stats()
    assert lookups == 1 << 20 and hits * 10 < lookups         # only the sample consulted the cache
    # a window that repeats, slowly: 24M packets over 6M flows (4 packets per flow; 8% hits within the sample)
    rng = np.random.default_rng(5)
    pick = rng.integers(0, 6_000_000, size=n)
    rc, ro = cand[:6_000_000][pick], opp[:6_000_000][pick]
    ora2 = O.OracleSketch()
    ora2.update_batch(rc, ro, threads=8)
    cd, od = torch.from_numpy(rc.view(np.int32)).cuda(), torch.from_numpy(ro.view(np.int32)).cuda()
    for window, want_launches in ((0, 4), (1, 1), (2, 1)):   # gated once more, then the counters have shown repeats
        sk.reset()
        before = sk.launch_count
        sk.update_batch(cd, od)
        sk.seal()
        assert sk.launch_count - before == want_launches, window
        assert sha(sk.bits) == sha(ora2.bits)
        lookups, hits = sk.flow_cache_stats()
        assert lookups == n and hits > 0.65 * n


def test_auto_mode_learns_from_the_read_out_when_windows_are_pipelined():
    """reset() right behind restore_begin(): the host is a window ahead of the device, the side-stream snapshot of
    window k has not landed when window k + 1 is reset -- the prior comes from the counters in the read-out instead,
    so only the first two windows are sampled and gated."""
    import torch

    n = 16_000_000
    cand, opp = O.distinct_pairs(500_000, 93)
    pick = np.random.default_rng(7).integers(0, 500_000, size=n)
    cd = torch.from_numpy(cand[pick].view(np.int32)).cuda()
    od = torch.from_numpy(opp[pick].view(np.int32)).cuda()
    ora = O.OracleSketch()
    ora.update_batch(cand, opp)
    sk = P.Dhla(P.DhgParams())
    launches = []
    for w in range(5):
        sk.reset()
        before = sk.launch_count
        sk.update_batch(cd, od)
        launches.append(sk.launch_count - before)
        if w:
            sk.restore_superpoints_end()                 # window w - 1
        sk.restore_superpoints_begin(1024)
    sk.restore_superpoints_end()
    assert launches[0] == 4 and launches[-1] == 1 and launches[-2] == 1, launches
    assert sha(sk.bits) == sha(ora.bits)


def test_auto_mode_is_not_fooled_by_a_cold_table():
    """6M flows, 4 packets each, fed in six 4M-packet batches: after the first batch only a quarter of the
    lookups hit (the table was empty), though three quarters will over the window.  The policy projects the
    counts (projected_no_repeats) and stays behind the cache; on all-distinct pairs it still leaves it."""
    n = 24_000_000
    cand, opp = O.distinct_pairs(6_000_000, 92)
    pick = np.random.default_rng(6).integers(0, 6_000_000, size=n)
    rc, ro = cand[pick], opp[pick]
    ora = O.OracleSketch()
    ora.update_batch(rc, ro, threads=8)
    sk = P.Dhla(P.DhgParams())
    for lo in range(0, n, 4_000_000):
        sk.update_batch(rc[lo:lo + 4_000_000], ro[lo:lo + 4_000_000])
        lookups, hits = sk.flow_cache_stats()                # an engine's per-chunk bookkeeping: the snapshot lands
        if lo == 0:
            assert hits * 10 < lookups * 3                   # what the plain hit-rate rule would have fallen for
    assert sk.scan_mode_used == "flow_cache" and lookups == n and hits > 0.65 * n
    assert sha(sk.bits) == sha(ora.bits)


def test_reading_bits_does_not_keep_sketches_alive():
    """A sketch per window whose `bits` are read (what `dhsa bench` does, pkg/src/dhsa/cli.py:383): mirror and sketch
    must go with their last reference, without the cyclic collector -- 60 windows may not pile up 60 sketches."""
    import gc

    import torch

    def used():
        free, total = torch.cuda.mem_get_info()
        return (total - free) >> 20

    cand, opp = O.distinct_pairs(50_000, 3)
    gc.collect()
    gc.disable()
    try:
        for w in range(60):
            sk = P.Dhla(P.DhgParams(), window_id=w)
            sk.update_batch(cand, opp)
            assert sk.bits.any() and sk.bits[0].shape == (1 << 14, 128)
            if w == 5:
                base = used()                    # the parked sketches and their caches exist by now
            del sk
        assert used() - base < 256, (base, used())   # MiB; 54 leaked sketches would hold > 2 GiB
    finally:
        gc.enable()


def test_estimator_returns_one_cell():
    # pkg/src/dhsa/dhla.py:107-109
    sk = P.Dhla(P.DhgParams(**PARAM_SETS["small"]))
    rnd = np.random.default_rng(3).integers(0, 256, size=sk.bits.shape, dtype=np.uint8)
    sk.load_bits(rnd)
    for i, j in ((0, 0), (2, 517), (4, 1023)):
        assert np.array_equal(sk.estimator(i, j), rnd[i, j])
    with pytest.raises(P.ConfigError):
        sk.estimator(5, 0)
    with pytest.raises(P.ConfigError):
        sk.estimator(0, 1024)


def test_reset_and_load_bits_round_trip():
    sk = P.Dhla(P.DhgParams(**PARAM_SETS["small"]))
    rnd = np.random.default_rng(2).integers(0, 256, size=sk.bits.shape, dtype=np.uint8)
    sk.load_bits(rnd)
    assert np.array_equal(sk.bits, rnd)
    sk.reset(window_id=7)
    assert sk.window_id == 7 and not sk.bits.any()


# -------------------------------------------------------------------- read-out --


@pytest.mark.parametrize("g", [8, 16, 32, 64, 128, 1024, 4096])
def test_zero_counts_match_unpackbits(g):
    # pkg/tests/test_kernels.py:51-59
    sk = P.Dhla(P.DhgParams(r=3, g=g, k=8, alpha=8, key_width=16))
    rnd = np.random.default_rng(4).integers(0, 256, size=(3, 256, g // 8), dtype=np.uint8)
    sk.load_bits(rnd)
    assert np.array_equal(sk.zero_counts(), g - np.unpackbits(rnd, axis=2).sum(axis=2))


def test_hot_threshold_boundary_376_hot_377_not():
    # pkg/tests/test_dhla.py:84-95
    sk = P.Dhla(P.DhgParams())
    bits = np.zeros((5, 16384, 128), dtype=np.uint8)
    bits[0, 5, :81] = 0xFF
    bits[1, 9, :80] = 0xFF
    bits[1, 9, 80] = 0x7F
    sk.load_bits(bits)
    zc = sk.zero_counts()
    assert zc[0, 5] == 376 and zc[1, 9] == 377
    hot = sk.hot_sets(1024)
    assert hot[0].tolist() == [5] and hot[1].tolist() == []
    assert sk.restore_superpoints(1024) == []  # an empty hot set ends the restore


def test_empty_sketch():
    sk = P.Dhla(P.DhgParams())
    assert all(len(h) == 0 for h in sk.hot_sets(1024))
    assert sk.restore_superpoints(1024) == []
    assert sk.estimate_flow_count() == (0.0, False)
    assert sk._candidate_hosts(1024).tolist() == []


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_readout_matches_reference_fixture(case):
    sk = gpu_for_case(case)
    theta, mc = case["theta"], case["max_candidates"]
    assert sha(sk.bits) == case["bits_sha256"]
    zc = sk.zero_counts()
    assert zc.dtype == np.int64 and sha(zc) == case["zero_counts_sha256"]
    hot = sk.hot_sets(theta)
    assert [len(h) for h in hot] == case["hot_sizes"]
    assert [sha(h.astype(np.uint64)) for h in hot] == case["hot_sha256"]
    est = sk.estimate(theta)
    assert est["zero_totals"] == case["zero_totals"]
    assert est["flow_count"] == pytest.approx(case["flow_count"], rel=REL_TOL)
    assert est["flow_saturated"] == case["flow_saturated"]
    assert est["psi"] == pytest.approx(case["psi"], rel=REL_TOL)
    if "capacity_error" in case:
        with pytest.raises(P.CapacityError) as err:
            sk._candidate_hosts(theta, mc)
        assert str(err.value) == case["capacity_error"]
        with pytest.raises(P.CapacityError) as err:
            sk.restore_superpoints(theta, max_candidates=mc)
        assert str(err.value) == case["capacity_error"]
        return
    hosts = sk._candidate_hosts(theta, mc)
    assert hosts.dtype == np.uint64 and hosts.tolist() == case["candidates"]
    if case["stage_counts"]:
        assert sk.last_info["stage_counts"] == case["stage_counts"]
    assert sk.shared_zero_counts(hosts).tolist() == case["shared_zero_counts"]
    reps = sk.restore_superpoints(theta, max_candidates=mc)
    assert [r.host for r in reps] == [h for h, _, _ in case["reports"]]
    assert [r.saturated for r in reps] == [s for _, _, s in case["reports"]]
    for r, (_, e, _) in zip(reps, case["reports"]):
        assert r.estimate == pytest.approx(e, rel=REL_TOL)


@pytest.mark.parametrize("case", [c for c in CASES if c["name"] in
                                  ("small_dense", "toy_dense", "six_dense", "default_60_plants_noise1m")],
                         ids=lambda c: c["name"])
def test_readout_matches_live_oracle(case):
    """Same sketches against the C oracle's literal HE0 x HE1 x HE2 enumeration."""
    ora = oracle_for_case(case)
    sk = gpu_for_case(case)
    theta, mc = case["theta"], case["max_candidates"]
    hosts, stages = ora.candidate_hosts(theta, mc, return_stage_counts=True)
    assert sk._candidate_hosts(theta, mc).tolist() == hosts.tolist()
    assert sk.last_info["stage_counts"] == stages
    got, want = sk.restore_superpoints(theta, max_candidates=mc), ora.restore_superpoints(theta, mc)
    assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
    for a, b in zip(got, want):
        assert a.estimate == pytest.approx(b.estimate, rel=REL_TOL)


def test_config1_trace_matches_reference_fixture():
    exp = load_json("config1_expected.json")
    src, dst = config1_pairs()
    sk = P.Dhla(P.DhgParams())
    sk.update_batch(src, dst)
    assert sha(sk.bits) == exp["bits_sha256"]
    reps = sk.restore_superpoints(1024)
    assert [r.host for r in reps] == [h for h, _, _ in exp["reports"]]
    assert sorted(r.host for r in reps) == [h for h, _ in exp["truth_supers"]]
    assert sk.last_info["stage_counts"] == exp["stage_counts"]
    for r, (_, e, _) in zip(reps, exp["reports"]):
        assert r.estimate == pytest.approx(e, rel=REL_TOL)


def test_planted_host_golden_values():
    sk = P.Dhla(P.DhgParams())
    sk.update_batch(*O.plant_pairs(0xC63A1B02, 2048, 10))
    assert int(sk.shared_zero_counts([0xC63A1B02])[0]) == 147
    (rep,) = sk.restore_superpoints(1024)
    assert rep.host == 0xC63A1B02 and not rep.saturated
    assert rep.estimate == pytest.approx(1987.624160072414, rel=REL_TOL)
    est = sk.corrected_cardinality(0xC63A1B02, sk.bit_set_probability(sk.estimate_flow_count().value))
    assert est.value == pytest.approx(rep.estimate, rel=REL_TOL)


def test_restore_ties_break_by_ascending_host():
    # pkg/tests/test_dhla.py:255-269
    _, opp = O.plant_pairs(0, 2000, 12)
    sk = P.Dhla(P.DhgParams())
    for host in (5000, 4000):
        sk.update_batch(np.full(len(opp), host, dtype=np.uint32), opp)
    reps = sk.restore_superpoints(1024)
    assert [r.host for r in reps] == [4000, 5000]
    assert reps[0].estimate == reps[1].estimate


def test_all_cells_hot_large_sort_and_zero_class():
    """Every cell full: 2^16 candidates (> the single-CTA sorter's 8192), all
    saturated with estimate 0.0 (SZ clamp 1 >= denom), reported only at theta 0
    and then ordered by host alone."""
    kw = PARAM_SETS["toy"]
    sk = P.Dhla(P.DhgParams(**kw))
    full = np.full((4, 256, 8), 0xFF, dtype=np.uint8)
    sk.load_bits(full)
    ora = O.OracleSketch(**kw)
    ora.bits[:] = 0xFF
    with pytest.raises(P.CapacityError) as err:
        sk.restore_superpoints(0, max_candidates=1 << 20)
    with pytest.raises(O.OracleCapacityError) as want:
        ora.restore_superpoints(0, 1 << 20)
    assert str(err.value) == str(want.value)
    mc = 1 << 24
    hosts = sk._candidate_hosts(0, mc)
    assert hosts.tolist() == list(range(1 << 16))
    assert sk.last_info["stage_counts"] == [1 << 20, 1 << 24]
    reps = sk.restore_superpoints(0, max_candidates=mc)
    assert [r.host for r in reps] == list(range(1 << 16))
    assert all(r.saturated and r.estimate == 0.0 for r in reps)
    assert sk.restore_superpoints(1, max_candidates=mc) == []


def test_many_reports_sorted_like_the_reference():
    """65536 reports with many tied estimates through the global bitonic sorter:
    random 60%-full cells make every cell hot and every 16-bit key a candidate."""
    kw = PARAM_SETS["toy"]
    rnd = (np.random.default_rng(77).random((4, 256, 64)) < 0.6)
    bits = np.packbits(rnd, axis=2, bitorder="little")
    ora = O.OracleSketch(**kw)
    ora.bits[:] = bits
    sk = P.Dhla(P.DhgParams(**kw))
    sk.load_bits(bits)
    theta, mc = 0, 1 << 24
    want = ora.restore_superpoints(theta, mc)
    got = sk.restore_superpoints(theta, max_candidates=mc)
    assert len(want) == 1 << 16 and len({r.estimate for r in want}) > 8
    assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
    for a, b in zip(got, want):
        assert a.estimate == pytest.approx(b.estimate, rel=REL_TOL)
    theta = 3
    want = ora.restore_superpoints(theta, mc)
    got = sk.restore_superpoints(theta, max_candidates=mc)
    assert 0 < len(want) < 1 << 16
    assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]


def _random_param_sets(n, seed):
    """Valid DhgParams drawn at random (pkg/src/dhsa/dhg.py:78-105 rules), small enough for the
    oracle's literal enumeration."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        r = int(rng.integers(3, 9))
        k = int(rng.integers(4, 13))
        alpha = int(rng.integers(1, k + 1))
        w = int(rng.integers(max(8, k), 33))
        g = int(2 ** rng.integers(3, 10))
        if (r - 2) * alpha + k < w or (r - 2) * alpha + k > 64:
            continue
        out.append(dict(r=r, g=g, k=k, alpha=alpha, key_width=w,
                        seed_dh0=int(rng.integers(0, 2 ** 63)), seed_h1=int(rng.integers(0, 2 ** 63))))
    return out


@pytest.mark.parametrize("kw", _random_param_sets(24, 2024), ids=lambda kw: "r{r}g{g}k{k}a{alpha}w{key_width}".format(**kw))
def test_random_parameter_sets_match_oracle(kw):
    """Scan, zero counts, hot sets, candidates, per-stage counts, reports (or the CapacityError
    text) for parameter sets nobody hand-picked: every path choice (vector / general kernel,
    bitmap / list stage expansion, word / sub-word cells) gets exercised."""
    rng = np.random.default_rng(kw["seed_dh0"] & 0xFFFF)
    wmask = np.uint32((1 << kw["key_width"]) - 1) if kw["key_width"] < 32 else np.uint32(0xFFFFFFFF)
    cells = 1 << kw["k"]
    cand, opp = O.distinct_pairs(int(cells * kw["g"] * 0.02) + 200, int(rng.integers(1, 1000)))
    cand = cand & wmask
    theta = max(4, kw["g"] // 2)
    for n in range(3):
        c2, o2 = O.plant_pairs(int(rng.integers(0, 2 ** 32)) & int(wmask), int(theta * (1.5 + n)), 900 + n)
        cand, opp = np.concatenate([cand, c2]), np.concatenate([opp, o2])
    ora = O.OracleSketch(**kw)
    ora.update_batch(cand, opp)
    sk = P.Dhla(P.DhgParams(**kw))
    sk.update_batch(cand, opp)
    assert np.array_equal(sk.bits, ora.bits)
    assert np.array_equal(sk.zero_counts(), ora.zero_counts())
    for a, b in zip(sk.hot_sets(theta), ora.hot_sets(theta)):
        assert a.tolist() == b.tolist()
    mc = 1 << 18
    try:
        hosts, stages = ora.candidate_hosts(theta, mc, return_stage_counts=True)
    except O.OracleCapacityError as exc:
        with pytest.raises(P.CapacityError) as err:
            sk.restore_superpoints(theta, max_candidates=mc)
        assert str(err.value) == str(exc)
        return
    assert sk._candidate_hosts(theta, mc).tolist() == hosts.tolist()
    assert sk.last_info["stage_counts"] == stages
    got, want = sk.restore_superpoints(theta, max_candidates=mc), ora.restore_superpoints(theta, mc)
    assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
    for a, b in zip(got, want):
        assert a.estimate == pytest.approx(b.estimate, rel=REL_TOL)


# ----------------------------------------------------------------------- merge --


def test_merge_algebra():
    # pkg/tests/test_dhla.py:317-336
    cand, opp = O.distinct_pairs(20_000, 17)
    p = P.DhgParams()
    a, b, whole, empty = (P.Dhla(p) for _ in range(4))
    a.update_batch(cand[:10_000], opp[:10_000])
    b.update_batch(cand[10_000:], opp[10_000:])
    whole.update_batch(cand, opp)
    wb = whole.bits
    assert np.array_equal(P.merge(a, b).bits, wb)
    assert np.array_equal(P.merge(b, a).bits, wb)
    assert np.array_equal(P.merge(a, empty).bits, a.bits)
    m = P.merge(a, b)
    assert m.restore_superpoints(1024) == whole.restore_superpoints(1024)


def test_merge_rejects_parameter_mismatch():
    # pkg/tests/test_dhla.py:339-344
    p = P.DhgParams()
    other = P.DhgParams(seed_h1=p.seed_h1 + 1)
    with pytest.raises(P.ConfigError) as err:
        P.merge(P.Dhla(p), P.Dhla(other))
    assert str(p.seed_h1) in str(err.value) and str(other.seed_h1) in str(err.value)


def test_or_merge_peers_slices_equal_whole_merge():
    """The multi-GPU merge protocol on one device: each 'rank' ORs its byte range."""
    import ctypes as C

    from paper_1803_11449_b200 import _cabi

    p = P.DhgParams()
    parts = []
    for s in range(4):
        sk = P.Dhla(p)
        sk.update_batch(*O.distinct_pairs(30_000, 40 + s))
        parts.append(sk)
    want = parts[0].bits
    for sk in parts[1:]:
        want |= sk.bits
    n = p.sketch_bytes
    dst = parts[0]
    for sk in parts[1:]:
        sk.seal()
    ptrs = (C.c_void_p * 3)(*[sk.bits_device_ptr for sk in parts[1:]])
    cuts = [0, n // 4, n // 2, 3 * n // 4, n]
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        _cabi.check(_cabi.lib().dhsa_or_merge_peers(dst._h, ptrs, 3, lo, hi))
    assert np.array_equal(dst.bits, want)


# ------------------------------------------------- BASELINE sizes, by property --


def _window(n_packets, n_hosts, n_scanners, seed):
    """Distinct flows of a synthetic window + a shuffled, repeated packet stream on the GPU."""
    import torch

    rng = np.random.default_rng(seed)
    hosts = np.unique(rng.integers(0, 2 ** 32, size=n_hosts + n_scanners + 64, dtype=np.uint64))
    rng.shuffle(hosts)
    hosts = hosts[: n_hosts + n_scanners].astype(np.uint32)
    cards = np.minimum(rng.zipf(1.5, size=n_hosts), 256)
    cards = np.concatenate([cards, rng.integers(2048, 8193, size=n_scanners)])
    src = np.repeat(hosts, cards)
    dst = rng.integers(0, 2 ** 32, size=len(src), dtype=np.uint64).astype(np.uint32)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    pick = torch.randint(0, len(src), (n_packets,), device="cuda", generator=g)
    pick[: len(src)] = torch.arange(len(src), device="cuda")  # every flow at least once
    ct = torch.from_numpy(src.view(np.int32)).cuda()[pick]
    ot = torch.from_numpy(dst.view(np.int32)).cuda()[pick]
    return src, dst, ct, ot, hosts[n_hosts:]


@pytest.mark.parametrize("mode", ["flow_cache", "test_agg", "test", "red"])
def test_100m_packet_window_bits_and_superpoints_equal_oracle(mode):
    """BASELINE config 2 size.  The oracle scans the distinct flows only; the GPU
    scans all 100M packets; bits, super point set and estimates must agree."""
    src, dst, ct, ot, scanners = _window(100_000_000, 150_000, 50, seed=100)
    ora = O.OracleSketch()
    ora.update_batch(src, dst, threads=8)
    sk = P.Dhla(P.DhgParams())
    sk.set_scan_mode(mode)
    sk.update_batch(ct, ot)
    assert sha(sk.bits) == sha(ora.bits)
    got, want = sk.restore_superpoints(1024), ora.restore_superpoints(1024)
    assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
    assert set(scanners.tolist()) <= {r.host for r in got}
    for a, b in zip(got, want):
        assert a.estimate == pytest.approx(b.estimate, rel=REL_TOL)
    # idempotence at full size: a second pass over the same window changes nothing
    before = sk.estimate()["zero_totals"]
    sk.update_batch(ct, ot)
    assert sk.estimate()["zero_totals"] == before


def test_sharded_scan_plus_or_merge_equals_single_scan():
    """BASELINE config 3 shape on one device: 8 private sketches over 8 slices of
    the window, OR-merged, equal one sketch over the whole window."""
    src, dst, ct, ot, _ = _window(16_000_000, 100_000, 30, seed=101)
    whole = P.Dhla(P.DhgParams())
    whole.update_batch(ct, ot)
    shards = []
    per = (len(ct) // 8 + 3) & ~3
    for rnk in range(8):
        sk = P.Dhla(P.DhgParams())
        sk.update_batch(ct[rnk * per:(rnk + 1) * per], ot[rnk * per:(rnk + 1) * per])
        shards.append(sk)
    for sk in shards[1:]:
        shards[0].merge_from(sk)
    assert sha(shards[0].bits) == sha(whole.bits)
    assert shards[0].restore_superpoints(1024) == whole.restore_superpoints(1024)


# ------------------------------------------ multi-process merge over CUDA IPC --


def _ipc_rank(rank, world, port, mode, q):
    import os

    import torch.distributed as dist

    from paper_1803_11449_b200.multi import ShardedWindow, packet_slice

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cand, opp = O.distinct_pairs(300_000, 55)
        for n, host in enumerate((0x0A0B0C0D, 0x01020304, 0xC63A1B02)):
            c2, o2 = O.plant_pairs(host, 2048 + 100 * n, 70 + n)
            cand, opp = np.concatenate([cand, c2]), np.concatenate([opp, o2])
        order = np.random.default_rng(3).permutation(len(cand))
        cand, opp = cand[order], opp[order]
        lo, hi = packet_slice(len(cand), rank, world)
        win = ShardedWindow(P.DhgParams(), theta=1024, device=0, merge=mode)
        win.scan(cand[lo:hi], opp[lo:hi])
        used = win.merge()
        ora = O.OracleSketch()
        ora.update_batch(cand, opp, threads=2)
        want = ora.restore_superpoints(1024)
        if mode == "partition":
            # the merged bits stay with their owners: this rank holds its own range, reads the zero counts as
            # gathered and every candidate cell from the rank that owns it
            from paper_1803_11449_b200.multi import partition_ranges
            blo, bhi = partition_ranges(win.ops, world)[rank]
            mine = np.array_equal(win.sketch.bits.reshape(-1)[blo:bhi], ora.bits.reshape(-1)[blo:bhi])
            hosts = np.array([r.host for r in want] + [12345], dtype=np.uint64)
            mine = (mine and np.array_equal(win.sketch.zero_counts(), ora.zero_counts())
                    and np.array_equal(win.sketch.shared_zero_counts(hosts), ora.shared_zero_counts(hosts))
                    and np.array_equal(win.sketch._candidate_hosts(1024), ora.candidate_hosts(1024)))
        else:
            mine = np.array_equal(win.sketch.bits, ora.bits)
        got = win.restore()
        ok = (mine
              and [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
              and all(abs(a.estimate - b.estimate) <= 1e-6 * b.estimate for a, b in zip(got, want))
              and len(got) == 3)
        # a second window on the same sketches: peers stay mapped, the agreed merge kind is reused
        opened = len(win.ops._opened)
        win.reset()
        win.scan(cand[lo:hi][::2].copy(), opp[lo:hi][::2].copy())
        used2 = win.merge()
        ora2 = O.OracleSketch()
        ora2.update_batch(np.concatenate([cand[packet_slice(len(cand), r, world)[0]:packet_slice(len(cand), r, world)[1]][::2]
                                          for r in range(world)]),
                          np.concatenate([opp[packet_slice(len(cand), r, world)[0]:packet_slice(len(cand), r, world)[1]][::2]
                                          for r in range(world)]), threads=2)
        ok = ok and used2 == used and len(win.ops._opened) == opened == (0 if mode == "allgather" else world - 1)
        if mode == "partition":
            got2, want2 = win.restore(), ora2.restore_superpoints(1024)
            ok = ok and np.array_equal(win.sketch.zero_counts(), ora2.zero_counts()) \
                and [(r.host, r.saturated) for r in got2] == [(r.host, r.saturated) for r in want2]
        else:
            ok = ok and np.array_equal(win.sketch.bits, ora2.bits)
        q.put((rank, used, bool(ok)))
        dist.barrier()
        win.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world, mode", [(2, "p2p"), (3, "p2p"), (2, "allgather"), (2, "partition"), (3, "partition")])
def test_sharded_window_merges_over_cuda_ipc_between_processes(world, mode):
    """The real multi-process path -- one process per rank, sketches exported with
    cudaIpcGetMemHandle, peers mapped with cudaIpcOpenMemHandle, k_or_merge and
    k_copy_slice reading the mapped pointers -- with every rank on this one GPU
    (gloo does the rendezvous because NCCL refuses two ranks on one device)."""
    import os

    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 1000 + world + {"p2p": 0, "allgather": 7, "partition": 13}[mode]
    procs = [ctx.Process(target=_ipc_rank, args=(r, world, port, mode, q)) for r in range(world)]
    for p_ in procs:
        p_.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    assert sorted(r[0] for r in results) == list(range(world))
    assert all(used == mode and ok for _, used, ok in results), results


def _nccl_single_rank(port, q):
    import os

    import torch
    import torch.distributed as dist

    from paper_1803_11449_b200.multi import CudaMergeOps

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        sk = P.Dhla(P.DhgParams())
        ops = CudaMergeOps(sk)
        cand, opp = O.distinct_pairs(50_000, 3)
        results = []
        for stream in (None, torch.cuda.Stream()):          # the sketch's own stream, then a torch stream
            if stream is not None:
                sk.use_stream(stream.cuda_stream)
            sk.update_batch(cand, opp)
            results.append(ops.device_barrier(dist))         # a stream-ordered all-reduce behind the scan
            results.append(ops.device_barrier(dist))
            sk.seal()
        torch.cuda.synchronize()
        q.put((results, int(ops._token.item())))
    finally:
        dist.destroy_process_group()


def test_device_barrier_is_a_stream_ordered_nccl_all_reduce():
    """The merge's barriers under NCCL (multi.CudaMergeOps.device_barrier): enqueued on the sketch's
    stream, no host synchronisation.  One rank is all this box can give NCCL; the call sequence, the
    stream hand-over and the token are what is checked."""
    import os

    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p_ = ctx.Process(target=_nccl_single_rank, args=(29900 + os.getpid() % 1000, q))
    p_.start()
    results, token = q.get(timeout=300)
    p_.join(timeout=60)
    assert p_.exitcode == 0
    assert results == [True] * 4 and token == 0


# ------------------------------------------ max_candidates is a bound, not an allocation --


def test_huge_max_candidates_is_a_bound_not_an_allocation():
    """The reference treats max_candidates purely as a bound (pkg/src/dhsa/dhla.py:34,269-273); callers pass
    huge values for "unlimited".  The stage workspaces start at the default bound and grow on demand."""
    sk = P.Dhla(P.DhgParams())
    for n, host in enumerate((0x0A0B0C0D, 0xC63A1B02, 0x01020304)):
        sk.update_batch(*O.plant_pairs(host, 2048 + 300 * n, 20 + n))
    ora = O.OracleSketch()
    for n, host in enumerate((0x0A0B0C0D, 0xC63A1B02, 0x01020304)):
        ora.update_batch(*O.plant_pairs(host, 2048 + 300 * n, 20 + n))
    want = ora.restore_superpoints(1024)
    for bound in (1 << 40, 1 << 62):
        got = sk.restore_superpoints(1024, max_candidates=bound)
        assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
        assert sk._candidate_hosts(1024, max_candidates=bound).tolist() == sorted(r.host for r in want)
    sk.restore_superpoints_begin(1024, max_candidates=1 << 40)
    assert [r.host for r in sk.restore_superpoints_end()] == [r.host for r in want]


_GROWTH_SCRIPT = r"""
import json, sys
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import numpy as np
import paper_1803_11449_b200 as P
from helpers import restore_cases, case_batches
case = next(c for c in restore_cases() if c["name"] == "six_dense")
sk = P.Dhla(P.DhgParams(**case["params"]))
for c, o in case_batches(case):
    sk.update_batch(c, o)
out = {}
got = sk.restore_superpoints(case["theta"], max_candidates=1 << 30)        # synchronous: grows and reruns
out["stage_counts"] = sk.last_info["stage_counts"]
out["reports"] = [[r.host, r.estimate, r.saturated] for r in got]
out["candidates"] = sk._candidate_hosts(case["theta"], max_candidates=1 << 30).tolist()
tiny = P.Dhla(P.DhgParams(r=6, g=512, k=12, alpha=5, seed_dh0=99))           # other seeds: a new sketch, small buffers
for c, o in case_batches(case):
    tiny.update_batch(c, o)
tiny.restore_superpoints_begin(case["theta"], max_candidates=1 << 30)
tiny.reset()                                                                 # the next window is already in the bits
try:
    tiny.restore_superpoints_end()
    out["async_after_reset"] = "no error"
except P.ConfigError as exc:
    out["async_after_reset"] = str(exc)
tiny2 = P.Dhla(P.DhgParams(r=6, g=512, k=12, alpha=5, seed_dh0=98))
for c, o in case_batches(case):
    tiny2.update_batch(c, o)
tiny2.restore_superpoints_begin(case["theta"], max_candidates=1 << 30)       # untouched sketch: collected after growing
out["async_untouched"] = len(tiny2.restore_superpoints_end())
try:
    sk.restore_superpoints(case["theta"], max_candidates=1000)               # the bound itself still raises
    out["capacity"] = "no error"
except P.CapacityError as exc:
    out["capacity"] = str(exc)
print(json.dumps(out))
"""


def test_stage_workspaces_grow_on_demand_and_the_counts_stay_exact():
    """With the workspaces started at 4096 entries (DHSA_INITIAL_CANDIDATES), the dense six-array fixture --
    stage survivors [91677, 167552, 296923, 462877] -- has to grow them several times; counts, candidates and
    reports are the fixture's, a bound below the first stage still raises the reference's CapacityError, and a
    pipelined read-out that cannot be rerun (the window was reset meanwhile) says so instead of truncating."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DHSA_INITIAL_CANDIDATES="4096")
    proc = subprocess.run([sys.executable, "-c", _GROWTH_SCRIPT, root], capture_output=True, text=True, env=env, timeout=600)
    assert proc.returncode == 0, proc.stderr[-2000:]
    out = json.loads(proc.stdout.strip().splitlines()[-1])
    case = next(c for c in CASES if c["name"] == "six_dense")
    assert out["stage_counts"] == case["stage_counts"] == [91677, 167552, 296923, 462877]
    assert out["candidates"] == case["candidates"]
    assert [(h, s) for h, _, s in out["reports"]] == [(h, s) for h, _, s in case["reports"]]
    for (_, a, _), (_, b, _) in zip(out["reports"], case["reports"]):
        assert a == pytest.approx(b, rel=REL_TOL)
    assert out["capacity"] == "restore stage 1 produced 91677 partial keys (max_candidates=1000)"
    assert "sketch was modified" in out["async_after_reset"] and out["async_untouched"] >= 0
