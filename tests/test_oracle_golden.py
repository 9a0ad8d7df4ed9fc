"""Pins the CPU oracle (oracle/dhsa_oracle.c) to the reference.

Sources of truth, in order:
  * constants the reference's own tests assert
    (pkg/tests/test_dhla.py:43,86-95; pkg/tests/test_estimator.py:57-62;
     pkg/tests/test_dhla.py:159-163,216-221);
  * tests/golden/*.json|npz, recorded from the live reference package by
    tests/golden/make_golden.py (compiled backend);
  * when oracle/_ref holds the reference's own compiled loops, a direct
    byte-for-byte comparison against them.
"""
import hashlib
import math

import numpy as np
import pytest

from oracle import oracle as O

from helpers import (case_batches, config1_pairs, load_json, oracle_for_case, restore_cases)

CONST = load_json("constants.json")
CASES = restore_cases()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_states_and_mix64_match_reference():
    sk = O.OracleSketch()
    assert sk.state_dh0 == CONST["state_dh0"] == 0x9DA44F6E0275D406
    assert sk.state_h1 == CONST["state_h1"] == 0x7644699CA1FCAE3B
    for x, want in CONST["mix64"].items():
        assert O.mix64(int(x)) == want
    xs = np.random.default_rng(1).integers(0, 2 ** 64, size=500, dtype=np.uint64)
    vec = O.mix64_many(xs)
    for x, v in zip(xs.tolist(), vec.tolist()):
        assert O.mix64(x) == v


def test_forward_and_h1_match_reference():
    sk = O.OracleSketch()
    for a, want in CONST["forward"].items():
        assert list(sk.forward(int(a))) == want
    for b, want in CONST["h1"].items():
        assert sk.h1(int(b)) == want
    assert sk.forward(0xC0A80101) == (7363, 7618, 15559, 5699, 11497)
    assert sk.h1(0x08080808) == 378


def test_reconstruct_key_matches_reference():
    sk = O.OracleSketch()
    for key, idx, good, bad in CONST["reconstruct"]:
        assert sk.reconstruct_key(idx) == good == key
        corrupted = list(idx)
        corrupted[2] ^= 1
        assert sk.reconstruct_key(corrupted) == bad


def test_exhaustive_16bit_reconstruction():
    # pkg/tests/test_dhg.py:84-89
    sk = O.OracleSketch(r=4, g=64, k=8, alpha=4, key_width=16)
    for key in range(0, 1 << 16, 7):
        assert sk.reconstruct_key(sk.forward(key)) == key


def test_single_update_sets_exactly_r_bits():
    sk = O.OracleSketch()
    sk.update(0xC0A80101, 0x08080808)
    got = [[int(i), int(j), int(b), int(sk.bits[i, j, b])] for i, j, b in np.argwhere(sk.bits)]
    assert got == CONST["single_update"]
    assert int(np.unpackbits(sk.bits).sum()) == 5
    assert sk.bits.nbytes == CONST["sketch_bytes"] == 10_485_760  # pkg/tests/test_dhla.py:43


def test_hot_threshold_constants():
    # pkg/tests/test_dhla.py:86
    assert O.lib().oracle_hot_threshold(1024, 1024.0) == pytest.approx(376.70854775955695, abs=0)
    for key, want in CONST["hot_threshold"].items():
        g, t = (int(v) for v in key.split(","))
        assert O.lib().oracle_hot_threshold(g, float(t)) == want


def test_hot_boundary_376_hot_377_not():
    # pkg/tests/test_dhla.py:84-95
    sk = O.OracleSketch()
    sk.bits[0, 5, :81] = 0xFF
    sk.bits[1, 9, :80] = 0xFF
    sk.bits[1, 9, 80] = 0x7F
    zc = sk.zero_counts()
    assert zc[0, 5] == 376 and zc[1, 9] == 377
    hot = sk.hot_sets(1024)
    assert 5 in hot[0] and 9 not in hot[1]


@pytest.mark.parametrize("g", [8, 64])
def test_zero_counts_match_unpackbits(g):
    # pkg/tests/test_kernels.py:51-59
    sk = O.OracleSketch(r=3, g=g, k=8, alpha=8, key_width=16)
    sk.bits[:] = np.random.default_rng(4).integers(0, 256, size=sk.bits.shape, dtype=np.uint8)
    assert np.array_equal(sk.zero_counts(), g - np.unpackbits(sk.bits, axis=2).sum(axis=2))


def test_estimator_closed_forms():
    sk = O.OracleSketch()
    # pkg/tests/test_estimator.py:57-62: half-full 1024-bit vector -> 709.78
    assert -1024 * math.log(512 / 1024) == pytest.approx(709.78, abs=0.01)
    assert sk.bit_set_probability(0.0) == 0.0
    assert sk.bit_set_probability(1024 * 16384) == pytest.approx(0.6321205588285577)
    assert sk.estimate_flow_count() == (0.0, False)
    est, sat = sk.corrected_estimate(0, 0.0)
    assert sat and est == pytest.approx(-1024 * math.log(1 / 1024))
    assert sk.corrected_estimate(1024, 0.0) == (0.0, False)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_readout_matches_reference_fixture(case):
    sk = oracle_for_case(case)
    theta = case["theta"]
    assert sha(sk.bits) == case["bits_sha256"]
    zc = sk.zero_counts()
    assert sha(zc) == case["zero_counts_sha256"]
    assert [int(v) for v in sk.zero_totals(zc)] == case["zero_totals"]
    hot = sk.hot_sets(theta, zc)
    assert [len(h) for h in hot] == case["hot_sizes"]
    assert [sha(h) for h in hot] == case["hot_sha256"]
    flow, sat = sk.estimate_flow_count(zc)
    assert flow == pytest.approx(case["flow_count"], rel=1e-12) and sat == case["flow_saturated"]
    assert sk.bit_set_probability(flow) == pytest.approx(case["psi"], rel=1e-12)
    mc = case["max_candidates"]
    if "capacity_error" in case:
        with pytest.raises(O.OracleCapacityError) as err:
            sk.candidate_hosts(theta, mc)
        assert str(err.value) == case["capacity_error"]
        with pytest.raises(O.OracleCapacityError) as err:
            sk.restore_superpoints(theta, mc)
        assert str(err.value) == case["capacity_error"]
        return
    hosts, stages = sk.candidate_hosts(theta, mc, return_stage_counts=True)
    assert [int(h) for h in hosts] == case["candidates"]
    if case["stage_counts"]:
        assert stages == case["stage_counts"]
    assert [int(v) for v in sk.shared_zero_counts(hosts)] == case["shared_zero_counts"]
    reps = sk.restore_superpoints(theta, mc)
    assert [r.host for r in reps] == [h for h, _, _ in case["reports"]]
    assert [r.saturated for r in reps] == [s for _, _, s in case["reports"]]
    for r, (_, e, _) in zip(reps, case["reports"]):
        assert r.estimate == pytest.approx(e, rel=1e-12)


def test_config1_trace_matches_reference_fixture():
    exp = load_json("config1_expected.json")
    src, dst = config1_pairs()
    sk = O.OracleSketch()
    sk.update_batch(src, dst, threads=4)
    assert sha(sk.bits) == exp["bits_sha256"]
    reps = sk.restore_superpoints(1024)
    assert [r.host for r in reps] == [h for h, _, _ in exp["reports"]]
    assert sorted(r.host for r in reps) == [h for h, _ in exp["truth_supers"]]
    for r, (_, e, _) in zip(reps, exp["reports"]):
        assert r.estimate == pytest.approx(e, rel=1e-12)


def test_planted_host_golden_values():
    # host 0xC63A1B02, 2048 opposites, seed 10 -> SZ 147, estimate 1987.62416...
    sk = O.OracleSketch()
    sk.update_batch(*O.plant_pairs(0xC63A1B02, 2048, 10))
    assert int(sk.shared_zero_counts([0xC63A1B02])[0]) == 147
    (rep,) = sk.restore_superpoints(1024)
    assert rep.host == 0xC63A1B02 and not rep.saturated
    assert rep.estimate == pytest.approx(1987.624160072414, rel=1e-12)


def test_threaded_update_equals_sequential():
    # pkg/tests/test_kernels.py:62-74
    cand, opp = O.distinct_pairs(400_000, 5)
    a, b = O.OracleSketch(), O.OracleSketch()
    a.update_batch(cand, opp)
    b.update_batch(cand, opp, threads=8)
    assert np.array_equal(a.bits, b.bits)


def test_merge_equals_concatenated_stream():
    # pkg/tests/test_dhla.py:323-329
    cand, opp = O.distinct_pairs(20_000, 17)
    a, b, w = O.OracleSketch(), O.OracleSketch(), O.OracleSketch()
    a.update_batch(cand[:10_000], opp[:10_000])
    b.update_batch(cand[10_000:], opp[10_000:])
    w.update_batch(cand, opp)
    assert np.array_equal(a.merged_with(b).bits, w.bits)


@pytest.mark.skipif(O.load_ref_core() is None, reason="oracle/_ref not built")
@pytest.mark.parametrize("kw", [dict(), dict(r=4, g=64, k=8, alpha=4, key_width=16),
                                dict(r=3, g=8, k=8, alpha=8, key_width=16)])
def test_oracle_equals_reference_compiled_loops(kw):
    """Byte-for-byte against the reference's own update_batch / zero_counts."""
    core = O.load_ref_core()
    sk = O.OracleSketch(**kw)
    cand, opp = O.distinct_pairs(50_000, 3)
    sk.update_batch(cand, opp)
    ref_bits = np.zeros_like(sk.bits)
    core.update_batch(ref_bits, sk.state_dh0, sk.state_h1, sk.k, sk.alpha, cand, opp)
    assert np.array_equal(ref_bits, sk.bits)
    assert np.array_equal(core.zero_counts(ref_bits), sk.zero_counts())
    if not kw:
        assert sha(sk.bits) == "38d4cac25b1922468b09d87d40a536699a03d0a58ac44cdc776a8ed1995dd136"


ENGINE_CASES = load_json("engine_cases.json")


@pytest.mark.parametrize("case", ENGINE_CASES, ids=[f"{c['seed']}-{c['direction']}" for c in ENGINE_CASES])
def test_engine_oracle_matches_reference_engine_fixture(case):
    """oracle.run_windows against what the reference's DetectionEngine produced."""
    trace = O.engine_trace(case["seed"])
    assert sha(trace) == case["trace_sha256"]
    got = O.run_windows(trace, case["window_seconds"], case["theta"], case["direction"])
    assert [(w, p, d) for w, p, d, _ in got] == \
        [(w["window_id"], w["pairs"], w["dropped"]) for w in case["windows"]]
    for (_, _, _, reps), w in zip(got, case["windows"]):
        assert [(r.host, r.saturated) for r in reps] == [(h, s) for h, _, s in w["reports"]]
        for r, (_, e, _) in zip(reps, w["reports"]):
            assert r.estimate == pytest.approx(e, rel=1e-12)


EXACT_CASES = load_json("exact_cases.json")


@pytest.mark.parametrize("case", EXACT_CASES, ids=[c["direction"] for c in EXACT_CASES])
def test_exact_counts_oracle_matches_reference_fixture(case):
    truth = O.exact_counts(O.engine_trace(case["seed"]), case["direction"])
    assert len(truth) == case["n_hosts"] and sum(truth.values()) == case["n_pairs"]
    assert sha(np.array(sorted(truth), dtype=np.uint64)) == case["hosts_sha256"]
    assert sha(np.array([truth[h] for h in sorted(truth)], dtype=np.uint64)) == case["counts_sha256"]
