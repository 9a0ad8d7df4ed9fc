"""Closed forms and statistical laws the reference's own suite pins for the read-out
(pkg/tests/test_dhla.py:97-221), run against the device sketch through the C ABI."""
import math

import numpy as np
import pytest

import paper_1803_11449_b200 as P
from paper_1803_11449_b200 import dhg
from oracle import oracle as O

pytestmark = pytest.mark.gpu

SMALL = dict(r=5, g=256, k=10, alpha=8, key_width=32, seed_dh0=1, seed_h1=2)


def plant(sk, host, fanout, seed):
    sk.update_batch(*O.plant_pairs(host, fanout, seed))


def test_super_host_estimators_all_become_hot_and_hot_sets_only_grow():
    # pkg/tests/test_dhla.py:101-118
    p = P.DhgParams()
    sk = P.Dhla(p)
    host = 0x0A0B0C0D
    plant(sk, host, 2048, 5)
    hot = sk.hot_sets(1024)
    for i, j in enumerate(dhg.forward(p, host)):
        assert j in set(hot[i].tolist())
    before = [set(h.tolist()) for h in hot]
    sk.update_batch(*O.distinct_pairs(50_000, 7))
    after = [set(h.tolist()) for h in sk.hot_sets(1024)]
    assert all(b <= a for b, a in zip(before, after))


def test_flow_count_closed_forms():
    # empty sketch: exactly 0.0, not saturated (pkg/tests/test_dhla.py:124-127)
    est = P.Dhla(P.DhgParams()).estimate_flow_count()
    assert est.value == 0.0 and not est.saturated
    # zero ratio 1/e -> the estimate is the capacity (pkg/tests/test_dhla.py:130-145)
    p = P.DhgParams(**SMALL)
    capacity = p.g * p.index_count
    flat = np.zeros(capacity, dtype=np.uint8)
    flat[: capacity - round(capacity / math.e)] = 1
    one = np.packbits(flat, bitorder="little").reshape(p.index_count, p.g // 8)
    sk = P.Dhla(p)
    sk.load_bits(np.stack([one] * p.r))
    assert sk.estimate_flow_count().value == pytest.approx(capacity, rel=1e-5)
    # every bit set: evaluated at one zero bit, flagged saturated (pkg/src/dhsa/estimator.py:26-34)
    sk.load_bits(np.full((p.r, p.index_count, p.g // 8), 0xFF, dtype=np.uint8))
    full = sk.estimate_flow_count()
    assert full.saturated and full.value == pytest.approx(capacity * math.log(capacity), rel=1e-12)


def test_flow_count_tracks_distinct_pairs():
    # pkg/tests/test_dhla.py:148-153: mean over 20 traces within 5% of the truth
    sk = P.Dhla(P.DhgParams())
    values = []
    for seed in range(20):
        sk.reset()
        sk.update_batch(*O.distinct_pairs(100_000, 30 + seed))
        values.append(sk.estimate_flow_count().value)
    assert abs(np.mean(values) - 100_000) / 100_000 <= 0.05


def test_bit_set_probability_closed_forms_and_observed_fill():
    # pkg/tests/test_dhla.py:156-174
    sk = P.Dhla(P.DhgParams())
    assert sk.bit_set_probability(0.0) == 0.0
    assert sk.bit_set_probability(1024 * 16384) == pytest.approx(0.6321205588285577)
    p = P.DhgParams(r=3, g=256, k=10, alpha=10, key_width=20, seed_dh0=5, seed_h1=6)
    capacity = p.g * p.index_count
    small = P.Dhla(p)
    fractions = []
    for seed in range(5):
        small.reset()
        small.update_batch(*O.distinct_pairs(capacity, 60 + seed))
        fractions.append((capacity * p.r - small.zero_counts().sum()) / (capacity * p.r))
    assert abs(np.mean(fractions) - small.bit_set_probability(capacity)) <= 0.02


def test_corrected_cardinality_closed_forms():
    p = P.DhgParams()
    # psi = 0: the plain linear estimate of the intersection of the host's r cells
    # (pkg/tests/test_dhla.py:180-189; the intersection is rebuilt here from estimator(i, j))
    sk = P.Dhla(p)
    host = 0x11223344
    plant(sk, host, 600, 8)
    cells = [sk.estimator(i, j) for i, j in enumerate(dhg.forward(p, host))]
    inter = np.bitwise_and.reduce(np.stack(cells), axis=0)
    zeros = p.g - int(np.unpackbits(inter).sum())
    est = sk.corrected_cardinality(host, psi=0.0)
    assert est.value == pytest.approx(-p.g * math.log(zeros / p.g)) and not est.saturated
    # idle host: estimate 0.0 (pkg/tests/test_dhla.py:192-194)
    assert P.Dhla(p).corrected_cardinality(0x7F000001, psi=0.0).value == 0.0
    # full intersection: saturated, evaluated at one zero bit (pkg/tests/test_dhla.py:197-203)
    sat = P.Dhla(p)
    plant(sat, 99, 20_000, 9)
    e = sat.corrected_cardinality(99, sat.bit_set_probability(sat.estimate_flow_count().value))
    assert e.saturated and e.value == pytest.approx(-1024 * math.log(1 / 1024), rel=1e-3)


def test_correction_tracks_truth_with_heavy_background():
    # pkg/tests/test_dhla.py:206-221: at small g the sharing correction must help, and land within 10%
    p = P.DhgParams(r=5, g=256, k=8, alpha=8, key_width=32, seed_dh0=7, seed_h1=8)
    host, fanout = 0x0A000001, 300
    corrected, plain = [], []
    sk = P.Dhla(p)
    for seed in range(10):
        sk.reset()
        plant(sk, host, fanout, 100 + seed)
        cand, opp = O.distinct_pairs(60_000, 200 + seed)
        sk.update_batch(np.where(cand == host, cand + 1, cand), opp)
        psi = sk.bit_set_probability(sk.estimate_flow_count().value)
        corrected.append(sk.corrected_cardinality(host, psi).value)
        plain.append(sk.corrected_cardinality(host, 0.0).value)
    assert abs(np.mean(corrected) - fanout) < abs(np.mean(plain) - fanout)
    assert abs(np.mean(corrected) - fanout) / fanout <= 0.10


def test_restore_capacity_overflow_aborts_loudly_with_the_reference_text():
    # pkg/tests/test_dhla.py (CapacityError): never a silent truncation, stage number and count in the text
    sk = P.Dhla(P.DhgParams())
    for n, host in enumerate(range(0x0B000000, 0x0B000000 + 40)):
        plant(sk, host, 2048, 300 + n)
    ora = O.OracleSketch()
    for n, host in enumerate(range(0x0B000000, 0x0B000000 + 40)):
        ora.update_batch(*O.plant_pairs(host, 2048, 300 + n))
    with pytest.raises(O.OracleCapacityError) as want:
        ora.restore_superpoints(1024, max_candidates=100)
    with pytest.raises(P.CapacityError) as got:
        sk.restore_superpoints(1024, max_candidates=100)
    assert str(got.value) == str(want.value)
    assert len(sk.restore_superpoints(1024)) == 40          # the default budget restores them all


def test_in_place_writes_to_bits_reach_the_device():
    # the reference paints cells through the live array (pkg/tests/test_dhla.py:85-95; test_kernels.py:53-59)
    p = P.DhgParams()
    sk = P.Dhla(p)
    sk.bits[0, 5, :81] = 0xFF        # 648 ones -> 376 zeros
    sk.bits[1, 9, :80] = 0xFF
    sk.bits[1, 9, 80] = 0x7F         # 647 ones -> 377 zeros
    zc = sk.zero_counts()
    assert zc[0, 5] == 376 and zc[1, 9] == 377 and int(zc.sum()) == p.r * p.index_count * p.g - 648 - 647
    hot = sk.hot_sets(1024)
    assert 5 in hot[0] and 9 not in hot[1]
    small = P.DhgParams(r=3, g=8, k=8, alpha=8, key_width=16)
    sk = P.Dhla(small)
    paint = np.random.default_rng(4).integers(0, 256, size=sk.bits.shape, dtype=np.uint8)
    sk.bits[:] = paint
    assert np.array_equal(sk.bits, paint)
    assert np.array_equal(sk.zero_counts(), small.g - np.unpackbits(paint, axis=2).sum(axis=2))
    copy = sk.bits.copy()
    copy[:] = 0                      # a copy is detached
    assert np.array_equal(sk.bits, paint)
    # a scan after a painted upload still lands (the flow cache was emptied by the upload)
    sk.update_batch(np.array([1, 2, 3], np.uint32), np.array([4, 5, 6], np.uint32))
    assert np.array_equal(sk.bits & paint, paint)
