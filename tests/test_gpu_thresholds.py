"""Both threshold decisions of the read-out as integer compares.

hot  <=> zc < g exp(-theta/g)  <=> zc <= hot_cut        (pkg/src/dhsa/dhla.py:45-47,111-119)
keep <=> -g ln(SZ'/denom) >= theta <=> SZ' <= sz_cut    (pkg/src/dhsa/dhla.py:183-194)
with both cuts derived on the host from the reference's own float64 formulas.  The tests paint
cells directly (as pkg/tests/test_dhla.py:84-95 does) so SZ and zc take every value around a cut.
"""
import math

import numpy as np
import pytest

import paper_1803_11449_b200 as P
from paper_1803_11449_b200 import dhg
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _paint(bits, params, host, zeros):
    """Give each of the host's r cells exactly `zeros` zero bits (the first ones): SZ == zeros."""
    g = params.g
    cell = np.zeros(g // 8, dtype=np.uint8)
    ones = np.arange(zeros, g)
    np.bitwise_or.at(cell, ones >> 3, (1 << (ones & 7)).astype(np.uint8))
    for i, j in enumerate(dhg.forward(params, host)):
        bits[i, j] = cell


def _reference_cut(g, denom, theta):
    """The largest SZ' whose estimate, by the reference's formula, reaches theta (0: none)."""
    best = 0
    for sz in range(1, g + 1):
        est = 0.0 if sz >= denom else -g * math.log(sz / denom)
        if est >= theta:
            best = sz
    return best


@pytest.mark.parametrize("theta, g", [(1024, 1024), (256, 1024), (4096, 4096), (700, 512), (1, 64)])
def test_hot_cut_equals_the_float_compare(theta, g):
    p = P.DhgParams(g=g, r=3, k=10, alpha=10, key_width=20)
    zmin = P.hot_threshold(g, theta)
    want_cut = max((z for z in range(0, g + 1) if z < zmin), default=-1)
    sk = P.Dhla(p)
    bits = np.zeros((p.r, p.index_count, g // 8), dtype=np.uint8)
    values = sorted({0, 1, g} | {min(g, max(0, want_cut + d)) for d in (-2, -1, 0, 1, 2)})
    for n, zeros in enumerate(values):            # cell n of array 0 gets `zeros` zero bits
        ones = np.arange(zeros, g)
        np.bitwise_or.at(bits[0, n], ones >> 3, (1 << (ones & 7)).astype(np.uint8))
    sk.load_bits(bits)
    hot = sk.hot_sets(theta)[0].tolist()
    assert hot == [n for n, zeros in enumerate(values) if zeros < zmin]
    assert sk.estimate(theta)["hot_cut"] == want_cut


def test_report_filter_straddles_theta_by_one_sz_step():
    """Hosts whose SZ sits on either side of the cut, one step apart: exactly those at or below
    sz_cut are reported -- over background fill levels (psi) that move the cut."""
    p = P.DhgParams()
    theta = 1024
    rng = np.random.default_rng(3)
    sk = P.Dhla(p)
    ora = O.OracleSketch()
    shape = (p.r, p.index_count, p.g // 8)
    rand = lambda: rng.integers(0, 256, size=shape, dtype=np.uint8)
    backgrounds = {0.0: lambda: np.zeros(shape, np.uint8), 0.25: lambda: rand() & rand(),
                   0.4375: lambda: (rand() & rand()) | (rand() & rand()), 0.5: rand}
    seen_cuts = set()
    for trial, (density, make) in enumerate(list(backgrounds.items()) * 2):
        bits = make()
        sk.load_bits(bits)
        info = sk.estimate(theta)
        assert info["psi"] == pytest.approx(density, abs=2e-3)
        cut = info["sz_cut"]
        assert cut == _reference_cut(p.g, info["denom"], theta)
        hosts = {0x0A000000 + 7919 * (trial + 1) + 104729 * d: cut + d for d in (-1, 0, 1, 2)}
        for host, zeros in hosts.items():
            _paint(bits, p, host, zeros)
        sk.load_bits(bits)
        ora.bits[:] = bits
        got, want = sk.restore_superpoints(theta), ora.restore_superpoints(theta)
        assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
        assert all(a.estimate == pytest.approx(b.estimate, rel=1e-12) for a, b in zip(got, want))
        assert sk.shared_zero_counts(list(hosts)).tolist() == list(hosts.values())
        new_cut = sk.last_info["sz_cut"]                # painting four hosts may move psi by a hair
        assert new_cut == _reference_cut(p.g, sk.last_info["denom"], theta)
        assert new_cut in hosts.values() and new_cut + 1 in hosts.values()      # one SZ step apart, both sides
        assert {r.host for r in got} == {h for h, z in hosts.items() if z <= new_cut}
        seen_cuts.add(new_cut)
    assert len(seen_cuts) >= 3                          # 376 on an empty sketch down to 365 at psi = 0.5


def test_report_cut_equals_reference_formula_for_many_psi():
    """10^4 random fill states: sz_cut from the read-out == the cut the reference's float64 formula
    gives for the same zero totals (the filter is then an integer compare on exact SZ values)."""
    p = P.DhgParams(r=3, g=1024, k=8, alpha=8, key_width=16)
    sk = P.Dhla(p)
    rng = np.random.default_rng(11)
    cap = p.g * p.index_count
    checked = 0
    for trial in range(40):
        zc = rng.integers(0, p.g + 1, size=(p.r, p.index_count)).astype(np.int64)
        if trial % 4 == 0:
            zc[:] = p.g - rng.integers(0, 3, size=zc.shape)       # nearly empty sketch: psi ~ 0
        for theta in rng.integers(1, 7000, size=250):
            info = sk.estimate(float(theta), zero_counts=zc)
            flow = sum(-cap * math.log((int(z) or 1) / cap) for z in zc.sum(axis=1)) / p.r
            psi = 1.0 - math.exp(-flow / cap)
            denom = p.g * (1.0 - psi ** p.r)
            assert info["flow_count"] == flow and info["psi"] == psi and info["denom"] == denom   # bit-equal: host libm
            assert info["sz_cut"] == _reference_cut(p.g, denom, float(theta))
            checked += 1
    assert checked == 10_000


def test_zero_counts_argument_is_used_not_ignored():
    # pkg/src/dhsa/dhla.py:111-128: hot_sets / estimate_flow_count take the counts they are given
    p = P.DhgParams()
    sk = P.Dhla(p)
    sk.update_batch(*O.distinct_pairs(10_000, 3))
    zc = np.full((p.r, p.index_count), p.g, dtype=np.int64)
    zc[:, 5] = 100
    zc[2, 9] = 376
    zc[2, 10] = 377
    hot = sk.hot_sets(1024, zero_counts=zc)
    assert [h.tolist() for h in hot] == [[5], [5], [5, 9], [5], [5]]
    own = sk.hot_sets(1024)                              # the hand-in is one-shot
    assert all(len(h) == 0 for h in own)
    flow = sk.estimate_flow_count(zero_counts=zc)
    cap = p.g * p.index_count
    want = sum(-cap * math.log(int(z) / cap) for z in zc.sum(axis=1)) / p.r
    assert flow.value == want and not flow.saturated
    assert sk.estimate_flow_count().value == pytest.approx(10_000, rel=0.02)
    with pytest.raises(ValueError):
        sk.hot_sets(1024, zero_counts=zc[:, :100])
