"""Row 8a-10: the hash group's inverse as a product function (dhsa_forward_many /
dhsa_reconstruct_many behind dhg.forward_many, dhg.reconstruct_key / reconstruct_many and the
Dhla-level methods), mirroring pkg/tests/test_dhg.py:23-101 and the C1 release criterion
(pkg/tests/test_acceptance.py:31-50)."""
import numpy as np
import pytest

import paper_1803_11449_b200 as P
from paper_1803_11449_b200 import dhg
from oracle import oracle as O

from helpers import load_json

pytestmark = pytest.mark.gpu

DEFAULTS = P.DhgParams()
TOY = P.DhgParams(r=4, g=64, k=8, alpha=4, key_width=16)     # pkg/tests/conftest.py:14-16


def test_forward_many_equals_scalar_forward_and_golden_constants():
    const = load_json("constants.json")
    keys = np.array([int(a) for a in const["forward"]], dtype=np.uint64)
    got = dhg.forward_many(DEFAULTS, keys)
    assert got.dtype == np.uint64 and got.shape == (len(keys), DEFAULTS.r)
    assert got.tolist() == [const["forward"][str(int(a))] for a in keys]
    rng = np.random.default_rng(5)
    for p in (DEFAULTS, TOY, P.DhgParams(r=6, g=512, k=12, alpha=5), P.DhgParams(r=3, g=256, k=18, alpha=14)):
        ks = rng.integers(0, 2 ** p.key_width, size=500, dtype=np.uint64)
        assert dhg.forward_many(p, ks).tolist() == [list(dhg.forward(p, int(a))) for a in ks]


def test_dh_i_xor_involution_and_range():
    # pkg/tests/test_dhg.py:23-45
    rng = np.random.default_rng(5)
    for a in rng.integers(0, 2 ** 32, size=200).tolist():
        d0 = dhg.dh0(DEFAULTS, a)
        for i in range(1, DEFAULTS.r):
            block = (a >> ((i - 1) * DEFAULTS.alpha)) % DEFAULTS.index_count
            assert dhg.dh_i(DEFAULTS, a, i) ^ d0 == block
            assert dhg.recover_block(DEFAULTS, d0, dhg.dh_i(DEFAULTS, a, i)) == block
    for i in range(1, DEFAULTS.r):
        assert dhg.dh_i(DEFAULTS, 0, i) == dhg.dh0(DEFAULTS, 0)
    for bad in (0, DEFAULTS.r):
        with pytest.raises(ValueError):
            dhg.dh_i(DEFAULTS, 1, bad)
    assert dhg.recover_block(DEFAULTS, 777, 777) == 0


def test_reconstruct_inverts_forward():
    # pkg/tests/test_dhg.py:48-51
    rng = np.random.default_rng(11)
    keys = rng.integers(0, 2 ** 32, size=5000, dtype=np.uint64)
    rebuilt, ok = dhg.reconstruct_many(DEFAULTS, dhg.forward_many(DEFAULTS, keys))
    assert ok.all() and np.array_equal(rebuilt, keys)
    for a in keys[:50].tolist():
        assert dhg.reconstruct_key(DEFAULTS, dhg.forward(DEFAULTS, a)) == a
    sk = P.Dhla(DEFAULTS)
    assert sk.reconstruct_key(dhg.forward(DEFAULTS, 0xC0A80101)) == 0xC0A80101
    assert sk.reconstruct_many(dhg.forward_many(DEFAULTS, keys[:10]))[1].all()


def test_reconstruct_rejections():
    # pkg/tests/test_dhg.py:54-74: broken overlap; a uniform XOR only the dh0 check can catch; arity
    indices = list(dhg.forward(DEFAULTS, 0xDEADBEEF))
    indices[2] ^= 1 << (DEFAULTS.k - 1)
    assert dhg.reconstruct_key(DEFAULTS, indices) is None
    indices = [v ^ 0x1F3 for v in dhg.forward(DEFAULTS, 0xC0A80101)]
    assert dhg.reconstruct_key(DEFAULTS, indices) is None
    with pytest.raises(ValueError):
        dhg.reconstruct_key(DEFAULTS, [1, 2, 3])
    with pytest.raises(ValueError):
        dhg.reconstruct_many(DEFAULTS, np.zeros((4, 3), dtype=np.uint64))
    # bits above the key width: a 24-bit key space whose blocks cover 26 bits
    p = P.DhgParams(r=4, g=32, k=10, alpha=8, key_width=24)
    tuples = dhg.forward_many(p, np.array([0x00ABCDEF], dtype=np.uint64))
    assert dhg.reconstruct_many(p, tuples)[1].all()
    tuples[0, 3] ^= np.uint64(1 << 9)          # sets key bit 25 through the last block
    assert not dhg.reconstruct_many(p, tuples)[1].any()


def test_random_tuples_essentially_never_accepted():
    # pkg/tests/test_dhg.py:77-87
    rng = np.random.default_rng(99)
    tuples = rng.integers(0, DEFAULTS.index_count, size=(100_000, DEFAULTS.r)).astype(np.uint64)
    _, ok = dhg.reconstruct_many(DEFAULTS, tuples)
    bound = 4 * 2 ** -((DEFAULTS.r - 2) * (DEFAULTS.k - DEFAULTS.alpha))
    assert ok.sum() / len(tuples) <= bound


def test_exhaustive_reconstruction_at_reduced_width():
    # pkg/tests/test_dhg.py:90-95
    keys = np.arange(1 << TOY.key_width, dtype=np.uint64)
    rebuilt, ok = dhg.reconstruct_many(TOY, dhg.forward_many(TOY, keys))
    assert ok.all() and np.array_equal(rebuilt, keys)


def test_device_reconstruct_agrees_with_the_oracle_tuple_by_tuple():
    # pkg/tests/test_dhg.py:98-107 (scalar == vectorised), here device == oracle's scalar restatement,
    # on random tuples AND on near-misses of real keys (one index perturbed), garbage keys included
    rng = np.random.default_rng(3)
    ora = O.OracleSketch(r=TOY.r, g=TOY.g, k=TOY.k, alpha=TOY.alpha, key_width=TOY.key_width)
    tuples = rng.integers(0, TOY.index_count, size=(2000, TOY.r)).astype(np.uint64)
    real = dhg.forward_many(TOY, rng.integers(0, 1 << TOY.key_width, size=2000, dtype=np.uint64))
    real[np.arange(1000), rng.integers(0, TOY.r, size=1000)] ^= np.uint64(1) << rng.integers(0, TOY.k, size=1000).astype(np.uint64)
    tuples = np.concatenate([tuples, real])
    rebuilt, ok = dhg.reconstruct_many(TOY, tuples)
    assert 900 <= int(ok.sum()) <= 1100 + 50
    for row, key, accepted in zip(tuples.tolist(), rebuilt.tolist(), ok.tolist()):
        scalar = ora.reconstruct_key(row)
        assert (scalar == key) if accepted else (scalar is None)


def test_c1_hash_group_reversibility_one_million_keys():
    # pkg/tests/test_acceptance.py:31-50
    rng = np.random.default_rng(4242)
    keys = rng.integers(0, 2 ** 32, size=1_000_000, dtype=np.uint64)
    tuples = dhg.forward_many(DEFAULTS, keys)
    rebuilt, ok = dhg.reconstruct_many(DEFAULTS, tuples)
    assert int(ok.sum()) == len(keys) and np.array_equal(rebuilt, keys)
    # restore's candidate set is exactly the tuples this predicate accepts: plant, restore, re-derive
    sk = P.Dhla(DEFAULTS)
    hosts = [0x0A000001 + 1009 * n for n in range(8)]
    for n, h in enumerate(hosts):
        sk.update_batch(*O.plant_pairs(h, 2048, 40 + n))
    cands = sk._candidate_hosts(1024)
    assert sorted(cands.tolist()) == sorted(hosts)
    hot = sk.hot_sets(1024)
    grid = np.stack(np.meshgrid(*hot, indexing="ij"), axis=-1).reshape(-1, DEFAULTS.r)     # HE0 x ... x HE4
    keys2, ok2 = dhg.reconstruct_many(DEFAULTS, grid)
    assert sorted(set(keys2[ok2].tolist())) == sorted(hosts)
