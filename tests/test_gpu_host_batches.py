"""Host input the way the reference engine feeds it (pkg/src/dhsa/engine.py:78-86): ordinary
pageable numpy arrays in batches of batch_pairs = 65,536, from one thread or from a pool onto one
sketch.  The library appends the batches to page-locked accumulation slots and copies + scans a slot
when it is full or at the next barrier / read-out; whatever the batching, the bits are the oracle's.
"""
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1803_11449_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _window(n, flows, seed):
    cand, opp = O.distinct_pairs(flows, seed)
    pick = np.random.default_rng(seed).integers(0, flows, size=n)
    return cand[pick].copy(), opp[pick].copy()


@pytest.mark.parametrize("workers", [1, 8])
@pytest.mark.parametrize("batch", [65536, 1000, 1 << 20, 3_000_001])
def test_small_pageable_batches_equal_the_oracle(batch, workers):
    n = 6_000_000
    cand, opp = _window(n, 300_000, 5)
    ora = O.OracleSketch()
    ora.update_batch(cand, opp, threads=8)
    sk = P.Dhla(P.DhgParams())
    if workers == 1:
        for lo in range(0, n, batch):
            sk.update_batch(cand[lo:lo + batch], opp[lo:lo + batch])
    else:
        with ThreadPoolExecutor(workers) as pool:
            futs = [pool.submit(sk.update_batch, cand[lo:lo + batch], opp[lo:lo + batch]) for lo in range(0, n, batch)]
            for f in futs:
                f.result()
    assert np.array_equal(sk.bits, ora.bits)          # the read-out flushes the partly filled slot
    assert sk.launch_count <= 2 * (n // (1 << 20) + 2)   # ~one scan per full slot, not one per batch


def test_every_readout_sees_batches_still_waiting_in_a_slot():
    cand, opp = O.plant_pairs(0xC63A1B02, 2048, 10)
    want = O.OracleSketch()
    want.update_batch(cand, opp)
    for read in ("bits", "zero_counts", "hot_sets", "estimate", "candidates", "shared", "restore", "cell", "seal"):
        sk = P.Dhla(P.DhgParams())
        sk.update_batch(cand, opp)                     # 2048 pairs: far from a full slot, nothing queued yet
        if read == "bits":
            assert np.array_equal(sk.bits, want.bits)
        elif read == "zero_counts":
            assert np.array_equal(sk.zero_counts(), want.zero_counts())
        elif read == "hot_sets":
            assert [len(h) for h in sk.hot_sets(1024)] == [1] * 5
        elif read == "estimate":
            assert sk.estimate()["zero_totals"] == [int(z) for z in want.zero_counts().sum(axis=1)]
        elif read == "candidates":
            assert sk._candidate_hosts(1024).tolist() == [0xC63A1B02]
        elif read == "shared":
            assert int(sk.shared_zero_counts([0xC63A1B02])[0]) == 147      # SURVEY 8(c) golden value
        elif read == "restore":
            assert [r.host for r in sk.restore_superpoints(1024)] == [0xC63A1B02]
        elif read == "cell":
            i, j = (int(v) for v in np.argwhere(want.bits.any(axis=2))[0])
            assert np.array_equal(sk.estimator(i, j), want.bits[i, j])
        else:
            sk.seal()
            assert np.array_equal(sk.bits, want.bits)


def test_reset_merge_and_upload_order_with_pending_batches():
    a_c, a_o = O.distinct_pairs(70_000, 31)
    b_c, b_o = O.distinct_pairs(50_000, 32)
    sk = P.Dhla(P.DhgParams())
    sk.update_batch(a_c, a_o)
    sk.reset()                                        # the pending batch belongs to the window that ended
    sk.update_batch(b_c, b_o)
    only_b = O.OracleSketch()
    only_b.update_batch(b_c, b_o)
    assert np.array_equal(sk.bits, only_b.bits)
    other = P.Dhla(P.DhgParams())
    other.update_batch(a_c, a_o)                      # pending in `other` when it is merged
    sk.update_batch(a_c[:100], a_o[:100])             # pending in `sk` when it is merged into
    sk.merge_from(other)
    both = O.OracleSketch()
    both.update_batch(b_c, b_o)
    both.update_batch(a_c, a_o)
    assert np.array_equal(sk.bits, both.bits)
    sk.update_batch(a_c, a_o)
    sk.load_bits(only_b.bits)                         # an upload replaces everything handed over before it
    assert np.array_equal(sk.bits, only_b.bits)


def test_feeders_racing_a_reader_never_lose_a_batch():
    """8 feeder threads while another thread keeps reading: every batch handed over before the final
    seal is in the bits (slots closed by a reader and slots closed by a full reservation interleave)."""
    n = 4_000_000
    cand, opp = _window(n, 200_000, 9)
    ora = O.OracleSketch()
    ora.update_batch(cand, opp, threads=8)
    sk = P.Dhla(P.DhgParams())
    stop = threading.Event()

    def reader():
        while not stop.is_set():
            sk.estimate()

    t = threading.Thread(target=reader)
    t.start()
    try:
        with ThreadPoolExecutor(8) as pool:
            futs = [pool.submit(sk.update_batch, cand[lo:lo + 30_011], opp[lo:lo + 30_011]) for lo in range(0, n, 30_011)]
            for f in futs:
                f.result()
    finally:
        stop.set()
        t.join()
    assert np.array_equal(sk.bits, ora.bits)


def test_pinned_and_pageable_large_arrays():
    import torch

    n = 5_000_003
    cand, opp = _window(n, 250_000, 12)
    ora = O.OracleSketch()
    ora.update_batch(cand, opp, threads=8)
    ch = torch.from_numpy(cand.view(np.int32)).pin_memory()
    oh = torch.from_numpy(opp.view(np.int32)).pin_memory()
    a, b = P.Dhla(P.DhgParams()), P.Dhla(P.DhgParams())
    a.update_batch(ch.numpy().view(np.uint32), oh.numpy().view(np.uint32))   # page-locked: DMA'd in place
    b.update_batch(cand, opp)                                                # pageable: through the slots
    assert np.array_equal(a.bits, ora.bits) and np.array_equal(b.bits, ora.bits)
