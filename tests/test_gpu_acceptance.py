"""The reference's release criteria that involve the hot path (pkg/tests/test_acceptance.py C5-C8),
run against the device sketch, engine, generator and ground-truth counter."""
import os

import numpy as np
import pytest

import paper_1803_11449_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def test_c5_end_to_end_detection():
    # pkg/tests/test_acceptance.py:115-141: FNR 0, mean FPR <= 0.05, mean relative error <= 10%
    fprs, fnrs, errs = [], [], []
    for seed in range(5):
        gcfg = P.GeneratorConfig(background_hosts=200_000, background_max_cardinality=256, superpoints=50,
                                 super_cardinality=(2048, 8192))
        got = P.generate_trace_device(gcfg, seed=100 + seed, fmt="records")
        result = P.DetectionEngine(P.WindowConfig(theta=1024)).run(got["records"])[0]
        assert result.pairs == got["total"] and result.dropped == 0
        # the ground truth is counted on the device too (N3) and must agree with the generator's
        exact = P.exact_oracle(got["records"])
        assert {h: c for h, c in exact.items() if c >= 1024} == {h: c for h, c in got["truth"].items() if c >= 1024}
        m = P.evaluate(result.reports, got["truth"], theta=1024)
        fprs.append(m.fpr), fnrs.append(m.fnr), errs.append(m.mean_rel_err)
    assert all(v == 0.0 for v in fnrs)
    assert float(np.mean(fprs)) <= 0.05 and float(np.mean(errs)) <= 0.10


def test_c6_merge_homomorphism_and_snapshots(tmp_path):
    # pkg/tests/test_acceptance.py:144-176
    records, _ = P.generate_trace(P.GeneratorConfig(background_hosts=20_000, superpoints=8), seed=321)
    split = np.random.default_rng(321).random(len(records)) < 0.5
    cfg = P.WindowConfig(theta=1024)
    sketches = {}
    for name, part in (("s1", records[split]), ("s2", records[~split]), ("all", records)):
        sealed = []
        P.DetectionEngine(cfg).run(part, on_sealed=sealed.append)
        sketches[name] = sealed[0]
    merged = P.merge(sketches["s1"], sketches["s2"])
    assert np.array_equal(merged.bits, sketches["all"].bits)
    path = str(tmp_path / "snap.dhla")
    P.write_snapshot(merged, path)
    back = P.read_snapshot(path)
    assert np.array_equal(back.bits, merged.bits) and back.params == P.DhgParams()
    whole = sketches["all"].restore_superpoints(1024)
    assert merged.restore_superpoints(1024) == whole and back.restore_superpoints(1024) == whole
    assert len(whole) >= 8


def test_c7_determinism_across_chunking_threads_and_scan_modes():
    # pkg/tests/test_acceptance.py:179-199 (workers 1/2/8 there; here chunk sizes, feeding threads and kernels)
    from concurrent.futures import ThreadPoolExecutor

    records, _ = P.generate_trace(P.GeneratorConfig(background_hosts=30_000, superpoints=10), seed=654)
    digests, reports = [], []
    for chunk in (1 << 24, 100_003, 4096):
        sealed = []
        res = P.DetectionEngine(P.WindowConfig(theta=1024), chunk_records=chunk).run(
            records, on_sealed=lambda s: sealed.append(s.bits.tobytes()))
        digests.append(sealed[0]), reports.append(res[0].reports)
    cand, opp = P.split_pairs(records, "src")
    for mode, workers in (("red", 1), ("test_agg", 8), ("flow_cache", 8)):
        sk = P.Dhla(P.DhgParams())
        sk.set_scan_mode(mode)
        with ThreadPoolExecutor(workers) as pool:
            list(pool.map(lambda lo: sk.update_batch(cand[lo:lo + 65536], opp[lo:lo + 65536]),
                          range(0, len(cand), 65536)))
        digests.append(sk.bits.tobytes()), reports.append(sk.restore_superpoints(1024))
    assert all(d == digests[0] for d in digests)
    assert all(r == reports[0] for r in reports) and len(reports[0]) >= 10


def test_c8_fixed_memory(tmp_path):
    # pkg/tests/test_acceptance.py:202-227
    sk = P.Dhla(P.DhgParams())
    sizes = [sk.memory_bytes]
    for seed in (1, 2):
        sk.update_batch(*O.distinct_pairs(500_000, seed))
        sizes.append(sk.memory_bytes)
    path = str(tmp_path / "mem.dhla")
    P.write_snapshot(sk, path)
    assert all(s == 10_485_760 for s in sizes) and os.path.getsize(path) - 42 == 10_485_760
