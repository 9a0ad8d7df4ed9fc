"""Row N4: the on-device synthetic trace generator.  Every byte against the oracle's numpy
restatement of the same counter-based definition; the statistics and structure against the
reference generator's semantics (pkg/src/dhsa/ingest.py:109-153)."""
import numpy as np
import pytest

import paper_1803_11449_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu

CASES = [
    dict(background_hosts=2000, superpoints=5, seed=7),
    dict(background_hosts=500, superpoints=0, duplicate_factor=3, seed=8, start_ts=900, window_seconds=60),
    dict(background_hosts=0, superpoints=3, super_cardinality=(100, 100), duplicate_factor=2, seed=9),
    dict(background_hosts=300, background_max_cardinality=1, superpoints=1, seed=10),
    dict(background_hosts=1000, background_zipf=1.1, background_max_cardinality=64, superpoints=2, seed=11),
]


@pytest.mark.parametrize("kw", CASES, ids=[str(i) for i in range(len(CASES))])
def test_generator_is_byte_identical_to_its_oracle(kw):
    kw = dict(kw)
    seed = kw.pop("seed")
    want_rec, want_truth = O.generate_trace_spec(seed=seed, **kw)
    rec, truth = P.generate_trace(P.GeneratorConfig(**kw), seed)
    assert truth == want_truth
    assert rec.tobytes() == want_rec.tobytes()


def test_generator_has_the_reference_generators_semantics():
    cfg = P.GeneratorConfig(background_hosts=37_000, superpoints=20, duplicate_factor=2)
    rec, truth = P.generate_trace(cfg, seed=7)
    n_flows = sum(truth.values())
    assert len(rec) == 2 * n_flows and len(truth) == 37_020                    # distinct hosts
    assert np.all(np.diff(rec["ts"].astype(np.int64)) >= 0)                    # time-ordered, ingest.py:148
    assert rec["ts"].min() == 0 and rec["ts"].max() == 299                     # inside the window
    assert O.exact_counts(rec, "src") == truth                                 # truth is exact, ingest.py:150
    cards = np.array(list(truth.values()))
    supers = cards[cards > 256]
    assert len(supers) == 20 and supers.min() >= 2048 and supers.max() <= 8192  # ingest.py:127-129
    bg = cards[cards <= 256]
    assert 0.36 <= np.mean(bg == 1) <= 0.41          # zipf(1.5): P(1) = 1/zeta(1.5) = 0.383
    assert 0.035 <= np.mean(bg == 256) <= 0.06       # mass of the truncated tail, ~0.048
    assert 20 <= bg.mean() <= 28                     # the reference's config 1 averages ~23.7 flows per host
    key = (rec["src"].astype(np.uint64) << np.uint64(32)) | rec["dst"].astype(np.uint64)
    _, reps = np.unique(key, return_counts=True)
    assert np.all(reps == 2)                          # every pair exactly duplicate_factor times, ingest.py:139-141
    first_half = rec["src"][: len(rec) // 2]
    assert len(np.unique(first_half)) > 0.8 * len(truth) * 0.5   # shuffled, not host-major


def test_generator_slices_agree_with_the_whole_and_feed_the_detector():
    """Ranks of a multi-GPU window generate their own slices; the detector finds the planted hosts."""
    import torch

    cfg = P.GeneratorConfig(background_hosts=20_000, superpoints=10, duplicate_factor=4)
    whole = P.generate_trace_device(cfg, seed=21, fmt="both")
    total = whole["total"]
    cut = (total // 3) & ~3
    a = P.generate_trace_device(cfg, seed=21, fmt="both", lo=0, hi=cut)
    b = P.generate_trace_device(cfg, seed=21, fmt="both", lo=cut, hi=total)
    assert torch.equal(torch.cat([a["cand"], b["cand"]]), whole["cand"])
    assert torch.equal(torch.cat([a["records"], b["records"]]), whole["records"])
    sk = P.Dhla(P.DhgParams())
    sk.update_batch(whole["cand"], whole["opp"])
    reports = sk.restore_superpoints(1024)
    m = P.evaluate(reports, whole["truth"], 1024)
    assert m.n_true == 10 and m.fnr == 0.0 and m.fpr == 0.0
    res = P.DetectionEngine(P.WindowConfig()).run(whole["records"])
    assert [(r.window_id, r.pairs, r.dropped) for r in res] == [(0, total, 0)]
    assert [x.host for x in res[0].reports] == [x.host for x in reports]


def test_generator_config_validation():
    # ingest.py:90-106
    for kw in (dict(background_hosts=-1), dict(background_max_cardinality=0), dict(super_cardinality=(5, 4)),
               dict(duplicate_factor=0), dict(window_seconds=0), dict(background_zipf=1.0)):
        with pytest.raises(P.ConfigError):
            P.GeneratorConfig(**kw)
    rec, truth = P.generate_trace(P.GeneratorConfig(), 1)
    assert len(rec) == 0 and truth == {}
