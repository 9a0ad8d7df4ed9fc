"""Shared builders for the parity tests: golden fixtures and seeded inputs."""
import json
import os
from types import SimpleNamespace

import numpy as np

from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def restore_cases():
    return load_json("restore_cases.json")


def case_params(case):
    return SimpleNamespace(**case["params"])


def case_batches(case):
    """The (cand, opp) batches a golden case was built from, in feed order."""
    p = case["params"]
    out = []
    for host, fanout, seed in case["plants"]:
        out.append(O.plant_pairs(host, fanout, seed))
    if case["noise"]:
        c, o = O.distinct_pairs(*case["noise"])
        if case["mask_cand"]:
            c = c & np.uint32((1 << p["key_width"]) - 1)
        out.append((c, o))
    return out


def config1_pairs():
    """Distinct (src, dst) pair set of BASELINE config 1, from its stored triples."""
    z = np.load(os.path.join(GOLDEN, "config1_trace.npz"))
    hosts, cards, bases = z["hosts"], z["cards"].astype(np.int64), z["bases"].astype(np.uint64)
    src = np.repeat(hosts, cards)
    starts = np.repeat(np.cumsum(cards) - cards, cards).astype(np.uint64)
    ramp = np.arange(len(src), dtype=np.uint64) - starts
    dst = ((np.repeat(bases, cards) + ramp) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return src.astype(np.uint32), dst


def oracle_for_case(case):
    sk = O.OracleSketch(**case["params"])
    for c, o in case_batches(case):
        sk.update_batch(c, o)
    return sk
