"""Generate tests/golden/*.json|npz from the LIVE reference package.

Run in the build container only (needs /root/reference; the GPU box has none):

    make -C oracle ref && python tests/golden/make_golden.py

It imports the reference's pure-Python modules from /root/reference/pkg/src
(read-only, nothing is copied), plugs the reference's compiled `_core`
(oracle/_ref, built from its .pyx) in as `dhsa._core`, and records what the
reference itself computes on seeded inputs.  Inputs are not stored when a seed
regenerates them (oracle.distinct_pairs / oracle.plant_pairs restate the
reference fixtures pkg/tests/conftest.py:25-34 and pkg/tests/test_dhla.py:30-37);
the config-1 trace is stored as its (host, cardinality, base) triples.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import oracle as O  # noqa: E402

core = O.load_ref_core()
if core is not None:
    sys.modules["dhsa._core"] = core
import dhsa  # noqa: E402
from dhsa import dhg, dhla  # noqa: E402
from dhsa.dhg import DhgParams  # noqa: E402
from dhsa.dhla import Dhla, hot_threshold  # noqa: E402
from dhsa.errors import CapacityError  # noqa: E402
from dhsa.ingest import GeneratorConfig, generate_trace  # noqa: E402

BACKEND = "compiled" if core is not None else "python"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pdict(p: DhgParams) -> dict:
    return dict(r=p.r, g=p.g, k=p.k, alpha=p.alpha, key_width=p.key_width,
                seed_dh0=p.seed_dh0, seed_h1=p.seed_h1)


def stage_counts(sk: Dhla, theta, max_candidates=1 << 62):
    hot = sk.hot_sets(theta)
    if any(len(h) == 0 for h in hot):
        return []
    p = sk.params
    sub, cl0 = dhla._stage_first(p, hot[0], hot[1], hot[2], max_candidates, 1)
    out = [len(sub)]
    for i in range(3, p.r):
        sub, cl0 = dhla._stage_next(p, i, sub, cl0, hot[i], max_candidates, 1)
        out.append(len(sub))
    return out


def readout(sk: Dhla, theta, max_candidates=1 << 20) -> dict:
    zc = sk.zero_counts()
    hot = sk.hot_sets(theta, zc)
    flow = sk.estimate_flow_count(zc)
    psi = sk.bit_set_probability(flow.value)
    out = dict(
        theta=theta,
        bits_sha256=sha(sk.bits),
        zero_counts_sha256=sha(zc.astype(np.int64)),
        zero_totals=[int(v) for v in zc.sum(axis=1)],
        hot_sizes=[len(h) for h in hot],
        hot_sha256=[sha(h.astype(np.uint64)) for h in hot],
        flow_count=flow.value,
        flow_saturated=bool(flow.saturated),
        psi=psi,
        stage_counts=stage_counts(sk, theta),
    )
    try:
        hosts = sk._candidate_hosts(theta, max_candidates, 1, zc)
        out["candidates"] = [int(h) for h in hosts]
        out["shared_zero_counts"] = [int(v) for v in sk.shared_zero_counts(hosts)] if len(hosts) else []
        reps = sk.restore_superpoints(theta, max_candidates=max_candidates)
        out["reports"] = [[r.host, r.estimate, bool(r.saturated)] for r in reps]
    except CapacityError as exc:
        out["capacity_error"] = str(exc)
    return out


def build_case(name, p: DhgParams, theta, plants, noise, max_candidates=1 << 20, mask_cand=False):
    """plants: [(host, fanout, seed)], noise: (n, seed) or None."""
    sk = Dhla(p, backend=BACKEND)
    for host, fanout, seed in plants:
        c, o = O.plant_pairs(host, fanout, seed)
        sk.update_batch(c, o)
    if noise:
        c, o = O.distinct_pairs(*noise)
        if mask_cand:
            c = c & np.uint32((1 << p.key_width) - 1)
        sk.update_batch(c, o)
    rec = dict(name=name, params=pdict(p), plants=[list(x) for x in plants],
               noise=list(noise) if noise else None, mask_cand=mask_cand,
               max_candidates=max_candidates)
    rec.update(readout(sk, theta, max_candidates))
    return rec


def main():
    P = DhgParams()
    consts = dict(
        backend=BACKEND,
        state_dh0=P.state_dh0, state_h1=P.state_h1,
        mix64={str(x): dhg.mix64(x) for x in (0, 1, 2, 0xC0A80101, 2 ** 32 - 1, 2 ** 63, 2 ** 64 - 1)},
        forward={str(a): list(dhg.forward(P, a)) for a in (0, 1, 0xC0A80101, 0x08080808, 0xFFFFFFFF)},
        h1={str(b): dhg.h1(P, b) for b in (0, 1, 0x08080808, 0xFFFFFFFF)},
        hot_threshold={f"{g},{t}": hot_threshold(g, t)
                       for g, t in ((1024, 256), (1024, 1024), (1024, 4096), (1024, 16384),
                                    (256, 256), (4096, 4096))},
        sketch_bytes=P.sketch_bytes,
    )
    # one update(0xC0A80101, 0x08080808): exactly r bits
    sk = Dhla(P, backend=BACKEND)
    sk.update(0xC0A80101, 0x08080808)
    nz = np.argwhere(sk.bits)
    consts["single_update"] = [[int(i), int(j), int(b), int(sk.bits[i, j, b])] for i, j, b in nz]
    # reconstruct: scalar inverse on true tuples and on corrupted ones
    rng = np.random.default_rng(99)
    keys = rng.integers(0, 2 ** 32, size=64, dtype=np.uint64)
    rec = []
    for key in keys.tolist():
        idx = list(dhg.forward(P, key))
        bad = list(idx)
        bad[2] ^= 1
        rec.append([key, idx, dhg.reconstruct_key(P, idx), dhg.reconstruct_key(P, bad)])
    consts["reconstruct"] = rec
    with open(os.path.join(HERE, "constants.json"), "w") as fh:
        json.dump(consts, fh, indent=1)

    toy = DhgParams(r=4, g=64, k=8, alpha=4, key_width=16)
    small = DhgParams(r=5, g=256, k=10, alpha=8, key_width=32, seed_dh0=1, seed_h1=2)
    minr = DhgParams(r=3, g=256, k=18, alpha=14, key_width=32, seed_dh0=3, seed_h1=4)
    trunc = DhgParams(r=5, g=1024, k=16, alpha=6)        # (r-2)a+k = 34 > 32: key-width cut matters
    six = DhgParams(r=6, g=512, k=12, alpha=5)
    g8 = DhgParams(r=3, g=8, k=8, alpha=8, key_width=16)
    g16 = DhgParams(r=4, g=16, k=10, alpha=8, key_width=24, seed_dh0=11, seed_h1=12)
    rng = np.random.default_rng(11)
    twenty = [int(h) for h in rng.integers(0, 2 ** 32, size=20, dtype=np.uint64)]
    cases = [
        build_case("default_pairs50k", P, 1024, [], (50_000, 3)),
        build_case("default_empty", P, 1024, [], None),
        build_case("default_single_plant", P, 1024, [(0xC63A1B02, 2048, 10)], None),
        build_case("default_20_plants", P, 1024,
                   [(h, 1500 + 100 * n, 300 + n) for n, h in enumerate(twenty)], None),
        build_case("default_ties", P, 1024, [(5000, 2000, 12), (4000, 2000, 12)], None),
        build_case("default_saturated", P, 1024, [(99, 20_000, 9)], None),
        build_case("default_10_plants_noise200k", P, 1024,
                   [(2_000_000 + n * 7, 2048, 600 + n) for n in range(10)], (200_000, 14)),
        build_case("default_60_plants_noise1m", P, 1024,
                   [(0x0A000000 + 7919 * n, 1100 + 37 * n, 700 + n) for n in range(60)],
                   (1_000_000, 21)),
        build_case("default_capacity_overflow", P, 1024,
                   [(1000 + n, 1500, 500 + n) for n in range(8)], None, max_candidates=2),
        build_case("default_theta256", P, 256,
                   [(0x0B000000 + 104729 * n, 300 + 40 * n, 800 + n) for n in range(12)],
                   (100_000, 22)),
        build_case("default_theta4096", P, 4096,
                   [(0x0C000000 + 15485863 * n, 4000 + 900 * n, 900 + n) for n in range(6)], None),
        build_case("toy_pairs", toy, 32, [(0x1234, 200, 1), (0xBEEF, 150, 2)], (3000, 3),
                   mask_cand=True),
        build_case("small_params", small, 256, [(0x0A000001, 700, 100), (0x0A000002, 900, 101)],
                   (20_000, 23)),
        build_case("min_r3", minr, 256, [(0xAC100005, 900, 15)], None),
        build_case("min_r3_noise", minr, 256, [(0xAC100005, 900, 15), (0x0D0D0D0D, 700, 16)],
                   (300_000, 24)),
        build_case("truncating_k16", trunc, 1024,
                   [(0xF00DF00D, 2500, 31), (0x00000001, 3000, 32), (0xFFFFFFFF, 1800, 33)],
                   (400_000, 25)),
        build_case("six_arrays", six, 512, [(0xDEADBEEF, 1200, 41), (0x01020304, 1000, 42)],
                   (150_000, 26)),
        # dense hot sets: spurious tuples survive the early stages (alpha = k - 2: 2-bit overlap)
        build_case("small_dense", small, 64, [(0x0A000001, 500, 110), (0x7B000002, 400, 111)],
                   (50_000, 33), max_candidates=1 << 22),
        build_case("small_dense_overflow_stage2", small, 64,
                   [(0x0A000001, 500, 110), (0x7B000002, 400, 111)], (50_000, 33),
                   max_candidates=30_000),
        build_case("toy_dense", toy, 16, [(0x4321, 120, 5)], (3000, 34), mask_cand=True),
        build_case("six_dense", six, 128, [(0xDEADBEEF, 700, 43)], (450_000, 35),
                   max_candidates=1 << 22),
        build_case("g8_bytes", g8, 8, [(0x0102, 40, 51)], (500, 27), mask_cand=True),
        build_case("g16_halfwords", g16, 16, [(0x00ABCDEF, 60, 61), (0x00123456, 50, 62)],
                   (4000, 28), mask_cand=True),
    ]
    with open(os.path.join(HERE, "restore_cases.json"), "w") as fh:
        json.dump(cases, fh, indent=1)

    # config 1 of BASELINE.json: reference generator, 37k background hosts + 20 supers, seed 7
    cfg = GeneratorConfig(background_hosts=37_000, superpoints=20)
    records, truth = generate_trace(cfg, seed=7)
    src = records["src"].astype(np.uint32)
    dst = records["dst"].astype(np.uint32)
    sk = Dhla(P, backend=BACKEND)
    sk.update_batch(src, dst)
    # the distinct pair set regenerates from (host, cardinality, ramp base): destinations of
    # one host are base + 0..card-1 (mod 2^32); the base is the one whose predecessor is absent
    pairs = np.unique((src.astype(np.uint64) << np.uint64(32)) | dst.astype(np.uint64))
    ps, pd = pairs >> np.uint64(32), pairs & np.uint64(0xFFFFFFFF)
    pred = (ps << np.uint64(32)) | ((pd - np.uint64(1)) & np.uint64(0xFFFFFFFF))
    is_base = ~np.isin(pred, pairs)
    hosts, cards = np.unique(ps, return_counts=True)
    assert int(is_base.sum()) == len(hosts) and np.array_equal(ps[is_base], hosts)
    bases = pd[is_base]
    np.savez_compressed(os.path.join(HERE, "config1_trace.npz"),
                        hosts=hosts.astype(np.uint32), cards=cards.astype(np.uint32),
                        bases=bases.astype(np.uint32))
    rec = dict(name="config1", params=pdict(P), records=int(len(records)),
               truth_supers=sorted([[int(h), int(c)] for h, c in truth.items() if c >= 1024]))
    rec.update(readout(sk, 1024))
    with open(os.path.join(HERE, "config1_expected.json"), "w") as fh:
        json.dump(rec, fh, indent=1)
    # snapshots (row N2): the reference's own file bytes for one sketch
    import io
    sk = Dhla(P, backend=BACKEND)
    sk.update_batch(*O.distinct_pairs(50_000, 19))
    sk.window_id = 77
    buf = io.BytesIO()
    dhla.write_snapshot(sk, buf)
    blob = buf.getvalue()
    with open(os.path.join(HERE, "snapshot_case.json"), "w") as fh:
        json.dump(dict(pairs=[50_000, 19], window_id=77, size=len(blob), header_hex=blob[:42].hex(),
                       file_sha256=hashlib.sha256(blob).hexdigest()), fh, indent=1)

    # window engine (row N1): the reference's DetectionEngine on a multi-window trace with late records
    from dhsa.engine import DetectionEngine, WindowConfig
    eng = []
    for seed in (9, 10):
        trace = O.engine_trace(seed)
        for direction in ("src", "dst", "both"):
            res = DetectionEngine(WindowConfig(direction=direction, batch_pairs=1000), backend=BACKEND).run(trace)
            eng.append(dict(seed=seed, direction=direction, window_seconds=300, theta=1024,
                            records=int(len(trace)), trace_sha256=sha(trace),
                            windows=[dict(window_id=r.window_id, pairs=r.pairs, dropped=r.dropped,
                                          reports=[[x.host, x.estimate, bool(x.saturated)] for x in r.reports])
                                     for r in res]))
    with open(os.path.join(HERE, "engine_cases.json"), "w") as fh:
        json.dump(eng, fh, indent=1)
    # exact oracle + metrics (row N3): the reference's ingest.exact_oracle / evaluate on the engine trace
    from dhsa.ingest import evaluate as ref_evaluate, exact_oracle as ref_exact
    from dhsa.dhla import SuperPointReport as RefReport
    ex = []
    trace = O.engine_trace(9)
    for direction in ("src", "dst", "both"):
        truth = ref_exact(trace, direction)
        top = sorted(truth.items(), key=lambda kv: (-kv[1], kv[0]))[:8]
        fake = [RefReport(h, c * 1.05, False) for h, c in top[:3]] + [RefReport(12345, 2000.0, False)]
        ex.append(dict(seed=9, direction=direction, n_hosts=len(truth), n_pairs=int(sum(truth.values())),
                       hosts_sha256=sha(np.array(sorted(truth), dtype=np.uint64)),
                       counts_sha256=sha(np.array([truth[h] for h in sorted(truth)], dtype=np.uint64)),
                       top=[[int(h), int(c)] for h, c in top],
                       metrics=ref_evaluate(fake, truth, 1024).as_dict()))
    with open(os.path.join(HERE, "exact_cases.json"), "w") as fh:
        json.dump(ex, fh, indent=1)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
