"""Bit parity at every BASELINE.json configuration, inside the suite the driver runs.

config 3  1B-packet window (whole, and as 8 packet shards OR-merged)        tests/checks/config3_window.py
config 4  100M-packet DDoS trace, victims as candidates and as opposites,  tests/checks/contention.py
          all five scan modes
config 5  every point of the threshold / DDH-size sweep                    tools/accuracy_sweep.py
(configs 1 and 2 are in test_gpu_parity.py.)  The sketch is a pure function of the window's
distinct pair set, so the oracle scans the distinct flows and the GPU
scans every packet; bits (SHA-256), the report list and the CapacityError text must be equal.
"""
import hashlib
import importlib.util
import os

import numpy as np
import pytest

import paper_1803_11449_b200 as P
from paper_1803_11449_b200.traces import trace_population
from oracle import oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 1e-6
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _flows(cfg, seed):
    """Distinct (src, dst) flows of a generated window, on the host (the generator's per-host half)."""
    hosts, cards, bases = trace_population(cfg, seed)
    src = np.repeat(hosts, cards)
    starts = np.repeat(np.cumsum(cards) - cards, cards)
    ramp = (np.arange(len(src), dtype=np.int64) - starts).astype(np.uint32)
    dst = np.repeat(bases, cards) + ramp        # uint32 wrap-around, as the device ramp does
    return src.astype(np.uint32), dst.astype(np.uint32)


def _outcome(restore, *args, **kw):
    try:
        return [(r.host, r.saturated, r.estimate) for r in restore(*args, **kw)]
    except (P.CapacityError, O.OracleCapacityError) as exc:
        return str(exc)


def _same_outcome(got, want):
    if isinstance(want, str) or isinstance(got, str):
        assert got == want
        return
    assert [(h, s) for h, s, _ in got] == [(h, s) for h, s, _ in want]
    for (_, _, a), (_, _, b) in zip(got, want):
        assert a == pytest.approx(b, rel=REL_TOL)


def _sweep_points():
    spec = importlib.util.spec_from_file_location("accuracy_sweep", os.path.join(ROOT, "tools", "accuracy_sweep.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod.POINTS, mod.point_config


POINTS, point_config = _sweep_points()


@pytest.mark.parametrize("theta, g, k, alpha", POINTS, ids=[f"theta{t}-g{g}-k{k}-a{a}" for t, g, k, a in POINTS])
@pytest.mark.parametrize("mode", ["auto", "test_agg"])
def test_config5_sweep_point_is_bit_exact(theta, g, k, alpha, mode):
    """The windows tools/accuracy_sweep.py scores, bit-compared: sketches of 10..160 MiB (g = 4096 /
    16384 and k = 16 / 18 leave L2), with and without the flow cache."""
    cfg = point_config(theta)
    tr = P.generate_trace_device(cfg, seed=100, fmt="pairs")
    kw = dict(g=g, k=k, alpha=alpha)
    ora = O.OracleSketch(**kw)
    ora.update_batch(*_flows(cfg, 100), threads=8)
    sk = P.Dhla(P.DhgParams(**kw))
    sk.set_scan_mode(mode)
    sk.update_batch(tr["cand"], tr["opp"])
    assert sha(sk.bits) == sha(ora.bits)
    assert np.array_equal(sk.zero_counts(), ora.zero_counts())
    _same_outcome(_outcome(sk.restore_superpoints, theta, max_candidates=1 << 22),
                  _outcome(ora.restore_superpoints, theta, max_candidates=1 << 22))


def test_config3_one_billion_packet_window_whole_and_as_eight_shards():
    import torch

    seed = 300
    flows_cfg = P.GeneratorConfig(background_hosts=150_000, superpoints=50, duplicate_factor=1)
    src, dst = _flows(flows_cfg, seed)
    dup = max(1, round(1_000_000_000 / len(src)))
    cfg = P.GeneratorConfig(background_hosts=150_000, superpoints=50, duplicate_factor=dup)
    win = P.generate_trace_device(cfg, seed, fmt="pairs")
    n, cand, opp = win["total"], win["cand"], win["opp"]
    assert n >= 990_000_000 and win["flows"] == len(src)
    ora = O.OracleSketch()
    ora.update_batch(src, dst, threads=8)
    want = _outcome(ora.restore_superpoints, 1024)
    whole = P.Dhla(P.DhgParams())
    whole.update_batch(cand, opp)
    assert sha(whole.bits) == sha(ora.bits)
    _same_outcome(_outcome(whole.restore_superpoints, 1024), want)
    assert len(want) >= 50
    # 8 packet shards -> 8 private sketches -> OR merge (the multi-GPU choreography on one device)
    cuts = [n * i // 8 // 4 * 4 for i in range(8)] + [n]
    parts = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        sk = P.Dhla(P.DhgParams())
        sk.update_batch(cand[lo:hi], opp[lo:hi])
        parts.append(sk)
    for sk in parts[1:]:
        parts[0].merge_from(sk)
    assert sha(parts[0].bits) == sha(ora.bits)
    _same_outcome(_outcome(parts[0].restore_superpoints, 1024), want)
    del cand, opp, win
    torch.cuda.empty_cache()


def _ddos_window(n):
    """1M sources -> 4 victims chosen by Zipf(1.2) (BASELINE config 4, tests/checks/contention.py)."""
    import torch

    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    victims = torch.tensor([0x0A000001, 0x0A000002, 0xC0A80101, 0x08080808], dtype=torch.int64, device="cuda")
    w = torch.tensor([1.0 / (i + 1) ** 1.2 for i in range(4)], device="cuda")
    vic = victims[torch.multinomial(w, n, replacement=True, generator=g)]
    sources = torch.randint(0, 2 ** 32, (1_000_000,), device="cuda", generator=g, dtype=torch.int64)
    src = sources[torch.randint(0, 1_000_000, (n,), device="cuda", generator=g)]
    as_i32 = lambda t: torch.where(t >= 2 ** 31, t - 2 ** 32, t).to(torch.int32)
    return as_i32(vic), as_i32(src)


@pytest.fixture(scope="module")
def ddos():
    import torch

    vic, src = _ddos_window(100_000_000)
    out = {}
    for direction, (cand, opp) in (("dst", (vic, src)), ("src", (src, vic))):
        u = torch.unique(((cand.to(torch.int64) & 0xFFFFFFFF) << 32) | (opp.to(torch.int64) & 0xFFFFFFFF))
        uc = ((u >> 32) & 0xFFFFFFFF).cpu().numpy().astype(np.uint32)
        uo = (u & 0xFFFFFFFF).cpu().numpy().astype(np.uint32)
        ora = O.OracleSketch()
        ora.update_batch(uc, uo, threads=8)
        out[direction] = (cand, opp, sha(ora.bits), _outcome(ora.restore_superpoints, 1024))
        del u
    yield out
    del out, vic, src
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["red", "test", "test_agg", "flow_cache", "auto"])
@pytest.mark.parametrize("direction", ["dst", "src"])
def test_config4_ddos_contention_100m_packets(ddos, direction, mode):
    """Victims as candidates ("dst": every packet lands in the same 5 x 4 cells -- same-address
    atomics) and as opposites ("src"), in every scan mode."""
    cand, opp, want_bits, want = ddos[direction]
    sk = P.Dhla(P.DhgParams())
    sk.set_scan_mode(mode)
    sk.update_batch(cand, opp)
    assert sha(sk.bits) == want_bits
    _same_outcome(_outcome(sk.restore_superpoints, 1024), want)
    if direction == "dst":
        assert [s for _, s, _ in want] == [True] * 4        # the four victims, saturated
