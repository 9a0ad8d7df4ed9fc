"""The reference's OWN engine holding the CUDA sketch.

The installed, unmodified reference (baseline/_ref) runs ``WindowSession`` / ``DetectionEngine``
twice: with its compiled CPU backend, live, and with ``dhsa.engine.Dhla`` replaced -- by this
package's ``Dhla`` and by the ctypes-only binding of integration/dhsa_cuda.py
(INTEGRATION 2b).  Windows, pair counts, drops, bits and reports must be equal.
"""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1803_11449_b200 as P
from oracle import oracle as O

import refpkg

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not refpkg.available(), reason="baseline/_ref not installed")]

REL_TOL = 1e-6


@pytest.fixture()
def ref():
    dhsa, dhsa_cuda = refpkg.load()
    original = dhsa.engine.Dhla
    yield dhsa, dhsa_cuda
    dhsa.engine.Dhla = original


def _plug(dhsa, dhsa_cuda, how):
    if how == "package":      # the package's sketch class in the engine's seam (engine.py:63)
        dhsa.engine.Dhla = lambda params, backend="auto", window_id=0: P.Dhla(params, backend="cuda", window_id=window_id)
    else:                     # the ctypes-only binding
        dhsa_cuda.install(dhsa.engine)


def _same_reports(got, want):
    assert [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
    for a, b in zip(got, want):
        assert a.estimate == pytest.approx(b.estimate, rel=REL_TOL)


@pytest.mark.parametrize("how", ["package", "ctypes_stub"])
@pytest.mark.parametrize("direction", ["src", "dst", "both"])
def test_reference_detection_engine_runs_on_the_cuda_sketch(ref, how, direction):
    dhsa, dhsa_cuda = ref
    from dhsa.engine import DetectionEngine, WindowConfig

    trace = O.engine_trace(9)
    cfg = WindowConfig(direction=direction, workers=4)
    want = DetectionEngine(cfg, backend="compiled").run(trace)          # the reference, live, on the CPU
    _plug(dhsa, dhsa_cuda, how)
    sealed = []
    got = DetectionEngine(cfg, backend="auto").run(trace, on_sealed=lambda sk: sealed.append(sk.bits.copy()))
    assert [(w.window_id, w.pairs, w.dropped) for w in got] == [(w.window_id, w.pairs, w.dropped) for w in want]
    assert len(want) >= 2 and any(w.dropped for w in want)
    for a, b in zip(got, want):
        _same_reports(a.reports, b.reports)
    assert len(sealed) == len(want) and all(b.any() for b in sealed)


@pytest.mark.parametrize("how", ["package", "ctypes_stub"])
@pytest.mark.parametrize("workers", [1, 8])
def test_reference_window_session_feed_seal_restore(ref, how, workers):
    """`dhsa bench`'s sequence (pkg/src/dhsa/cli.py:368-383): feed_batch splits into 65,536-pair
    batches submitted from a thread pool onto one sketch, seal, restore, bits digest."""
    dhsa, dhsa_cuda = ref
    from dhsa.engine import WindowConfig, WindowSession

    cand, opp = O.distinct_pairs(400_000, 21)
    for n, host in enumerate((0x0A0B0C0D, 0xC63A1B02)):
        c2, o2 = O.plant_pairs(host, 3000 + 500 * n, 90 + n)
        cand, opp = np.concatenate([cand, c2]), np.concatenate([opp, o2])
    order = np.random.default_rng(8).permutation(len(cand))
    cand, opp = cand[order], opp[order]
    cfg = WindowConfig(workers=workers)

    def run(backend):
        pool = ThreadPoolExecutor(max_workers=workers) if workers > 1 else None
        session = WindowSession(cfg, 5, backend, pool)
        session.feed_batch(cand, opp)
        session.seal()
        if pool is not None:
            pool.shutdown()
        return session, session.restore()

    s_ref, want = run("compiled")
    _plug(dhsa, dhsa_cuda, how)
    s_gpu, got = run("auto")
    assert s_gpu.pairs == s_ref.pairs == len(cand) and s_gpu.sketch.window_id == 5
    assert s_gpu.sketch.bits.tobytes() == s_ref.sketch.bits.tobytes()
    assert s_gpu.sketch.memory_bytes == s_ref.sketch.memory_bytes == 10_485_760
    _same_reports(got, want)
    assert {r.host for r in got} == {0x0A0B0C0D, 0xC63A1B02}
    with pytest.raises(dhsa.errors.SealedWindowError):
        s_gpu.feed_batch(cand[:4], opp[:4])


def test_reference_capacity_error_text_through_the_stub(ref):
    dhsa, dhsa_cuda = ref
    from dhsa.dhla import Dhla
    from dhsa.dhg import DhgParams

    params = DhgParams()
    cpu, gpu = Dhla(params, backend="compiled"), dhsa_cuda.CudaDhla(params)
    for n in range(40):
        c, o = O.plant_pairs(0x0B000000 + 977 * n, 1500, 300 + n)
        cpu.update_batch(c, o)
        gpu.update_batch(c, o)
    with pytest.raises(dhsa.errors.CapacityError) as want:
        cpu.restore_superpoints(1024, max_candidates=10)
    with pytest.raises(dhsa.errors.CapacityError) as got:
        gpu.restore_superpoints(1024, max_candidates=10)
    assert str(got.value) == str(want.value)


def test_backend_argument_follows_the_reference_rules(ref):
    """pkg/src/dhsa/_kernels.py:42-55: names are a closed set; a Backend INSTANCE passes through.
    Here a record naming this backend is accepted, CPU backends are refused in the same wording."""
    dhsa, _ = ref
    from dhsa._kernels import Backend, get_backend

    with pytest.raises(P.ConfigError, match="unknown backend 'compiled'; expected auto or cuda"):
        P.Dhla(P.DhgParams(), backend="compiled")
    with pytest.raises(P.ConfigError, match="unknown backend 'compiled'"):
        P.Dhla(P.DhgParams(), backend=get_backend("compiled"))       # a CPU Backend instance
    sk = P.Dhla(P.DhgParams(), backend=Backend("cuda", None, None, True))
    assert sk.backend_name == "cuda"
    with pytest.raises(dhsa.errors.ConfigError):
        get_backend("cuda")                                          # pkg/tests/test_kernels.py:89-91 still holds
