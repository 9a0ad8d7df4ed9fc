"""pytest plugin: the reference's OWN test files, unmodified, against the CUDA sketch.

    PYTHONPATH=<repo>:<repo>/integration:<repo>/baseline/_ref \\
        python -m pytest -p dhsa_cuda_suite <reference>/pkg/tests/test_dhla.py ...

Loaded with ``-p`` it runs before any test module is imported and puts this repository's
device-resident classes into the seams of the installed reference package (baseline/_ref):

    dhsa.dhla.Dhla / merge / read_snapshot / write_snapshot   -> paper_1803_11449_b200
    dhsa.engine.Dhla                                          -> the same sketch class (engine.py:63)
    dhsa.dhg.forward_many / reconstruct_many                  -> the library's kernels (the scalar
                                                                 reconstruct_key stays the reference's: its C1 test
                                                                 calls it 10^6 times from a Python loop)

so that ``from dhsa.dhla import Dhla`` in /root/reference/pkg/tests/*.py binds the CUDA sketch and
every assertion the reference makes about its sketch is made about this one.  Backend names are
ignored (``Dhla(p, backend="python")`` is still the CUDA sketch): a test that compares two backends
then compares the device path with itself, which is vacuous but harmless; the cross-checks against
the reference's CPU kernels live in tests/test_gpu_reference_engine.py and the oracle tests.
With ``DHSA_CUDA_SUITE_ENGINE=device`` the window engine itself is replaced as well
(``dhsa.engine.DetectionEngine / WindowSession / WindowConfig / split_pairs`` -> the package's
engine, which decodes, windows and orients raw records on the GPU), so test_engine.py and the
engine-driven release criteria run against the device record path.
tests/test_gpu_reference_suite.py drives both on the B200 box.
"""
import os

import dhsa.dhg
import dhsa.dhla
import dhsa.engine
from dhsa.estimator import LinearEstimator

import paper_1803_11449_b200 as P
from paper_1803_11449_b200 import dhg as cuda_dhg


class Dhla(P.Dhla):
    """The package's sketch under the reference's constructor (dhla.py:60); ``params`` stays the
    reference's own DhgParams object, so equality with reference-built parameters holds."""

    def __init__(self, params, backend="auto", window_id=0):
        super().__init__(params, backend="cuda", window_id=window_id)
        self.params = params

    def estimator(self, i, j):          # dhla.py:107-109 returns the reference's LinearEstimator
        return LinearEstimator(self.params.g, super().estimator(i, j))


def merge(a, b):                        # dhla.py:305-318
    out = P.merge(a, b)
    out.params = a.params
    return out


def read_snapshot(src, backend="auto"):  # dhla.py:340-373
    sketch = P.read_snapshot(src)
    p = sketch.params
    sketch.params = dhsa.dhg.DhgParams(r=p.r, g=p.g, k=p.k, alpha=p.alpha, key_width=p.key_width,
                                       seed_dh0=p.seed_dh0, seed_h1=p.seed_h1)
    return sketch


dhsa.dhla.Dhla = Dhla
dhsa.dhla.merge = merge
dhsa.dhla.read_snapshot = read_snapshot
dhsa.dhla.write_snapshot = P.write_snapshot
dhsa.engine.Dhla = Dhla
dhsa.dhg.forward_many = cuda_dhg.forward_many
dhsa.dhg.reconstruct_many = cuda_dhg.reconstruct_many


if os.environ.get("DHSA_CUDA_SUITE_ENGINE") == "device":
    for _name in ("DetectionEngine", "WindowSession", "WindowConfig", "WindowResult", "split_pairs"):
        setattr(dhsa.engine, _name, getattr(P, _name))

BANNER = "dhsa_cuda_suite: dhsa.dhla / dhsa.engine / dhsa.dhg seams bound to libdhsa_b200.so"


def pytest_report_header(config):
    return BANNER


def pytest_terminal_summary(terminalreporter):
    try:
        sketch = dhsa.dhla.Dhla(dhsa.dhg.DhgParams())
        where = f"{sketch.backend_name}:{sketch.device}"
    except Exception as exc:  # no device (a collect-only run on a CPU box)
        where = f"no device ({type(exc).__name__})"
    terminalreporter.write_line(f"{BANNER}; sketches on {where}; engine: "
                                f"{dhsa.engine.DetectionEngine.__module__}")
