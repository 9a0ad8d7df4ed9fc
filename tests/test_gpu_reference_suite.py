"""The reference's own test files, unmodified, run against the CUDA sketch.

baseline/install_reference.sh leaves /root/reference/pkg/tests/*.py in baseline/_ref_tests
(git-ignored; it travels to the GPU box like baseline/_ref).  They are run here in a child pytest
with the plugin integration/dhsa_cuda_suite.py, which binds ``dhsa.dhla.Dhla`` / ``merge`` /
snapshots, ``dhsa.engine.Dhla`` and ``dhsa.dhg.*_many`` to this repository's device classes before
the reference's test modules import them.  Every assertion the reference makes about its sketch --
in-place writes to ``sketch.bits`` included -- is then made about the sketch in HBM.

Files: test_dhla.py (sketch, hot sets, flow count, restore, merge, snapshots), test_engine.py
(WindowSession / DetectionEngine), test_dhg.py (hash group), test_acceptance.py (release criteria
C1-C8), test_kernels.py (backend parity; its Backend-record tests exercise the reference's own
CPU kernels and pass trivially).  test_cli.py, test_ingest.py and test_estimator.py cover
subsystems outside the hot path and are not run.
"""
import os
import re
import subprocess
import sys

import pytest

import refpkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref_tests")
FILES = ["test_dhla.py", "test_engine.py", "test_dhg.py", "test_acceptance.py", "test_kernels.py"]

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (refpkg.available() and os.path.isdir(REF_TESTS)),
                                 reason="baseline/_ref(_tests) not installed (bash baseline/install_reference.sh)")]


def _run(tmp_path, files, engine):
    env = dict(os.environ)
    env["DHSA_CUDA_SUITE_ENGINE"] = engine
    env["PYTHONPATH"] = os.pathsep.join([ROOT, refpkg.INTEGRATION_DIR, refpkg.REF_DIR, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "dhsa_cuda_suite", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS, "-o", "addopts=", *[os.path.join(REF_TESTS, f) for f in files]]
    proc = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=1500)
    tail = "\n".join(proc.stdout.splitlines()[-40:]) + proc.stderr[-2000:]
    assert "dhsa_cuda_suite: dhsa.dhla / dhsa.engine / dhsa.dhg seams bound" in proc.stdout, tail
    summary = proc.stdout.strip().splitlines()[-1]
    counts = {k: int(v) for v, k in re.findall(r"(\d+) (passed|failed|error|errors|skipped)", summary)}
    print(summary)
    assert proc.returncode == 0, tail
    assert not counts.get("failed") and not counts.get("error") and not counts.get("errors"), tail
    return counts.get("passed", 0)


def test_reference_test_files_pass_against_the_cuda_sketch(tmp_path):
    """The reference's engine, unmodified, building CUDA sketches (engine.py:63)."""
    assert _run(tmp_path, FILES, "reference") >= 100   # the five files hold 109 test cases


def test_reference_engine_tests_pass_against_the_device_record_engine(tmp_path):
    """The package's own engine (records decoded, windowed and oriented on the GPU) under the
    reference's engine tests and its engine-driven release criteria (C5, C7)."""
    assert _run(tmp_path, ["test_engine.py", "test_acceptance.py"], "device") >= 25
