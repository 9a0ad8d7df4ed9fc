"""CPU-side checks: parameter validation, the C-ABI surface, loud failure without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_1803_11449_b200 as P
from paper_1803_11449_b200 import _cabi, dhg

from helpers import load_json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONST = load_json("constants.json")


def _have_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def test_default_params_and_states_match_reference():
    p = P.DhgParams()
    assert (p.r, p.g, p.k, p.alpha, p.key_width) == (5, 1024, 14, 6, 32)
    assert p.state_dh0 == CONST["state_dh0"] and p.state_h1 == CONST["state_h1"]
    assert p.sketch_bytes == 10_485_760 and p.index_count == 16384
    for x, want in CONST["mix64"].items():
        assert dhg.mix64(int(x)) == want
    for a, want in CONST["forward"].items():
        assert list(dhg.forward(p, int(a))) == want
    for b, want in CONST["h1"].items():
        assert dhg.h1(p, int(b)) == want


@pytest.mark.parametrize("kw, fragment", [
    # pkg/tests/test_dhg.py:152-175 -- every rule names its inequality
    (dict(r=2), "r >= 3"),
    (dict(g=100), "power of two"),
    (dict(g=4), "power of two"),
    (dict(k=0), "1 <= k <= 30"),
    (dict(k=31), "1 <= k <= 30"),
    (dict(key_width=7), "8 <= key_width <= 32"),
    (dict(key_width=33), "8 <= key_width <= 32"),
    (dict(k=14, key_width=12), "k <= key_width"),
    (dict(alpha=0), "1 <= alpha <= k"),
    (dict(alpha=15), "1 <= alpha <= k"),
    (dict(r=3, alpha=6, k=14), "(r-2)*alpha + k >= key_width"),
    (dict(r=5, k=30, alpha=30, key_width=32), "<= 64"),
    (dict(seed_dh0=-1), "unsigned 64-bit"),
    (dict(seed_h1=2 ** 64), "unsigned 64-bit"),
])
def test_param_validation_names_the_rule(kw, fragment):
    with pytest.raises(P.ConfigError) as err:
        P.DhgParams(**kw)
    assert fragment in str(err.value)
    assert isinstance(err.value, ValueError)  # ConfigError is a ValueError, as in the reference


def test_coerce_accepts_reference_shaped_records():
    from types import SimpleNamespace

    rec = SimpleNamespace(r=4, g=64, k=8, alpha=4, key_width=16, seed_dh0=1, seed_h1=2)
    p = P.DhgParams.coerce(rec)
    assert (p.r, p.g, p.k, p.alpha, p.key_width, p.seed_dh0, p.seed_h1) == (4, 64, 8, 4, 16, 1, 2)


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "dhsa_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dhsa_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _cabi.lib()
    declared = _declared_symbols()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in include/dhsa_b200.h but not exported"
    assert sorted(_cabi.SIGNATURES) == declared
    assert lib.dhsa_abi_version() == _cabi.ABI_VERSION == 2


def test_struct_layouts_match_header():
    assert C.sizeof(_cabi.Params) == 40
    assert C.sizeof(_cabi.Report) == 24
    assert C.sizeof(_cabi.RestoreInfo) == 8 * 2 + 4 * 2 + 8 + 8 * 3 + 64 * 8 * 3 + 4 * 2
    assert _cabi.RestoreInfo.n_reports.offset == 8 and _cabi.RestoreInfo.sz_cut.offset == 1596
    # the header's own words for the same structs: field order and types, parsed from include/dhsa_b200.h
    text = open(os.path.join(ROOT, "include", "dhsa_b200.h")).read()
    ctype = {"int32_t": C.c_int32, "uint64_t": C.c_uint64, "int64_t": C.c_int64, "double": C.c_double}
    for name, binding in (("dhsa_params_t", _cabi.Params), ("dhsa_report_t", _cabi.Report),
                          ("dhsa_restore_info_t", _cabi.RestoreInfo)):
        body = re.search(r"typedef struct \{([^}]*)\} " + name + ";", text).group(1)
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        fields = re.findall(r"(int32_t|uint64_t|int64_t|double)\s+(\w+)(?:\[(\d+)\])?;", body)
        want = [(f, ctype[t] * int(n) if n else ctype[t]) for t, f, n in fields]
        got = [(f, t) for f, t in binding._fields_]
        assert [f for f, _ in got] == [f for f, _ in want], name
        assert [C.sizeof(t) for _, t in got] == [C.sizeof(t) for _, t in want], name


def test_reference_side_binding_structs_match_the_library_binding():
    """integration/dhsa_cuda.py (the file a maintainer adds to the reference) declares
    the ABI's structs on its own; they must be the ones the library was built with."""
    import refpkg

    if not refpkg.available():
        pytest.skip("baseline/_ref not installed (bash baseline/install_reference.sh)")
    _, stub = refpkg.load()
    assert stub.ABI_VERSION == _cabi.ABI_VERSION
    for mine, theirs in ((_cabi.Params, stub.Params), (_cabi.RestoreInfo, stub.RestoreInfo)):
        assert C.sizeof(mine) == C.sizeof(theirs)
        assert [(f, C.sizeof(t)) for f, t in mine._fields_] == [(f, C.sizeof(t)) for f, t in theirs._fields_]
    assert stub.REPORT.itemsize == C.sizeof(_cabi.Report)
    assert os.path.samefile(stub._LIB_PATH, os.path.join(ROOT, "paper_1803_11449_b200", "libdhsa_b200.so"))
    lib = C.CDLL(stub._LIB_PATH)
    for name in re.findall(r"lib\(\)\.(dhsa_\w+)", open(stub.__file__).read()):
        assert hasattr(lib, name), name


def test_installed_reference_is_the_unmodified_package_with_its_compiled_backend():
    import refpkg

    if not refpkg.available():
        pytest.skip("baseline/_ref not installed (bash baseline/install_reference.sh)")
    dhsa, _ = refpkg.load()
    from dhsa._kernels import available_backends

    assert available_backends() == ("compiled", "python")
    assert os.path.realpath(dhsa.__file__).startswith(os.path.realpath(refpkg.REF_DIR))
    src = "/root/reference/pkg/src/dhsa"
    if os.path.isdir(src):          # in this container: byte-identical to the reference's sources
        for f in sorted(os.listdir(src)):
            if f.endswith(".py"):
                assert open(os.path.join(src, f), "rb").read() == \
                    open(os.path.join(refpkg.REF_DIR, "dhsa", f), "rb").read(), f


def test_c_side_validation_maps_to_config_error():
    lib = _cabi.lib()
    bad = _cabi.Params(2, 1024, 14, 6, 32, 0, 1, 2)
    h = C.c_void_p()
    rc = lib.dhsa_create(C.byref(bad), 0, C.byref(h))
    assert rc == 2
    with pytest.raises(P.ConfigError, match="r >= 3"):
        _cabi.check(rc)


def test_unknown_backend_is_config_error():
    # pkg/tests/test_kernels.py:89-91: closed set of names; CPU names do not exist here
    for name in ("compiled", "python", "numpy"):
        with pytest.raises(P.ConfigError):
            P.Dhla(P.DhgParams(), backend=name)


@pytest.mark.skipif(_have_gpu(), reason="only meaningful without a GPU")
def test_no_gpu_fails_loudly_not_silently():
    with pytest.raises(P.CudaError):
        P.Dhla(P.DhgParams())


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1803_11449_b200")
    for base, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(base, f)).read()
                # `exact_oracle` is the reference's name for the ground-truth counter
                # (ingest.py:159-176), mirrored in exact.py; it is not the oracle/ directory.
                text = text.replace("no CPU oracle", "").replace("exact_oracle", "exact_truth")
                text = text.replace("the exact oracle", "").replace("Exact oracle", "")
                assert not re.search(r"(^\s*import\s+oracle|^\s*from\s+\.*oracle|dhsa_oracle|liboracle|oracle/_ref|oracle\.oracle)", text, re.M), \
                    f"{f} reaches into oracle/"


def test_library_has_no_device_function_host_stubs_on_call_paths():
    """nvcc compiles a __device__ function that host code calls inside a template into an
    exit(1) stub instead of an error; make sure none is reachable in the built library."""
    import shutil
    import subprocess

    from paper_1803_11449_b200 import _build

    if shutil.which("objdump") is None:
        pytest.skip("objdump not available")
    _cabi.lib()
    asm = subprocess.run(["objdump", "-d", "--no-show-raw-insn", _build.LIB_PATH], capture_output=True, text=True).stdout
    assert "<exit@plt>" not in asm.replace("<__cxa_atexit@plt>", "")


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_copy_pool_is_exact_under_concurrent_callers(threads):
    """The helper-thread pool that copies host batches into the page-locked slots (lock-free share claims,
    helpers that go to sleep and wake late): every byte of every copy arrives, whoever shares the pool.
    Host-only: runs without a GPU."""
    lib = _cabi.lib()
    bad = C.c_uint64(12345)
    _cabi.check(lib.dhsa_selftest_copy_pool(1 << 20, 400, threads, C.byref(bad)))
    assert bad.value == 0
    _cabi.check(lib.dhsa_selftest_copy_pool(200_000, 3000, threads, C.byref(bad)))     # small jobs: share count varies
    assert bad.value == 0


def test_bits_mirror_writes_through_and_copies_detach():
    """Dhla.bits is a write-through host mirror (the reference writes sketch.bits[...] in place,
    pkg/tests/test_dhla.py:88-90,139; test_kernels.py:57): item assignment on the mirror or a view
    uploads it, copies and arithmetic results are detached.  Host-only: a stand-in sketch."""
    from paper_1803_11449_b200.dhla import DeviceBits

    class Sketch:
        def __init__(self):
            self.dev, self.uploads = np.zeros((2, 4, 8), np.uint8), 0

        def load_bits(self, a):
            self.dev[...] = a
            self.uploads += 1

        @property
        def bits(self):
            m = self.dev.copy().view(DeviceBits)
            m._sketch = self                 # as Dhla.bits builds it: the root carries no reference to itself
            return m

    s = Sketch()
    s.bits[0, 1, :3] = 0xFF
    assert s.dev[0, 1, :3].tolist() == [255] * 3 and s.uploads == 1
    s.bits[:] = 1
    assert s.dev.sum() == s.dev.size and s.uploads == 2
    view = s.bits[1]
    view[0, 0] = 7                                   # a view writes the whole mirror back
    assert s.dev[1, 0, 0] == 7 and s.dev[0].sum() == 32 and s.uploads == 3
    detached = s.bits.copy()
    detached[0, 0, 0] = 9
    (s.bits | 1)[0, 0, 0] = 9
    np.asarray(s.bits)[0, 0, 0] = 9
    assert s.uploads == 3 and s.dev[0, 0, 0] == 1
    assert np.array_equal(s.bits, s.dev) and len(s.bits.tobytes()) == s.dev.size
    import pickle

    assert type(pickle.loads(pickle.dumps(s.bits))) is np.ndarray
    # a mirror (and the sketch it points to) goes away with its last reference, not with the next cyclic collection:
    # `sketch.bits` per window must not pile up 10 MiB arrays and device sketches
    import gc
    import weakref

    gc.disable()
    try:
        t = Sketch()
        mirror = t.bits
        row = mirror[1]
        probe_m, probe_s = weakref.ref(mirror), weakref.ref(t)
        del mirror
        assert probe_m() is not None                 # the view keeps its root alive (it uploads the whole mirror)
        row[0, 0] = 3
        assert t.dev[1, 0, 0] == 3
        del row, t
        assert probe_m() is None and probe_s() is None
    finally:
        gc.enable()


def test_exceptions_derive_from_the_reference_classes_when_it_is_importable():
    """`except dhsa.errors.CapacityError` in a host application must catch what the CUDA sketch
    raises (errors.py); without the reference on the path the hierarchy stands alone."""
    import subprocess
    import sys

    import refpkg
    import paper_1803_11449_b200.errors as E

    for name, bases in (("ConfigError", (E.DhsaError, ValueError)), ("DataError", (E.DhsaError,)),
                        ("CapacityError", (E.DhsaError,)), ("SealedWindowError", (E.DhsaError, RuntimeError)),
                        ("CudaError", (E.DhsaError, RuntimeError))):
        assert all(issubclass(getattr(E, name), b) for b in bases), name
    if not refpkg.available():
        pytest.skip("baseline/_ref not installed (bash baseline/install_reference.sh)")
    code = ("import sys; sys.path[:0] = [%r, %r]\n"
            "import dhsa.errors as R, paper_1803_11449_b200.errors as E\n"
            "for n in ('DhsaError', 'ConfigError', 'DataError', 'CapacityError', 'SealedWindowError'):\n"
            "    assert issubclass(getattr(E, n), getattr(R, n)) and issubclass(getattr(E, n), E.DhsaError), n\n"
            "assert issubclass(E.ConfigError, ValueError) and issubclass(E.CudaError, R.DhsaError)\n"
            % (ROOT, refpkg.REF_DIR))
    subprocess.run([sys.executable, "-c", code], check=True)
