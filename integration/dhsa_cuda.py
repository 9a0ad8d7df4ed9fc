"""Reference-side binding of libdhsa_b200.so -- the file a maintainer of the reference would add
as ``pkg/src/dhsa/_cuda.py``.

It depends on the reference's own package (``dhsa``), numpy and ctypes only -- NOT on this
repository's Python layer -- and talks to the library through the C ABI of
``include/dhsa_b200.h``.  ``CudaDhla`` offers what the reference's window engine and CLI touch
on a sketch (``/root/reference/pkg/src/dhsa/engine.py:63,74,84-86,99-103``,
``cli.py:383,395``, ``dhla.py:321-333``), so

    import dhsa.engine, dhsa_cuda
    dhsa_cuda.install(dhsa.engine)          # engine.py:63 now builds CudaDhla sketches

lets the UNMODIFIED ``WindowSession`` / ``DetectionEngine`` run on the GPU.
``tests/test_gpu_reference_engine.py`` executes exactly this against the installed reference
(baseline/_ref) and compares with its compiled CPU backend; INTEGRATION.md walks through it.
"""
import ctypes as C
import os

import numpy as np

from dhsa.dhla import SuperPointReport
from dhsa.errors import CapacityError, ConfigError, DataError

_LIB_PATH = os.environ.get("DHSA_B200_LIB") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1803_11449_b200", "libdhsa_b200.so")
ABI_VERSION = 2


class Params(C.Structure):          # dhsa_params_t
    _fields_ = [("r", C.c_int32), ("g", C.c_int32), ("k", C.c_int32), ("alpha", C.c_int32),
                ("key_width", C.c_int32), ("reserved", C.c_int32),
                ("state_dh0", C.c_uint64), ("state_h1", C.c_uint64)]


class RestoreInfo(C.Structure):     # dhsa_restore_info_t
    _fields_ = [("n_candidates", C.c_uint64), ("n_reports", C.c_uint64),
                ("fail_stage", C.c_int32), ("flow_saturated", C.c_int32), ("fail_count", C.c_uint64),
                ("flow_count", C.c_double), ("psi", C.c_double), ("denom", C.c_double),
                ("hot_counts", C.c_uint64 * 64), ("stage_counts", C.c_uint64 * 64),
                ("zero_totals", C.c_int64 * 64), ("hot_cut", C.c_int32), ("sz_cut", C.c_int32)]


REPORT = np.dtype([("host", "<u8"), ("estimate", "<f8"), ("saturated", "<i4"), ("sz", "<i4")])   # dhsa_report_t

_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(_LIB_PATH)
        L.dhsa_last_error.restype = C.c_char_p
        if L.dhsa_abi_version() != ABI_VERSION:
            raise ConfigError(f"libdhsa_b200.so has ABI {L.dhsa_abi_version()}, this binding speaks {ABI_VERSION}")
        _lib = L
    return _lib


def _check(rc):
    if rc:
        msg = lib().dhsa_last_error().decode()
        raise {2: ConfigError, 3: DataError, 4: CapacityError}.get(rc, RuntimeError)(msg)


class CudaDhla:
    """dhsa.dhla.Dhla on a B200 (dhla.py:57-196), through the C ABI."""

    backend_name = "cuda"

    def __init__(self, params, backend="cuda", window_id=0, device=0):
        self.params, self.window_id = params, window_id
        p = Params(params.r, params.g, params.k, params.alpha, params.key_width, 0,
                   params.state_dh0, params.state_h1)             # dhg.py:112-118
        self._h = C.c_void_p()
        _check(lib().dhsa_create(C.byref(p), device, C.byref(self._h)))

    def update_batch(self, candidates, opposites):                # dhla.py:87-95
        c = np.ascontiguousarray(candidates, dtype=np.uint32)
        o = np.ascontiguousarray(opposites, dtype=np.uint32)
        if len(c) != len(o):
            raise ValueError("candidate and opposite arrays differ in length")
        _check(lib().dhsa_update_host(self._h, C.c_void_p(c.ctypes.data), C.c_void_p(o.ctypes.data),
                                      C.c_uint64(len(c))))

    def restore_superpoints(self, theta, max_candidates=1 << 20, workers=1):   # dhla.py:164-196
        info, cap = RestoreInfo(), 4096
        while True:
            rows = np.empty(cap, dtype=REPORT)
            rc = lib().dhsa_restore(self._h, C.c_double(theta), C.c_uint64(max_candidates),
                                    C.c_void_p(rows.ctypes.data), C.c_uint64(cap), C.byref(info))
            if rc == 3 and info.n_reports > cap:                  # more reports than rows: ask again
                cap = int(info.n_reports)
                continue
            _check(rc)
            return [SuperPointReport(int(r["host"]), float(r["estimate"]), bool(r["saturated"]))
                    for r in rows[: info.n_reports]]

    @property
    def bits(self):                                               # dhla.py:64-67 (a copy: the array lives in HBM)
        p = self.params
        out = np.empty((p.r, p.index_count, p.g // 8), dtype=np.uint8)
        _check(lib().dhsa_download_bits(self._h, C.c_void_p(out.ctypes.data), C.c_uint64(out.nbytes)))
        return out

    @property
    def memory_bytes(self):                                       # dhla.py:74-76
        n = C.c_uint64()
        _check(lib().dhsa_sketch_bytes(self._h, C.byref(n)))
        return int(n.value)

    def reset(self):                                              # dhla.py:97-99
        _check(lib().dhsa_reset(self._h))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().dhsa_destroy(self._h)
            self._h = None


def install(engine_module):
    """Make ``engine_module.WindowSession`` (engine.py:63) build CudaDhla sketches; returns the
    class it replaced so a caller can put it back."""
    previous = engine_module.Dhla
    engine_module.Dhla = lambda params, backend="auto", window_id=0: CudaDhla(params, "cuda", window_id)
    return previous
