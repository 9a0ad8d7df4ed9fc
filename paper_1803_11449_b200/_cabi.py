"""ctypes binding of libdhsa_b200.so (include/dhsa_b200.h).

The library is the only implementation of the hot path: if it cannot be built
or loaded this module raises -- there is no CPU fallback to fall through to.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import _build
from .errors import CapacityError, ConfigError, CudaError, DataError


class Params(C.Structure):
    _fields_ = [
        ("r", C.c_int32), ("g", C.c_int32), ("k", C.c_int32), ("alpha", C.c_int32),
        ("key_width", C.c_int32), ("reserved", C.c_int32),
        ("state_dh0", C.c_uint64), ("state_h1", C.c_uint64),
    ]


class Report(C.Structure):
    _fields_ = [
        ("host", C.c_uint64), ("estimate", C.c_double),
        ("saturated", C.c_int32), ("shared_zero_count", C.c_int32),
    ]


class RestoreInfo(C.Structure):
    _fields_ = [
        ("n_candidates", C.c_uint64), ("n_reports", C.c_uint64),
        ("fail_stage", C.c_int32), ("flow_saturated", C.c_int32),
        ("fail_count", C.c_uint64),
        ("flow_count", C.c_double), ("psi", C.c_double), ("denom", C.c_double),
        ("hot_counts", C.c_uint64 * 64), ("stage_counts", C.c_uint64 * 64),
        ("zero_totals", C.c_int64 * 64),
        ("hot_cut", C.c_int32), ("sz_cut", C.c_int32),
    ]


_vp = C.c_void_p
_u64 = C.c_uint64
ABI_VERSION = 2   # DHSA_ABI_VERSION of include/dhsa_b200.h

# name -> argtypes; every symbol include/dhsa_b200.h declares (tests check the two agree)
SIGNATURES = {
    "dhsa_abi_version": [],
    "dhsa_last_error": [],
    "dhsa_create": [C.POINTER(Params), C.c_int, C.POINTER(_vp)],
    "dhsa_destroy": [_vp],
    "dhsa_release_cached": [],
    "dhsa_reset": [_vp],
    "dhsa_sketch_bytes": [_vp, C.POINTER(_u64)],
    "dhsa_bits_device_ptr": [_vp, C.POINTER(_vp)],
    "dhsa_set_stream": [_vp, _vp],
    "dhsa_set_own_stream": [_vp],
    "dhsa_get_stream": [_vp, C.POINTER(_vp)],
    "dhsa_set_scan_mode": [_vp, C.c_int],
    "dhsa_scan_mode_used": [_vp, C.POINTER(C.c_int)],
    "dhsa_set_flow_cache": [_vp, _u64],
    "dhsa_flow_cache_stats": [_vp, C.POINTER(_u64), C.POINTER(_u64)],
    "dhsa_launch_count": [_vp, C.POINTER(_u64)],
    "dhsa_update_device": [_vp, _vp, _vp, _u64],
    "dhsa_update_host": [_vp, _vp, _vp, _u64],
    "dhsa_update_device_from": [_vp, _vp, _vp, _u64, _vp],
    "dhsa_seal": [_vp],
    "dhsa_download_bits": [_vp, _vp, _u64],
    "dhsa_upload_bits": [_vp, _vp, _u64],
    "dhsa_download_range": [_vp, _u64, _u64, _vp],
    "dhsa_upload_range": [_vp, _u64, _u64, _vp],
    "dhsa_download_cell": [_vp, C.c_int32, _u64, _vp, _u64],
    "dhsa_zero_counts": [_vp, _vp, _vp],
    "dhsa_use_zero_counts": [_vp, _vp],
    "dhsa_hot_sets": [_vp, C.c_double, _vp, _vp],
    "dhsa_estimate": [_vp, C.c_double, C.POINTER(RestoreInfo)],
    "dhsa_candidate_hosts": [_vp, C.c_double, _u64, _vp, _u64, C.POINTER(RestoreInfo)],
    "dhsa_shared_zero_counts": [_vp, _vp, _u64, _vp],
    "dhsa_restore": [_vp, C.c_double, _u64, _vp, _u64, C.POINTER(RestoreInfo)],
    "dhsa_restore_begin": [_vp, C.c_double, _u64],
    "dhsa_restore_end": [_vp, _vp, _u64, C.POINTER(RestoreInfo)],
    "dhsa_forward_many": [C.POINTER(Params), C.c_int, _vp, _u64, _vp],
    "dhsa_reconstruct_many": [C.POINTER(Params), C.c_int, _vp, _u64, _vp, _vp],
    "dhsa_plan_windows": [_vp, _vp, _u64, C.c_uint32, C.c_int64, _vp, C.c_uint32, C.POINTER(C.c_uint32)],
    "dhsa_update_records_device": [_vp, _vp, _u64, _u64, _u64, C.c_uint32, C.c_uint32, C.c_int],
    "dhsa_record_tally": [_vp, C.POINTER(_u64), C.POINTER(_u64)],
    "dhsa_record_tally_at_restore": [_vp, C.POINTER(_u64), C.POINTER(_u64)],
    "dhsa_exact_create": [C.c_int, _u64, C.POINTER(_vp)],
    "dhsa_exact_destroy": [_vp],
    "dhsa_exact_add_pairs": [_vp, _vp, _vp, _u64, _vp],
    "dhsa_exact_add_records": [_vp, _vp, _u64, _u64, _u64, C.c_uint32, C.c_uint32, C.c_int, _vp],
    "dhsa_exact_result": [_vp, _u64, _vp, _vp, _u64, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), _vp],
    "dhsa_generate_trace": [C.c_int, _vp, _vp, _vp, C.c_uint32, _u64, _u64, _u64, C.c_uint32, C.c_uint32, _u64, _u64,
                            _vp, _vp, _vp, _vp],
    "dhsa_copy_to_device_async": [C.c_int, _vp, _vp, _u64, _vp],
    "dhsa_or_merge": [_vp, _vp],
    "dhsa_or_merge_peers": [_vp, C.POINTER(_vp), C.c_int, _u64, _u64],
    "dhsa_copy_slice_from_peer": [_vp, _vp, _u64, _u64],
    "dhsa_or_merge_buffer": [_vp, _vp, _u64],
    "dhsa_zero_counts_range": [_vp, _u64, _u64],
    "dhsa_zero_counts_offset": [_vp, C.POINTER(_u64)],
    "dhsa_gather_zero_counts_from_peer": [_vp, _vp, _u64, _u64],
    "dhsa_set_cell_owners": [_vp, C.POINTER(_vp), C.POINTER(_u64), C.c_int],
    "dhsa_ipc_export": [_vp, _vp],
    "dhsa_ipc_open": [C.c_int, _vp, C.POINTER(_vp)],
    "dhsa_ipc_close": [C.c_int, _vp],
    "dhsa_selftest_copy_pool": [_u64, C.c_int, C.c_int, C.POINTER(_u64)],
    "dhsa_probe_l2": [C.c_int, C.c_int, _u64, _u64, C.POINTER(C.c_double)],
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load (building first if the sources are newer) libdhsa_b200.so."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                path = _build.LIB_PATH
                if os.environ.get("DHSA_LIB"):      # a tuning variant built by _build.build_variant
                    path = os.environ["DHSA_LIB"]
                elif _build.stale():
                    if os.environ.get("DHSA_NO_BUILD") and os.path.exists(path):
                        pass
                    else:
                        path = _build.build()
                L = C.CDLL(path)
                for name, argtypes in SIGNATURES.items():
                    fn = getattr(L, name)  # AttributeError here = header and library disagree
                    fn.argtypes = argtypes
                    fn.restype = C.c_int
                L.dhsa_last_error.restype = C.c_char_p
                if L.dhsa_abi_version() != ABI_VERSION:
                    raise ConfigError(f"libdhsa_b200.so ABI {L.dhsa_abi_version()} != {ABI_VERSION}")
                _lib = L
    return _lib


def last_error() -> str:
    msg = lib().dhsa_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int) -> None:
    """Map a C-ABI return code onto the reference's exception classes."""
    if rc == 0:
        return
    msg = last_error()
    if rc == 2:
        raise ConfigError(msg)
    if rc == 3:
        raise DataError(msg)
    if rc == 4:
        raise CapacityError(msg)
    raise CudaError(f"libdhsa_b200 call failed ({rc}): {msg}")
