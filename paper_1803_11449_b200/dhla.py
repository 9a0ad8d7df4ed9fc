"""The device-resident sketch: drop-in for the reference's ``dhsa.dhla.Dhla``.

Same constructor, attributes and methods as
/root/reference/pkg/src/dhsa/dhla.py:57-196 (and ``merge`` :305-318), so the
reference's window engine (pkg/src/dhsa/engine.py:57-103) can hold one of these
where it holds a ``Dhla`` -- it only touches ``Dhla(params, backend=,
window_id=)``, ``update_batch``, ``window_id`` and ``restore_superpoints(theta,
max_candidates=, workers=)``.

Every data-path method is a call into libdhsa_b200.so (include/dhsa_b200.h);
Python only moves arguments and shapes results.  The one contract that needs
care is ``bits``: the array lives in HBM, so the attribute is a host mirror
taken after the sketch's stream drains.  The reference writes ``sketch.bits[...]``
in place (pkg/src/dhsa/dhla.py:372, pkg/tests/test_dhla.py:88-90,139); the mirror
is therefore write-through -- an item assignment into it (or into a view of it)
uploads the mirror to the device -- and ``load_bits`` is the explicit bulk write.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import NamedTuple, Optional

import numpy as np

from . import _cabi
from .dhg import DhgParams
from .errors import ConfigError

DEFAULT_MAX_CANDIDATES = 1 << 20  # pkg/src/dhsa/dhla.py:34

SCAN_MODES = {"red": 0, "test": 1, "test_agg": 2, "flow_cache": 3, "auto": 4}

_REPORT_DTYPE = np.dtype([("host", "<u8"), ("estimate", "<f8"), ("saturated", "<i4"), ("sz", "<i4")])
assert _REPORT_DTYPE.itemsize == C.sizeof(_cabi.Report)


def hot_threshold(g: int, theta: int) -> float:
    """Zmin = g exp(-theta/g) (pkg/src/dhsa/dhla.py:45-47)."""
    return g * math.exp(-theta / g)


@dataclass(frozen=True)
class SuperPointReport:  # pkg/src/dhsa/dhla.py:50-54
    host: int
    estimate: float
    saturated: bool


class Estimate(NamedTuple):  # pkg/src/dhsa/estimator.py:21-23
    value: float
    saturated: bool


def _default_device() -> int:
    env = os.environ.get("DHSA_DEVICE", os.environ.get("LOCAL_RANK"))
    return int(env) if env not in (None, "") else 0


def _same_params(a, b) -> bool:
    """Field-wise equality: a sketch may carry the reference's own DhgParams record (dhg.py:59-76)."""
    return DhgParams.coerce(a) == DhgParams.coerce(b)


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "data_ptr") and getattr(x, "is_cuda", False)


class DeviceBits(np.ndarray):
    """Host mirror of a device sketch's bit array, as ``Dhla.bits`` returns it.

    Reading is plain numpy.  ``mirror[...] = value`` -- on the mirror itself or on any view of it
    (``sketch.bits[1, 9, 80] = 0x7F``, ``sketch.bits[i] = cells``) -- also uploads the mirror, so
    code written against the reference's live host array (pkg/src/dhsa/dhla.py:64-67,372) keeps
    working.  Every such write moves the whole array (10 MiB at the defaults) over PCIe: edit a
    plain copy and call ``load_bits`` once for anything bulky.  Copies and arithmetic results are
    ordinary detached arrays.
    """

    _sketch = None  # the Dhla a write goes back to
    _root = None    # a view: the whole (r, 2^k, g/8) mirror it is a view of; the mirror itself: None (a reference to
                    # itself would be a cycle: 10 MiB per `sketch.bits`, and the sketch behind it, kept until the
                    # cyclic collector runs)

    def __array_finalize__(self, obj):
        if isinstance(obj, DeviceBits) and obj._sketch is not None and self.base is not None \
                and np.shares_memory(self, obj):
            self._sketch, self._root = obj._sketch, (obj if obj._root is None else obj._root)
        else:
            self._sketch = self._root = None

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        if self._sketch is not None:
            self._sketch.load_bits(np.asarray(self if self._root is None else self._root))

    def __reduce__(self):  # pickles as a plain array: a handle to a device sketch does not travel
        return np.asarray(self).__reduce__()


class Dhla:
    """r * 2^k byte-packed linear estimators in HBM, addressed by the hash group."""

    def __init__(self, params, backend="auto", window_id: int = 0, device: Optional[int] = None):
        # The reference resolves names through get_backend and passes a Backend INSTANCE through
        # unchanged (pkg/src/dhsa/_kernels.py:42-55, dhla.py:60-63).  Its Backend functions work on a
        # host bits array, which this sketch does not have: only a record naming this backend is
        # accepted, everything else is refused in the reference's wording.
        name = backend if isinstance(backend, str) else getattr(backend, "name", backend)
        if name not in ("auto", "cuda"):
            # the reference's names ("compiled", "python") are CPU kernels; none exist here
            raise ConfigError(f"unknown backend {name!r}; expected auto or cuda "
                              f"(this build has only the CUDA path)")
        self.params = DhgParams.coerce(params)
        self.window_id = window_id
        self.device = _default_device() if device is None else int(device)
        p = self.params
        self._cparams = _cabi.Params(p.r, p.g, p.k, p.alpha, p.key_width, 0, p.state_dh0, p.state_h1)
        self._lib = _cabi.lib()
        h = C.c_void_p()
        _cabi.check(self._lib.dhsa_create(C.byref(self._cparams), self.device, C.byref(h)))
        self._h = h
        self._stream_ref = None   # keeps a caller's stream object alive while the sketch launches on it
        self.last_info: Optional[dict] = None

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                self._lib.dhsa_destroy(h)
            except Exception:
                pass

    # --- identity -----------------------------------------------------------

    @property
    def backend_name(self) -> str:
        return "cuda"

    @property
    def memory_bytes(self) -> int:
        n = C.c_uint64()
        _cabi.check(self._lib.dhsa_sketch_bytes(self._h, C.byref(n)))
        return int(n.value)

    @property
    def bits_device_ptr(self) -> int:
        ptr = C.c_void_p()
        _cabi.check(self._lib.dhsa_bits_device_ptr(self._h, C.byref(ptr)))
        return int(ptr.value)

    @property
    def launch_count(self) -> int:
        n = C.c_uint64()
        _cabi.check(self._lib.dhsa_launch_count(self._h, C.byref(n)))
        return int(n.value)

    def use_stream(self, cuda_stream) -> None:
        """Launch on this stream: a stream object exposing ``cuda_stream`` (a torch.cuda.Stream --
        the sketch then holds a reference, so the handle stays valid for as long as it is used) or
        a raw cudaStream_t handle the caller keeps alive (0 = CUDA's legacy default stream, which
        is what torch's default stream reports); None -> back to the sketch's own stream."""
        if cuda_stream is None:
            _cabi.check(self._lib.dhsa_set_own_stream(self._h))
            self._stream_ref = None
            return
        handle = getattr(cuda_stream, "cuda_stream", cuda_stream)
        _cabi.check(self._lib.dhsa_set_stream(self._h, C.c_void_p(int(handle))))
        self._stream_ref = cuda_stream if handle is not cuda_stream else None

    @property
    def stream_handle(self) -> int:
        """The cudaStream_t this sketch launches on."""
        ptr = C.c_void_p()
        _cabi.check(self._lib.dhsa_get_stream(self._h, C.byref(ptr)))
        return int(ptr.value or 0)

    def set_scan_mode(self, mode) -> None:
        _cabi.check(self._lib.dhsa_set_scan_mode(self._h, SCAN_MODES.get(mode, mode)))

    @property
    def scan_mode_used(self) -> str:
        """The kernel variant the last vectorised scan launch used (what "auto" resolved to)."""
        m = C.c_int()
        _cabi.check(self._lib.dhsa_scan_mode_used(self._h, C.byref(m)))
        return {v: k for k, v in SCAN_MODES.items()}[int(m.value)]

    def set_flow_cache(self, n_sets: int) -> None:
        """Size of the flow cache used by scan mode "flow_cache": n_sets x 32 bytes."""
        _cabi.check(self._lib.dhsa_set_flow_cache(self._h, int(n_sets)))

    def flow_cache_stats(self) -> tuple:
        """(keys looked up, keys found) since the last reset."""
        a, b = C.c_uint64(), C.c_uint64()
        _cabi.check(self._lib.dhsa_flow_cache_stats(self._h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    # --- the bits attribute ----------------------------------------------------

    @property
    def bits(self) -> np.ndarray:
        """Host mirror, shape (r, 2^k, g/8) uint8, the reference's layout; item assignment
        writes through to the device (DeviceBits)."""
        p = self.params
        out = np.empty((p.r, p.index_count, p.g // 8), dtype=np.uint8)
        _cabi.check(self._lib.dhsa_download_bits(self._h, out.ctypes.data, out.nbytes))
        mirror = out.view(DeviceBits)
        mirror._sketch = self          # _root stays None: this IS the root
        return mirror

    def estimator(self, i: int, j: int) -> np.ndarray:
        """The g/8 bytes of estimator j of array i (pkg/src/dhsa/dhla.py:107-109).  A copy: the
        reference returns a LinearEstimator view over its host array; here the bits live on the
        device (wrap the bytes in the reference's LinearEstimator if that class is wanted)."""
        out = np.empty(self.params.g // 8, dtype=np.uint8)
        _cabi.check(self._lib.dhsa_download_cell(self._h, int(i), int(j), out.ctypes.data, out.nbytes))
        return out

    def load_bits(self, bits: np.ndarray) -> None:
        p = self.params
        arr = np.ascontiguousarray(bits, dtype=np.uint8)
        if arr.shape != (p.r, p.index_count, p.g // 8):
            raise ConfigError(f"bits must have shape {(p.r, p.index_count, p.g // 8)}, got {arr.shape}")
        _cabi.check(self._lib.dhsa_upload_bits(self._h, arr.ctypes.data, arr.nbytes))

    # --- update phase ------------------------------------------------------------

    def update(self, candidate: int, opposite: int) -> None:
        self.update_batch(np.array([candidate], dtype=np.uint32), np.array([opposite], dtype=np.uint32))

    def update_batch(self, candidates, opposites) -> None:
        """Scan a batch of pairs (pkg/src/dhsa/dhla.py:87-95).

        numpy (or any host array-like): staged to the device inside the call.
        torch CUDA tensors (int32/uint32, contiguous): scanned in place on
        torch's current stream.
        """
        if _is_cuda_tensor(candidates) or _is_cuda_tensor(opposites):
            self._update_device(candidates, opposites)
            return
        cand = np.ascontiguousarray(candidates, dtype=np.uint32)
        opp = np.ascontiguousarray(opposites, dtype=np.uint32)
        if cand.shape != opp.shape or cand.ndim != 1:
            raise ValueError("candidate and opposite arrays differ in length")
        _cabi.check(self._lib.dhsa_update_host(self._h, cand.ctypes.data, opp.ctypes.data, len(cand)))

    def _update_device(self, cand, opp) -> None:
        import torch

        if not (_is_cuda_tensor(cand) and _is_cuda_tensor(opp)):
            raise ValueError("candidates and opposites must both be CUDA tensors")
        if cand.numel() != opp.numel() or cand.dim() != 1 or opp.dim() != 1:
            raise ValueError("candidate and opposite arrays differ in length")
        for t in (cand, opp):
            if t.element_size() != 4 or t.is_floating_point() or not t.is_contiguous():
                raise ValueError("device inputs must be contiguous 32-bit integer tensors")
            if t.device.index != self.device:
                raise ConfigError(f"tensor on cuda:{t.device.index}, sketch on cuda:{self.device}")
        # The tensors were produced on torch's current stream.  The sketch keeps launching on its own
        # stream: the library orders the two with events in both directions (the scan waits for the
        # producer, the producer's later work -- e.g. the allocator reusing these tensors -- waits
        # for the scan), so no handle of a possibly short-lived torch stream is ever stored.
        producer = torch.cuda.current_stream(self.device).cuda_stream
        _cabi.check(self._lib.dhsa_update_device_from(self._h, cand.data_ptr(), opp.data_ptr(), cand.numel(),
                                                      C.c_void_p(producer)))

    def seal(self) -> None:
        """Drain the stream: every update issued so far is in the bits."""
        _cabi.check(self._lib.dhsa_seal(self._h))

    def reset(self, window_id: int = 0) -> None:
        _cabi.check(self._lib.dhsa_reset(self._h))
        self.window_id = window_id

    # --- read-out ------------------------------------------------------------------

    def zero_counts(self) -> np.ndarray:
        p = self.params
        out = np.empty((p.r, p.index_count), dtype=np.int64)
        _cabi.check(self._lib.dhsa_zero_counts(self._h, out.ctypes.data, None))
        return out

    def _hand_in(self, zero_counts) -> None:
        """The reference's optional ``zero_counts=`` argument: the next read-out call starts from
        these counts instead of counting the bits (pkg/src/dhsa/dhla.py:111-128,198-207)."""
        if zero_counts is None:
            return
        p = self.params
        zc = np.ascontiguousarray(zero_counts, dtype=np.int64)
        if zc.shape != (p.r, p.index_count):
            raise ValueError(f"zero_counts must have shape {(p.r, p.index_count)}, got {zc.shape}")
        _cabi.check(self._lib.dhsa_use_zero_counts(self._h, zc.ctypes.data))

    def hot_sets(self, theta, zero_counts=None) -> list:
        """Per-array ascending hot indices (pkg/src/dhsa/dhla.py:111-119)."""
        p = self.params
        self._hand_in(zero_counts)
        lists = np.empty((p.r, p.index_count), dtype=np.uint64)
        counts = np.empty(p.r, dtype=np.uint64)
        _cabi.check(self._lib.dhsa_hot_sets(self._h, float(theta), lists.ctypes.data, counts.ctypes.data))
        return [lists[i, : int(counts[i])].copy() for i in range(p.r)]

    def _info_dict(self, info: _cabi.RestoreInfo) -> dict:
        r = self.params.r
        return dict(
            n_candidates=int(info.n_candidates), n_reports=int(info.n_reports),
            fail_stage=int(info.fail_stage), fail_count=int(info.fail_count),
            flow_count=float(info.flow_count), flow_saturated=bool(info.flow_saturated),
            psi=float(info.psi), denom=float(info.denom),
            hot_counts=[int(info.hot_counts[i]) for i in range(r)],
            stage_counts=[int(info.stage_counts[i]) for i in range(r - 2)],
            zero_totals=[int(info.zero_totals[i]) for i in range(r)],
            hot_cut=int(info.hot_cut), sz_cut=int(info.sz_cut),
        )

    def estimate(self, theta=0.0, zero_counts=None) -> dict:
        """Zero totals, hot-set sizes, flow count, psi and denom in one device pass."""
        self._hand_in(zero_counts)
        info = _cabi.RestoreInfo()
        _cabi.check(self._lib.dhsa_estimate(self._h, float(theta), C.byref(info)))
        self.last_info = self._info_dict(info)
        return self.last_info

    def estimate_flow_count(self, zero_counts=None) -> Estimate:
        d = self.estimate(zero_counts=zero_counts)
        return Estimate(d["flow_count"], d["flow_saturated"])

    def bit_set_probability(self, flow_count: float) -> float:
        """psi = 1 - exp(-w / (g 2^k)) (pkg/src/dhsa/dhla.py:130-134)."""
        if flow_count < 0:
            raise ValueError("flow count must be nonnegative")
        return 1.0 - math.exp(-flow_count / (self.params.g * self.params.index_count))

    def shared_zero_counts(self, hosts) -> np.ndarray:
        hosts = np.ascontiguousarray(hosts, dtype=np.uint64)
        out = np.empty(len(hosts), dtype=np.int64)
        _cabi.check(self._lib.dhsa_shared_zero_counts(self._h, hosts.ctypes.data, len(hosts),
                                                      out.ctypes.data))
        return out

    def corrected_cardinality(self, host: int, psi: float) -> Estimate:
        """One host's sharing-corrected estimate (pkg/src/dhsa/dhla.py:145-160)."""
        g = self.params.g
        sz = int(self.shared_zero_counts(np.asarray([host], dtype=np.uint64))[0])
        denom = g * (1.0 - psi ** self.params.r)
        saturated = sz == 0
        if saturated:
            sz = 1
        if sz >= denom:
            return Estimate(0.0, saturated)
        return Estimate(-g * math.log(sz / denom), saturated)

    def _candidate_hosts(self, theta, max_candidates: int = DEFAULT_MAX_CANDIDATES,
                         workers: int = 1, zero_counts=None) -> np.ndarray:
        """Distinct, forward-verified keys, ascending (pkg/src/dhsa/dhla.py:198-217)."""
        info = _cabi.RestoreInfo()
        cap = 4096
        while True:
            self._hand_in(zero_counts)
            out = np.empty(cap, dtype=np.uint64)
            rc = self._lib.dhsa_candidate_hosts(self._h, float(theta), int(max_candidates),
                                                out.ctypes.data, cap, C.byref(info))
            self.last_info = self._info_dict(info)
            if rc == 3 and info.n_candidates > cap:
                cap = int(info.n_candidates)
                continue
            _cabi.check(rc)
            return out[: int(info.n_candidates)].copy()

    def restore_superpoints(self, theta, max_candidates: int = DEFAULT_MAX_CANDIDATES,
                            workers: int = 1) -> list:
        """Every host whose corrected estimate reaches theta, sorted by
        (-estimate, host) (pkg/src/dhsa/dhla.py:164-196).  `workers` is accepted
        and ignored: the device chain has no host threads to size."""
        info = _cabi.RestoreInfo()
        cap = 1024
        while True:
            rows = np.empty(cap, dtype=_REPORT_DTYPE)
            rc = self._lib.dhsa_restore(self._h, float(theta), int(max_candidates),
                                        rows.ctypes.data, cap, C.byref(info))
            self.last_info = self._info_dict(info)
            if rc == 3 and info.n_reports > cap:
                cap = int(info.n_reports)
                continue
            _cabi.check(rc)
            n = int(info.n_reports)
            return [SuperPointReport(int(h), float(e), bool(s))
                    for h, e, s in zip(rows["host"][:n].tolist(), rows["estimate"][:n].tolist(),
                                       rows["saturated"][:n].tolist())]

    def restore_superpoints_begin(self, theta, max_candidates: int = DEFAULT_MAX_CANDIDATES) -> None:
        """Enqueue the read-out of restore_superpoints and return at once.  The next window's
        reset() and update_batch() may be queued on this sketch before the reports are
        collected with restore_superpoints_end(): stream order keeps them behind the read-out,
        and the device never waits for the host."""
        _cabi.check(self._lib.dhsa_restore_begin(self._h, float(theta), int(max_candidates)))

    def restore_superpoints_end(self) -> list:
        """Reports of the read-out begun with restore_superpoints_begin."""
        info = _cabi.RestoreInfo()
        cap = 1024
        while True:
            rows = np.empty(cap, dtype=_REPORT_DTYPE)
            rc = self._lib.dhsa_restore_end(self._h, rows.ctypes.data, cap, C.byref(info))
            self.last_info = self._info_dict(info)
            if rc == 3 and info.n_reports > cap:
                cap = int(info.n_reports)
                continue
            _cabi.check(rc)
            n = int(info.n_reports)
            return [SuperPointReport(int(h), float(e), bool(s))
                    for h, e, s in zip(rows["host"][:n].tolist(), rows["estimate"][:n].tolist(),
                                       rows["saturated"][:n].tolist())]

    # --- the hash group, inverse (row 8a-10) ----------------------------------------------

    def reconstruct_key(self, indices) -> Optional[int]:
        """dhg.reconstruct_key for this sketch's parameters (pkg/src/dhsa/dhg.py:161-185)."""
        from . import dhg
        return dhg.reconstruct_key(self.params, indices, device=self.device)

    def reconstruct_many(self, tuples):
        """dhg.reconstruct_many for this sketch's parameters (pkg/src/dhsa/dhg.py:213-233)."""
        from . import dhg
        return dhg.reconstruct_many(self.params, tuples, device=self.device)

    # --- merge -------------------------------------------------------------------------

    def merge_from(self, other: "Dhla") -> None:
        """self |= other, on the device (peer access when the devices differ)."""
        if not _same_params(self.params, other.params):
            raise ConfigError(
                f"cannot merge sketches with different parameters: {self.params} vs {other.params}"
            )
        _cabi.check(self._lib.dhsa_or_merge(self._h, other._h))


def release_cached() -> None:
    """Free what destroyed sketches left parked for reuse (bit arrays, workspaces, page-locked slots).  The
    reference builds a new Dhla per window (pkg/src/dhsa/engine.py:63); the library recycles them instead of paying
    tens of milliseconds of allocation per window.  Call this to hand the memory back."""
    _cabi.check(_cabi.lib().dhsa_release_cached())


def merge(a: Dhla, b: Dhla) -> Dhla:
    """Union of two sketches with identical parameters (pkg/src/dhsa/dhla.py:305-318)."""
    if not _same_params(a.params, b.params):
        raise ConfigError(
            f"cannot merge sketches with different parameters: {a.params} vs {b.params}"
        )
    out = Dhla(a.params, window_id=a.window_id, device=a.device)
    out.merge_from(a)
    out.merge_from(b)
    return out
