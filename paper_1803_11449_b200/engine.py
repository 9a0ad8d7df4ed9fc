"""Windowed detection over a timestamped record stream, on the device.

Host-side mirror of the reference's window engine
(/root/reference/pkg/src/dhsa/engine.py:27-194): same ``WindowConfig`` fields and
validation, ``WindowSession.feed_batch / seal / restore`` with the same
``SealedWindowError`` rules, ``DetectionEngine.run`` returning one
``WindowResult(window_id, reports, pairs, dropped)`` per tumbling window, and
``split_pairs``.  What the reference does per record on the host with numpy --
``ts // window_seconds``, the running-maximum arrival window, the late-record
drop, the direction policy, the byte swap of network-order addresses
(engine.py:140-158, 179-194; record layout ingest.py:20) -- runs on the GPU
instead: ``dhsa_plan_windows`` finds the window segments of a chunk and
``dhsa_update_records_device`` scans raw 12-byte records with the decode fused
into the scan kernel, so a record is read from HBM once and never materialised
as (cand, opp) arrays.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Iterable, Iterator, List, Optional

import numpy as np

from . import _cabi
from .dhg import DhgParams
from .dhla import DEFAULT_MAX_CANDIDATES, Dhla, SuperPointReport
from .errors import ConfigError, SealedWindowError

DEFAULT_BATCH_PAIRS = 65536  # engine.py:22 (accepted for compatibility; the device needs no batching)
DIRECTIONS = ("src", "dst", "both")
TRACE_DTYPE = np.dtype([("ts", "<u4"), ("src", ">u4"), ("dst", ">u4")])  # ingest.py:20
RECORD_BYTES = 12
DEFAULT_CHUNK_RECORDS = 1 << 24  # records staged per host->device copy (192 MiB)

_BOUNDARY_DTYPE = np.dtype([("position", "<u8"), ("window_id", "<i8")])


@dataclass(frozen=True)
class WindowConfig:
    """Everything one detection window needs (engine.py:27-46)."""

    dhg: DhgParams = field(default_factory=DhgParams)
    window_seconds: int = 300
    theta: int = 1024
    workers: int = 1
    batch_pairs: int = DEFAULT_BATCH_PAIRS
    direction: str = "src"
    max_candidates: int = DEFAULT_MAX_CANDIDATES

    def __post_init__(self):
        for name in ("window_seconds", "theta", "workers", "batch_pairs", "max_candidates"):
            if getattr(self, name) <= 0:
                raise ConfigError(f"{name} must be positive (got {getattr(self, name)})")
        if self.direction not in DIRECTIONS:
            raise ConfigError(
                f"direction must be one of {DIRECTIONS} (got {self.direction!r})"
            )


@dataclass
class WindowResult:  # engine.py:49-54
    window_id: int
    reports: List[SuperPointReport]
    pairs: int
    dropped: int


def split_pairs(records: np.ndarray, direction: str):
    """(candidate, opposite) host arrays of a record batch (engine.py:179-194).

    Only for callers that want the arrays; the engine itself never builds them."""
    src = records["src"].astype(np.uint32)
    dst = records["dst"].astype(np.uint32)
    if direction == "src":
        return src, dst
    if direction == "dst":
        return dst, src
    if direction == "both":
        return np.concatenate([src, dst]), np.concatenate([dst, src])
    raise ConfigError(f"direction must be one of {DIRECTIONS} (got {direction!r})")


class WindowSession:
    """One open window: accepts batches until sealed, then restores (engine.py:57-103)."""

    def __init__(self, cfg: WindowConfig, window_id: int = 0, backend: str = "auto", pool=None,
                 device: Optional[int] = None, sketch: Optional[Dhla] = None):
        self.cfg = cfg
        self.sketch = sketch if sketch is not None else Dhla(cfg.dhg, backend=backend, window_id=window_id,
                                                             device=device)
        self.sealed = False
        self.pairs = 0
        self.dropped = 0
        self._pool = pool  # accepted and unused: launches are asynchronous already
        self._lib = _cabi.lib()

    def _check_open(self):
        if self.sealed:
            raise SealedWindowError(
                f"window {self.sketch.window_id} is sealed; no further updates accepted"
            )

    def feed_batch(self, candidates, opposites) -> None:
        self._check_open()
        if len(candidates) != len(opposites):
            raise ValueError("candidate and opposite arrays differ in length")
        self.sketch.update_batch(candidates, opposites)
        self.pairs += len(candidates)

    def feed_records(self, records_dev_ptr: int, n_in_buffer: int, lo: int, hi: int) -> None:
        """Scan raw records [lo, hi) of a device buffer into this window; late records are
        dropped and counted on the device (read back by ``seal``)."""
        self._check_open()
        _cabi.check(self._lib.dhsa_update_records_device(
            self.sketch._h, C.c_void_p(records_dev_ptr), n_in_buffer, lo, hi,
            self.cfg.window_seconds, self.sketch.window_id, DIRECTIONS.index(self.cfg.direction)))
        self._fed_records = True

    def seal(self) -> None:
        """Barrier: every update issued so far is in the bits; the window freezes."""
        self.sketch.seal()
        if getattr(self, "_fed_records", False):
            fed, late = C.c_uint64(), C.c_uint64()
            _cabi.check(self._lib.dhsa_record_tally(self.sketch._h, C.byref(fed), C.byref(late)))
            self.pairs += int(fed.value)
            self.dropped += int(late.value)
            self._fed_records = False
        self.sealed = True

    def restore(self) -> List[SuperPointReport]:
        if not self.sealed:
            raise SealedWindowError("window must be sealed before restoration")
        return self.sketch.restore_superpoints(
            self.cfg.theta, max_candidates=self.cfg.max_candidates, workers=self.cfg.workers
        )

    def seal_and_restore_begin(self) -> None:
        """seal() + restore() without stopping the device: the window freezes, its read-out is
        queued behind its last update, and the caller goes on feeding the next window (another
        sketch, same stream) before collecting with ``restore_end``."""
        self._check_open()
        self.sealed = True
        self.sketch.restore_superpoints_begin(self.cfg.theta, max_candidates=self.cfg.max_candidates)

    def restore_end(self) -> List[SuperPointReport]:
        reports = self.sketch.restore_superpoints_end()
        if getattr(self, "_fed_records", False):   # the tally came back with the reports
            fed, late = C.c_uint64(), C.c_uint64()
            _cabi.check(self._lib.dhsa_record_tally_at_restore(self.sketch._h, C.byref(fed), C.byref(late)))
            self.pairs += int(fed.value)
            self.dropped += int(late.value)
            self._fed_records = False
        return reports


def _as_record_bytes(records) -> np.ndarray:
    """Flat uint8 view of host records in the IPPR layout."""
    if isinstance(records, (bytes, bytearray, memoryview)):
        arr = np.frombuffer(records, dtype=np.uint8)
    else:
        if not isinstance(records, np.ndarray):
            records = np.array(list(records), dtype=TRACE_DTYPE)
        if records.dtype != TRACE_DTYPE:
            if records.dtype == np.uint8:
                arr = np.ascontiguousarray(records).reshape(-1)
                if arr.size % RECORD_BYTES:
                    raise ValueError(f"raw record buffer is {arr.size} bytes, not a multiple of {RECORD_BYTES}")
                return arr
            records = records.astype(TRACE_DTYPE)
        arr = np.ascontiguousarray(records).view(np.uint8).reshape(-1)
    if arr.size % RECORD_BYTES:
        raise ValueError(f"raw record buffer is {arr.size} bytes, not a multiple of {RECORD_BYTES}")
    return arr


class DetectionEngine:
    """Runs the window lifecycle over a timestamped record stream (engine.py:106-176)."""

    def __init__(self, cfg: WindowConfig, backend: str = "auto", device: Optional[int] = None,
                 chunk_records: int = DEFAULT_CHUNK_RECORDS):
        self.cfg = cfg
        self.backend = backend
        self.device = device
        self.chunk_records = max(4, (int(chunk_records) + 3) & ~3)
        self._idle: List[Dhla] = []   # sketches nobody else holds any more, reset for reuse
        self._planner: Optional[Dhla] = None

    def run(self, records, on_sealed: Optional[Callable[[Dhla], None]] = None) -> List[WindowResult]:
        """Detect super points per tumbling window.

        ``records``: a structured array with ts/src/dst fields (TRACE_DTYPE), raw IPPR
        record bytes (host), an iterable of (ts, src, dst) tuples, or a 1-D uint8 torch
        CUDA tensor of raw records already on the device.  Records older than the window
        being filled are dropped and counted; ``on_sealed`` sees each sealed sketch before
        its result is emitted."""
        return list(self._run(records, on_sealed))

    # -- chunk sources -------------------------------------------------------------------

    def _device_chunks(self, records):
        """Yield (device uint8 tensor, n_records) chunks; host input is double-buffered so
        the copy of chunk i+1 overlaps the scan of chunk i."""
        import torch

        if hasattr(records, "is_cuda") and records.is_cuda:
            flat = records.reshape(-1)
            if flat.dtype != torch.uint8 or flat.numel() % RECORD_BYTES:
                raise ValueError("device records must be a uint8 tensor of whole 12-byte records")
            n = flat.numel() // RECORD_BYTES
            # already on the device: nothing to stage, so plan and scan it whole (chunk_records only
            # bounds staging buffers); a caller-chosen smaller chunk is still honoured for tests
            step = max(self.chunk_records, n) if self.chunk_records >= DEFAULT_CHUNK_RECORDS else self.chunk_records
            for lo in range(0, n, step):
                hi = min(n, lo + step)
                yield flat[lo * RECORD_BYTES: hi * RECORD_BYTES], hi - lo
            return
        host = _as_record_bytes(records)
        n = host.size // RECORD_BYTES
        if n == 0:
            return
        dev_index = self._device_index()
        dev = torch.device("cuda", dev_index)
        step = min(self.chunk_records, (n + 3) & ~3)
        bufs = [torch.empty(step * RECORD_BYTES, dtype=torch.uint8, device=dev) for _ in range(2 if n > step else 1)]
        copy_stream = torch.cuda.Stream(dev)
        ready = [torch.cuda.Event() for _ in bufs]
        consumed = [torch.cuda.Event() for _ in bufs]
        lib = _cabi.lib()
        base = host.ctypes.data

        def start_copy(c):
            lo = c * step
            hi = min(n, lo + step)
            b = c % len(bufs)
            copy_stream.wait_event(consumed[b])      # the scans of the chunk that used this buffer are done
            _cabi.check(lib.dhsa_copy_to_device_async(
                dev_index, C.c_void_p(bufs[b].data_ptr()), C.c_void_p(base + lo * RECORD_BYTES),
                (hi - lo) * RECORD_BYTES, C.c_void_p(copy_stream.cuda_stream)))
            ready[b].record(copy_stream)
            return hi - lo

        n_chunks = (n + step - 1) // step
        counts = {0: start_copy(0)}
        for c in range(n_chunks):
            if c + 1 < n_chunks:
                counts[c + 1] = start_copy(c + 1)
            b = c % len(bufs)
            torch.cuda.current_stream(dev).wait_event(ready[b])
            yield bufs[b][: counts[c] * RECORD_BYTES], counts[c]
            consumed[b].record(torch.cuda.current_stream(dev))

    def _device_index(self) -> int:
        if self.device is not None:
            return int(self.device)
        from .dhla import _default_device

        return _default_device()

    # -- the window lifecycle ------------------------------------------------------------------

    def _run(self, records, on_sealed) -> Iterator[WindowResult]:
        cfg = self.cfg
        lib = _cabi.lib()
        session: Optional[WindowSession] = None
        cap = 4096
        bounds = np.empty(cap, dtype=_BOUNDARY_DTYPE)
        for chunk, n in self._device_chunks(records):
            import torch

            if self._planner is None:  # a 768-byte sketch whose handle runs the plan kernels; kept across runs
                self._planner = Dhla(DhgParams(r=3, g=8, k=8, alpha=8, key_width=16), device=self._device_index())
            planner = self._planner
            planner.use_stream(torch.cuda.current_stream(planner.device))   # the sketch keeps the stream object alive
            ptr = chunk.data_ptr()
            open_window = session.sketch.window_id if session is not None else -1
            n_b = C.c_uint32()
            while True:
                rc = lib.dhsa_plan_windows(planner._h, C.c_void_p(ptr), n, cfg.window_seconds, open_window,
                                           C.c_void_p(bounds.ctypes.data), cap, C.byref(n_b))
                if rc == 3 and cap < (1 << 26):   # more windows than planned for: grow and retry
                    cap *= 16
                    bounds = np.empty(cap, dtype=_BOUNDARY_DTYPE)
                    continue
                _cabi.check(rc)
                break
            cuts = [(int(b["position"]), int(b["window_id"])) for b in bounds[: n_b.value]]
            # segments of this chunk: [start, next start) belongs to window wid
            segments = []
            if session is not None and (not cuts or cuts[0][0] > 0):
                segments.append((0, open_window))
            segments.extend(cuts)
            for idx, (lo, wid) in enumerate(segments):
                hi = segments[idx + 1][0] if idx + 1 < len(segments) else n
                closing = None
                if session is not None and wid > session.sketch.window_id:
                    if on_sealed is not None:          # the hook wants the sealed sketch now: no overlap
                        yield self._finish(session, on_sealed)
                    else:                              # queue its read-out, collect after the next feed
                        session.seal_and_restore_begin()
                        closing = session
                    session = None
                if session is None:
                    session = WindowSession(cfg, wid, self.backend, device=self._device_index(),
                                            sketch=self._take_idle(wid))
                    session.sketch.use_stream(torch.cuda.current_stream(session.sketch.device))
                session.feed_records(ptr, n, lo, hi)
                if closing is not None:
                    yield self._collect(closing)
        if session is not None:
            yield self._finish(session, on_sealed)

    def _take_idle(self, window_id: int) -> Optional[Dhla]:
        if not self._idle:
            return None
        sk = self._idle.pop()
        sk.reset(window_id=window_id)
        return sk

    def _finish(self, session: WindowSession, on_sealed) -> WindowResult:
        if on_sealed is None:
            session.seal_and_restore_begin()
            return self._collect(session)
        session.seal()
        on_sealed(session.sketch)
        return self._collect(session, session.restore(), recycle=False)   # the hook may have kept the sketch

    def _collect(self, session: WindowSession, reports=None, recycle: bool = True) -> WindowResult:
        if reports is None:
            reports = session.restore_end()
        result = WindowResult(
            window_id=session.sketch.window_id,
            reports=reports,
            pairs=session.pairs,
            dropped=session.dropped,
        )
        # Every window owns its sketch, as in the reference.  Allocating one costs milliseconds
        # (cudaMalloc of the bits and the flow cache), so a sketch that never left the engine -- no
        # on_sealed hook saw it -- goes back to the idle list instead of being freed.
        sk, session.sketch = session.sketch, None
        if recycle and len(self._idle) < 2:
            self._idle.append(sk)
        return result
