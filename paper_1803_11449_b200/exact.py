"""Exact ground truth and accuracy metrics on the device (evaluation tooling).

``exact_oracle`` is the reference's brute-force counter
(/root/reference/pkg/src/dhsa/ingest.py:159-176) -- exact distinct-opposite count per
candidate host -- built as a hash set of whole pairs in HBM (csrc ``k_exact_insert``), so a
10^8..10^9-packet window can be scored in milliseconds instead of the minutes numpy's
sort/unique takes.  ``evaluate`` mirrors ``ingest.evaluate`` (ingest.py:179-233); it is a few
set operations on the report list and stays on the host.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np

from . import _cabi
from .engine import DIRECTIONS, RECORD_BYTES, _as_record_bytes
from .errors import CapacityError, ConfigError


class ExactCounter:
    """Accumulates pairs on one device; ``result`` returns exact per-host distinct counts."""

    def __init__(self, expected_pairs: int = 1 << 22, device: Optional[int] = None):
        from .dhla import _default_device

        self.device = _default_device() if device is None else int(device)
        self.expected_pairs = int(expected_pairs)
        self._lib = _cabi.lib()
        self._h = C.c_void_p()
        _cabi.check(self._lib.dhsa_exact_create(self.device, self.expected_pairs, C.byref(self._h)))

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h:
            try:
                self._lib.dhsa_exact_destroy(h)
            except Exception:
                pass

    def _stream(self) -> int:
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def add_pairs(self, cand, opp) -> None:
        """torch CUDA tensors of 32-bit integers (any length; padded internally to 4)."""
        import torch

        if cand.numel() != opp.numel():
            raise ValueError("candidate and opposite arrays differ in length")
        n = cand.numel()
        if n == 0:
            return
        if n % 4 or cand.data_ptr() % 16 or opp.data_ptr() % 16 or not cand.is_contiguous() or not opp.is_contiguous():
            pad = (-n) % 4  # repeat the last pair: duplicates do not change a distinct count
            cand = torch.cat([cand.reshape(-1), cand.reshape(-1)[-1:].expand(pad)]).contiguous()
            opp = torch.cat([opp.reshape(-1), opp.reshape(-1)[-1:].expand(pad)]).contiguous()
            n += pad
        _cabi.check(self._lib.dhsa_exact_add_pairs(self._h, C.c_void_p(cand.data_ptr()), C.c_void_p(opp.data_ptr()),
                                                   n, C.c_void_p(self._stream())))

    def add_records(self, raw_dev, direction: str = "src", window_seconds: int = 0, window_id: int = 0,
                    lo: int = 0, hi: Optional[int] = None) -> None:
        """Raw 12-byte records on the device (uint8 tensor).  window_seconds 0 = whole trace."""
        import torch

        if direction not in DIRECTIONS:
            raise ConfigError(f"direction must be src, dst, or both (got {direction!r})")
        flat = raw_dev.reshape(-1)
        n = flat.numel() // RECORD_BYTES
        hi = n if hi is None else hi
        if n % 4 or flat.data_ptr() % 16:
            pad = (-n) % 4
            flat = torch.cat([flat, flat.new_zeros(pad * RECORD_BYTES)]).contiguous()
        _cabi.check(self._lib.dhsa_exact_add_records(
            self._h, C.c_void_p(flat.data_ptr()), flat.numel() // RECORD_BYTES, lo, hi, window_seconds, window_id,
            DIRECTIONS.index(direction), C.c_void_p(self._stream())))
        torch.cuda.current_stream(self.device).synchronize()  # `flat` may be a temporary

    def result(self, min_count: int = 1):
        """(hosts uint64 ascending, counts uint64, distinct pairs, distinct hosts)."""
        n, pairs, hosts_n = C.c_uint64(), C.c_uint64(), C.c_uint64()
        cap = 1 << 16
        while True:
            hosts = np.empty(cap, dtype=np.uint64)
            counts = np.empty(cap, dtype=np.uint64)
            rc = self._lib.dhsa_exact_result(self._h, int(min_count), hosts.ctypes.data, counts.ctypes.data, cap,
                                             C.byref(n), C.byref(pairs), C.byref(hosts_n), C.c_void_p(self._stream()))
            if rc == 3 and n.value > cap:
                cap = int(n.value)
                continue
            _cabi.check(rc)
            k = int(n.value)
            return hosts[:k].copy(), counts[:k].copy(), int(pairs.value), int(hosts_n.value)


def exact_oracle(records, direction: str = "src", device: Optional[int] = None, min_count: int = 1) -> Dict[int, int]:
    """Exact distinct-opposite count per candidate host (ingest.py:159-176).

    ``records``: TRACE_DTYPE array, raw record bytes, or a uint8 torch CUDA tensor of raw records."""
    import torch

    if direction not in DIRECTIONS:
        raise ConfigError(f"direction must be src, dst, or both (got {direction!r})")
    if hasattr(records, "is_cuda") and records.is_cuda:
        raw = records.reshape(-1)
        dev_index = raw.device.index
    else:
        host = _as_record_bytes(records)
        if host.size == 0:
            return {}
        from .dhla import _default_device

        dev_index = _default_device() if device is None else int(device)
        raw = torch.from_numpy(np.array(host, copy=True)).to(f"cuda:{dev_index}")
    n = raw.numel() // RECORD_BYTES
    if n == 0:
        return {}
    # plan for every record being a distinct pair (a trace without repeats), up to 2^27 pairs = a 4 GiB
    # table; a window with more distinct pairs than that grows by rebuilding
    expected = min(max(1 << 16, n * (2 if direction == "both" else 1)), 1 << 27)
    while True:
        counter = ExactCounter(expected, device=dev_index)
        counter.add_records(raw, direction)
        try:
            hosts, counts, _, _ = counter.result(min_count)
        except CapacityError:
            expected *= 4       # more distinct pairs than planned for: rebuild larger
            continue
        return {int(h): int(c) for h, c in zip(hosts.tolist(), counts.tolist())}


# Scoring.  The metric definitions and the record's field / key names are the reference's
# (pkg/src/dhsa/ingest.py:179-233: false reports and misses are both taken over the number of TRUE
# super points, rates are None -- undefined, not zero -- when there is none); this is host-side
# bookkeeping over a few hundred hosts, outside the hot path.
_METRIC_KEYS = (("n_true", "N"), ("n_reported", "N_reported"), ("n_false_pos", "N_false_pos"),
                ("n_false_neg", "N_false_neg"), ("fpr", "fpr"), ("fnr", "fnr"), ("tfr", "tfr"),
                ("mean_rel_err", "mean_rel_err"))


@dataclass
class EvalMetrics:
    n_true: int
    n_reported: int
    n_false_pos: int
    n_false_neg: int
    fpr: Optional[float]
    fnr: Optional[float]
    tfr: Optional[float]
    mean_rel_err: Optional[float]

    def as_dict(self) -> dict:
        return {key: getattr(self, field) for field, key in _METRIC_KEYS}


def evaluate(reports: Sequence, truth: Dict[int, int], theta: int) -> EvalMetrics:
    """Score a report list against exact per-host distinct-opposite counts."""
    supers = {host: count for host, count in truth.items() if count >= theta}
    hits, errors = set(), []
    false_pos = set()
    for rep in reports:
        exact = supers.get(rep.host)
        if exact is None:
            false_pos.add(rep.host)
        else:
            hits.add(rep.host)
            errors.append(abs(rep.estimate - exact) / exact)
    missed = len(supers) - len(hits)
    mean_err = sum(errors) / len(errors) if errors else None
    n_reported = len(hits) + len(false_pos)
    if not supers:
        return EvalMetrics(0, n_reported, len(false_pos), 0, None, None, None, mean_err)
    fpr, fnr = len(false_pos) / len(supers), missed / len(supers)
    return EvalMetrics(len(supers), n_reported, len(false_pos), missed, fpr, fnr, fpr + fnr, mean_err)
