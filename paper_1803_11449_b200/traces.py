"""Synthetic windows with ground truth, generated on the device (evaluation tooling).

Mirror of the reference's generator (/root/reference/pkg/src/dhsa/ingest.py:64-153): the
same ``GeneratorConfig`` fields and validation, the same population shape -- distinct
uniform hosts; background cardinalities from a truncated zipf, planted super points uniform
in ``super_cardinality``; every host's destinations a ramp from a random base, so distinct
by construction; ``duplicate_factor`` repeats of every pair; a shuffled, time-ordered
stream; truth = host -> exact distinct-destination count.

What differs is the random source: the reference draws from numpy's PCG64 stream, which a
GPU cannot replay, so this generator is defined over counters (splitmix64 of seed + index)
and a Feistel permutation of the output positions.  The small per-host part (at most a few
million hosts) is numpy on the host; the per-record part -- gigabytes at BASELINE config 3
-- is the CUDA kernel ``k_generate_trace``, and each rank of a multi-GPU window generates
only its own slice of positions.  tests/ checks every byte against the oracle's numpy
restatement of the same definition and the statistics against the reference's semantics.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from . import _cabi
from .dhg import mix64
from .engine import TRACE_DTYPE
from .errors import ConfigError

_M64 = (1 << 64) - 1
_TAG_HOST = 0x1F83D9ABFB41BD6B
_TAG_CARD = 0x5BE0CD19137E2179
_TAG_BASE = 0xCBBB9D5DC1059ED8
_TAG_PERM = 0x629A292A367CD507


@dataclass(frozen=True)
class GeneratorConfig:
    """Shape of one synthetic window (ingest.py:64-106)."""

    background_hosts: int = 0
    background_max_cardinality: int = 256
    background_zipf: float = 1.5
    superpoints: int = 0
    super_cardinality: Tuple[int, int] = (2048, 8192)
    duplicate_factor: int = 1
    start_ts: int = 0
    window_seconds: int = 300

    def __post_init__(self):
        if self.background_hosts < 0 or self.superpoints < 0:
            raise ConfigError("host counts must be nonnegative")
        if not 1 <= self.background_max_cardinality < 2 ** 32:
            raise ConfigError("background_max_cardinality must be in [1, 2^32)")
        lo, hi = self.super_cardinality
        if not 1 <= lo <= hi < 2 ** 32:
            raise ConfigError(f"super_cardinality range invalid: [{lo}, {hi}]")
        if self.duplicate_factor < 1:
            raise ConfigError("duplicate_factor must be >= 1")
        if self.window_seconds < 1:
            raise ConfigError("window_seconds must be >= 1")
        if self.background_zipf <= 1.0:
            raise ConfigError("background_zipf must be > 1")
        if self.background_max_cardinality > 1 << 22:
            raise ConfigError("background_max_cardinality must be <= 2^22 for the device generator's CDF table")


def _mix64_many(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def _fmix32_many(x: np.ndarray) -> np.ndarray:
    """murmur3's 32-bit finaliser: a bijection, so distinct indices give distinct hosts."""
    x = x.astype(np.uint32, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint32(16)
        x *= np.uint32(0x85EBCA6B)
        x ^= x >> np.uint32(13)
        x *= np.uint32(0xC2B2AE35)
        x ^= x >> np.uint32(16)
    return x


def _zipf_thresholds(a: float, kmax: int) -> np.ndarray:
    """floor(2^53 * P(card <= k)) for k = 1 .. kmax-1 of min(zipf(a), kmax) (ingest.py:123-126)."""
    if kmax <= 1:
        return np.empty(0, dtype=np.uint64)
    big = 1_000_000
    j = np.arange(1, big + 1, dtype=np.float64)
    zeta = float(np.sum(j ** -a)) + (big + 0.5) ** (1.0 - a) / (a - 1.0)
    cdf = np.cumsum(np.arange(1, kmax, dtype=np.float64) ** -a) / zeta
    return np.floor(np.minimum(cdf, 1.0) * float(1 << 53)).astype(np.uint64)


def trace_population(cfg: GeneratorConfig, seed: int):
    """(hosts uint32, cards int64, bases uint32): the per-host half of the generator."""
    n_hosts = cfg.background_hosts + cfg.superpoints
    seed64 = seed & _M64
    idx = np.arange(n_hosts, dtype=np.uint64)
    host_key = mix64(seed64 ^ _TAG_HOST) & 0xFFFFFFFF
    hosts = _fmix32_many(idx.astype(np.uint32) ^ np.uint32(host_key))
    with np.errstate(over="ignore"):
        u = _mix64_many(idx + np.uint64(seed64 ^ _TAG_CARD))
        bases = (_mix64_many(idx + np.uint64(seed64 ^ _TAG_BASE)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    cards = np.empty(n_hosts, dtype=np.int64)
    b = cfg.background_hosts
    if b:
        thr = _zipf_thresholds(cfg.background_zipf, cfg.background_max_cardinality)
        cards[:b] = 1 + np.searchsorted(thr, u[:b] >> np.uint64(11), side="right")
    if cfg.superpoints:
        lo, hi = cfg.super_cardinality
        cards[b:] = lo + (u[b:] % np.uint64(hi - lo + 1)).astype(np.int64)
    return hosts, cards, bases


def generate_trace_device(cfg: GeneratorConfig, seed: int, device: Optional[int] = None, fmt: str = "records",
                          lo: int = 0, hi: Optional[int] = None) -> dict:
    """Generate output positions [lo, hi) of the window on the device.

    fmt: "records" (uint8 tensor of 12-byte IPPR records), "pairs" (int32 cand / opp tensors in
    host order) or "both".  Returns dict(records, cand, opp, truth, total, flows)."""
    import torch

    from .dhla import _default_device

    if fmt not in ("records", "pairs", "both"):
        raise ConfigError(f"fmt must be records, pairs or both (got {fmt!r})")
    dev_index = _default_device() if device is None else int(device)
    dev = torch.device("cuda", dev_index)
    hosts, cards, bases = trace_population(cfg, seed)
    truth = {int(h): int(c) for h, c in zip(hosts.tolist(), cards.tolist())}
    out = dict(records=None, cand=None, opp=None, truth=truth, total=0, flows=0)
    if len(hosts) == 0:
        return out
    prefix = np.zeros(len(hosts) + 1, dtype=np.uint64)
    np.cumsum(cards, out=prefix[1:])
    flows = int(prefix[-1])
    total = flows * cfg.duplicate_factor
    hi = total if hi is None else min(int(hi), total)
    out["total"], out["flows"] = total, flows
    n = max(0, hi - lo)
    hosts_d = torch.from_numpy(hosts.view(np.int32)).to(dev)
    prefix_d = torch.from_numpy(prefix.view(np.int64)).to(dev)
    bases_d = torch.from_numpy(bases.view(np.int32)).to(dev)
    rec = torch.empty(n * 12, dtype=torch.uint8, device=dev) if fmt in ("records", "both") else None
    cand = torch.empty(n, dtype=torch.int32, device=dev) if fmt in ("pairs", "both") else None
    opp = torch.empty(n, dtype=torch.int32, device=dev) if fmt in ("pairs", "both") else None
    ptr = lambda t: C.c_void_p(t.data_ptr() if t is not None and t.numel() else 0)
    _cabi.check(_cabi.lib().dhsa_generate_trace(
        dev_index, ptr(hosts_d), ptr(prefix_d), ptr(bases_d), len(hosts), flows, cfg.duplicate_factor,
        mix64((seed & _M64) ^ _TAG_PERM), cfg.start_ts, cfg.window_seconds, lo, hi, ptr(rec), ptr(cand), ptr(opp),
        C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    torch.cuda.current_stream(dev).synchronize()   # the population tensors above are temporaries
    out.update(records=rec, cand=cand, opp=opp)
    return out


def generate_trace(cfg: GeneratorConfig, seed: int, device: Optional[int] = None):
    """(records, truth) with the reference's signature (ingest.py:109-153): the window is
    generated on the device and copied back as a TRACE_DTYPE array."""
    got = generate_trace_device(cfg, seed, device=device, fmt="records")
    if got["records"] is None:
        return np.empty(0, dtype=TRACE_DTYPE), {}
    return got["records"].cpu().numpy().view(TRACE_DTYPE).copy(), got["truth"]
