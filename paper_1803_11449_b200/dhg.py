"""Hash-group parameters: the host-side record the kernels are launched with.

Mirrors the reference's ``DhgParams`` (/root/reference/pkg/src/dhsa/dhg.py:59-123):
same field names, defaults, validation rules and messages, so a ``dhsa.DhgParams``
and this class are interchangeable at the sketch constructor.  The hashing
itself runs on the device (csrc/dhsa_device.cuh); only the two seed -> state
derivations and the scalar helpers a caller may want for a single key live
here, as plain integer arithmetic.  The array forms -- ``forward_many`` and the
inverse ``reconstruct_key`` / ``reconstruct_many`` (dhg.py:161-233) -- are calls
into libdhsa_b200.so like everything else on the path.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .errors import ConfigError

_MASK64 = (1 << 64) - 1

# domain-separation tags, dhg.py:29-30; default seeds, dhg.py:32-33
_DH0_TAG = 0x9E3779B97F4A7C15
_H1_TAG = 0xD1B54A32D192ED03
DEFAULT_SEED_DH0 = 0x243F6A8885A308D3
DEFAULT_SEED_H1 = 0x13198A2E03707344


def mix64(x: int) -> int:
    """splitmix64 finaliser (dhg.py:36-44); the device twin is dhsa::mix64."""
    x &= _MASK64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _MASK64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _MASK64
    x ^= x >> 31
    return x


@dataclass(frozen=True)
class DhgParams:
    """r arrays of 2^k estimators of g bits; blocks of k bits every alpha bits."""

    r: int = 5
    g: int = 1024
    k: int = 14
    alpha: int = 6
    key_width: int = 32
    seed_dh0: int = DEFAULT_SEED_DH0
    seed_h1: int = DEFAULT_SEED_H1

    def __post_init__(self):
        r, g, k, a, w = self.r, self.g, self.k, self.alpha, self.key_width
        if r < 3:
            raise ConfigError(f"r must satisfy r >= 3 (got r={r})")
        if r > 64:
            raise ConfigError(f"r must satisfy r <= 64 on the device path (got r={r})")
        if g < 8 or g & (g - 1):
            raise ConfigError(
                f"g must be a power of two >= 8 for byte-packed estimators (got g={g})"
            )
        if g > 1 << 30:
            raise ConfigError(f"g must satisfy g <= 2^30 on the device path (got g={g})")
        if not 1 <= k <= 30:
            raise ConfigError(f"k must satisfy 1 <= k <= 30 (got k={k})")
        if not 8 <= w <= 32:
            raise ConfigError(f"key_width must satisfy 8 <= key_width <= 32 (got {w})")
        if k > w:
            raise ConfigError(f"k must satisfy k <= key_width (got k={k}, key_width={w})")
        if not 1 <= a <= k:
            raise ConfigError(f"alpha must satisfy 1 <= alpha <= k (got alpha={a}, k={k})")
        if (r - 2) * a + k < w:
            raise ConfigError(
                f"block coverage must satisfy (r-2)*alpha + k >= key_width "
                f"(got ({r}-2)*{a}+{k}={(r - 2) * a + k} < {w})"
            )
        if (r - 2) * a + k > 64:
            raise ConfigError(
                f"partial keys are staged in 64-bit words: (r-2)*alpha + k <= 64 "
                f"(got {(r - 2) * a + k})"
            )
        if not 0 <= self.seed_dh0 <= _MASK64 or not 0 <= self.seed_h1 <= _MASK64:
            raise ConfigError("seeds must be unsigned 64-bit integers")

    @property
    def index_count(self) -> int:
        return 1 << self.k

    @property
    def state_dh0(self) -> int:
        return mix64(self.seed_dh0 ^ _DH0_TAG)

    @property
    def state_h1(self) -> int:
        return mix64(self.seed_h1 ^ _H1_TAG)

    @property
    def sketch_bytes(self) -> int:
        return self.r * self.index_count * (self.g // 8)

    @classmethod
    def coerce(cls, p) -> "DhgParams":
        """Accept this class or any record with the same fields (e.g. dhsa.DhgParams)."""
        if isinstance(p, cls):
            return p
        return cls(r=p.r, g=p.g, k=p.k, alpha=p.alpha, key_width=p.key_width,
                   seed_dh0=p.seed_dh0, seed_h1=p.seed_h1)


# Scalar helpers for a single key (dhg.py:126-158).  Not on the data path.

def dh0(params: DhgParams, a: int) -> int:
    return mix64(params.state_dh0 ^ a) & (params.index_count - 1)


def h1(params: DhgParams, b: int) -> int:
    return mix64(params.state_h1 ^ b) & (params.g - 1)


def forward(params: DhgParams, a: int) -> tuple:
    d0 = dh0(params, a)
    kmask = params.index_count - 1
    return (d0,) + tuple(
        ((a >> ((i - 1) * params.alpha)) & kmask) ^ d0 for i in range(1, params.r)
    )


def dh_i(params: DhgParams, a: int, i: int) -> int:
    """Index of host ``a`` in array ``i``, 1 <= i <= r-1 (dhg.py:131-139)."""
    if not 1 <= i <= params.r - 1:
        raise ValueError(f"array index i must be in [1, {params.r - 1}], got {i}")
    return ((a >> ((i - 1) * params.alpha)) & (params.index_count - 1)) ^ dh0(params, a)


def recover_block(params: DhgParams, cl0: int, cli: int) -> int:
    """The key block an index carries under its XOR mask (dhg.py:146-148)."""
    return cl0 ^ cli


# Array forms: kernels behind the C ABI (dhsa_forward_many / dhsa_reconstruct_many).

def _cparams(params: DhgParams):
    from . import _cabi
    p = DhgParams.coerce(params)
    return _cabi, _cabi.Params(p.r, p.g, p.k, p.alpha, p.key_width, 0, p.state_dh0, p.state_h1)


def _device(device: Optional[int]) -> int:
    if device is not None:
        return int(device)
    env = os.environ.get("DHSA_DEVICE", os.environ.get("LOCAL_RANK"))
    return int(env) if env not in (None, "") else 0


def forward_many(params: DhgParams, keys, device: Optional[int] = None) -> np.ndarray:
    """Estimator indices of a batch of keys, shape (len(keys), r), uint64 (dhg.py:203-210)."""
    _cabi, cp = _cparams(params)
    k = np.ascontiguousarray(keys, dtype=np.uint64).reshape(-1)
    out = np.empty((len(k), cp.r), dtype=np.uint64)
    _cabi.check(_cabi.lib().dhsa_forward_many(C.byref(cp), _device(device), k.ctypes.data, len(k), out.ctypes.data))
    return out


def reconstruct_many(params: DhgParams, tuples, device: Optional[int] = None):
    """(keys, ok) of an (n, r) index matrix: rebuilt keys (garbage where not ok) and the boolean
    acceptance mask (dhg.py:213-233)."""
    _cabi, cp = _cparams(params)
    t = np.ascontiguousarray(tuples, dtype=np.uint64)
    if t.ndim != 2 or t.shape[1] != cp.r:
        raise ValueError(f"expected an (n, {cp.r}) index matrix, got shape {t.shape}")
    keys = np.empty(len(t), dtype=np.uint64)
    ok = np.empty(len(t), dtype=np.uint8)
    _cabi.check(_cabi.lib().dhsa_reconstruct_many(C.byref(cp), _device(device), t.ctypes.data, len(t),
                                                  keys.ctypes.data, ok.ctypes.data))
    return keys, ok.astype(bool)


def reconstruct_key(params: DhgParams, indices: Sequence[int], device: Optional[int] = None) -> Optional[int]:
    """The host key of one r-tuple of indices, or None if they are inconsistent (dhg.py:161-185)."""
    if len(indices) != params.r:
        raise ValueError(f"expected {params.r} indices, got {len(indices)}")
    keys, ok = reconstruct_many(params, np.asarray([list(indices)], dtype=np.uint64), device=device)
    return int(keys[0]) if ok[0] else None
