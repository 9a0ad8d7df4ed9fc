"""`.dhla` snapshots of device sketches, byte-compatible with the reference's
(/root/reference/pkg/src/dhsa/dhla.py:321-373): a 42-byte little-endian header
``<4sHHIHHHQQQ`` (magic ``DHLA``, version, r, g, k, alpha, key_width, seed_dh0,
seed_h1, window_id) followed by the raw bit array in the snapshot layout, which is
also the layout the sketch has in HBM -- so writing is one device-to-host copy and
reading one host-to-device copy, and files are interchangeable with the reference's
in both directions.  Parse errors carry the same messages and offsets.
"""

from __future__ import annotations

import struct
from typing import BinaryIO, Optional, Union

import numpy as np

from .dhg import DhgParams
from .dhla import Dhla
from .errors import ConfigError, DataError

_SNAP_MAGIC = b"DHLA"
_SNAP_VERSION = 1
_SNAP_HEADER = struct.Struct("<4sHHIHHHQQQ")  # dhla.py:36-39


def write_snapshot(sketch: Dhla, dest: Union[str, BinaryIO]) -> None:
    p = sketch.params
    header = _SNAP_HEADER.pack(
        _SNAP_MAGIC, _SNAP_VERSION, p.r, p.g, p.k, p.alpha, p.key_width,
        p.seed_dh0, p.seed_h1, sketch.window_id,
    )
    payload = sketch.bits  # one D2H copy after the stream drains
    if isinstance(dest, str):
        with open(dest, "wb") as fh:
            fh.write(header)
            fh.write(payload.tobytes())
    else:
        dest.write(header)
        dest.write(payload.tobytes())


def read_snapshot(src: Union[str, BinaryIO], backend: str = "auto", device: Optional[int] = None) -> Dhla:
    if isinstance(src, str):
        with open(src, "rb") as fh:
            return read_snapshot(fh, backend, device)
    raw = src.read(_SNAP_HEADER.size)
    if len(raw) < _SNAP_HEADER.size:
        raise DataError(
            f"snapshot header truncated: got {len(raw)} bytes at offset 0, "
            f"need {_SNAP_HEADER.size}"
        )
    magic, version, r, g, k, alpha, key_width, seed_dh0, seed_h1, window_id = (
        _SNAP_HEADER.unpack(raw)
    )
    if magic != _SNAP_MAGIC:
        raise DataError(f"bad snapshot magic {magic!r} at offset 0")
    if version != _SNAP_VERSION:
        raise DataError(f"unsupported snapshot version {version} at offset 4")
    try:
        params = DhgParams(
            r=r, g=g, k=k, alpha=alpha, key_width=key_width,
            seed_dh0=seed_dh0, seed_h1=seed_h1,
        )
    except ConfigError as exc:
        raise DataError(f"invalid parameters in snapshot header (offset 6): {exc}") from exc
    payload = src.read(params.sketch_bytes + 1)
    if len(payload) < params.sketch_bytes:
        raise DataError(
            f"snapshot payload truncated at offset {_SNAP_HEADER.size + len(payload)}: "
            f"expected {params.sketch_bytes} payload bytes"
        )
    if len(payload) > params.sketch_bytes:
        raise DataError(
            f"trailing data after snapshot payload at offset "
            f"{_SNAP_HEADER.size + params.sketch_bytes}"
        )
    sketch = Dhla(params, backend=backend, window_id=window_id, device=device)
    sketch.load_bits(np.frombuffer(payload, dtype=np.uint8).reshape(
        params.r, params.index_count, params.g // 8))
    return sketch
