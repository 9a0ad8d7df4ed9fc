"""`.dhla` snapshots of device sketches, interchangeable with the reference's files.

The format is the reference's (/root/reference/pkg/src/dhsa/dhla.py:36-39,321-373): a 42-byte
little-endian header -- magic ``DHLA``, version, r, g, k, alpha, key_width, seed_dh0, seed_h1,
window_id -- followed by the bit array in the snapshot layout.  That layout is also the one the
sketch has in HBM, so the payload is never assembled on the host: it moves between the device and
the file object one chunk at a time through a single reusable buffer (``dhsa_download_range`` /
``dhsa_upload_range``), and a truncated or over-long file is noticed at the chunk where it
happens.  Parse errors carry the reference's messages and offsets (pkg/tests/test_dhla.py:369-391).
"""

from __future__ import annotations

import ctypes as C
import struct
from typing import BinaryIO, Optional, Union

from . import _cabi
from .dhg import DhgParams
from .dhla import Dhla
from .errors import ConfigError, DataError

CHUNK_BYTES = 1 << 20

# (field, struct code, offset): the header as a table; the offsets are the ones the messages quote
_FIELDS = (
    ("magic", "4s", 0), ("version", "H", 4),
    ("r", "H", 6), ("g", "I", 8), ("k", "H", 12), ("alpha", "H", 14), ("key_width", "H", 16),
    ("seed_dh0", "Q", 18), ("seed_h1", "Q", 26), ("window_id", "Q", 34),
)
HEADER_BYTES = 42
_MAGIC, _VERSION = b"DHLA", 1
assert struct.calcsize("<" + "".join(code for _, code, _ in _FIELDS)) == HEADER_BYTES


def _pack_header(sketch: Dhla) -> bytes:
    p = sketch.params
    values = dict(magic=_MAGIC, version=_VERSION, r=p.r, g=p.g, k=p.k, alpha=p.alpha, key_width=p.key_width,
                  seed_dh0=p.seed_dh0, seed_h1=p.seed_h1, window_id=sketch.window_id)
    raw = bytearray(HEADER_BYTES)
    for name, code, off in _FIELDS:
        struct.pack_into("<" + code, raw, off, values[name])
    return bytes(raw)


def _parse_header(raw: bytes) -> dict:
    if len(raw) < HEADER_BYTES:
        raise DataError(f"snapshot header truncated: got {len(raw)} bytes at offset 0, need {HEADER_BYTES}")
    head = {name: struct.unpack_from("<" + code, raw, off)[0] for name, code, off in _FIELDS}
    if head["magic"] != _MAGIC:
        raise DataError(f"bad snapshot magic {head['magic']!r} at offset 0")
    if head["version"] != _VERSION:
        raise DataError(f"unsupported snapshot version {head['version']} at offset 4")
    return head


def _open(target, mode):
    if isinstance(target, str):
        return open(target, mode), True
    return target, False


def write_snapshot(sketch: Dhla, dest: Union[str, BinaryIO]) -> None:
    fh, own = _open(dest, "wb")
    try:
        fh.write(_pack_header(sketch))
        lib, total = _cabi.lib(), sketch.params.sketch_bytes
        chunk = bytearray(min(CHUNK_BYTES, total))
        ptr = (C.c_uint8 * len(chunk)).from_buffer(chunk)
        view = memoryview(chunk)
        for lo in range(0, total, len(chunk)):      # device -> chunk -> file; the first call drains the stream
            n = min(len(chunk), total - lo)
            _cabi.check(lib.dhsa_download_range(sketch._h, lo, n, ptr))
            fh.write(view[:n])
    finally:
        if own:
            fh.close()


def _read_into(fh: BinaryIO, view: memoryview) -> int:
    """Fill `view` from a file object that may return short reads; bytes actually read."""
    got = 0
    while got < len(view):
        n = fh.readinto(view[got:]) if hasattr(fh, "readinto") else None
        if n is None:                               # no readinto: plain read
            data = fh.read(len(view) - got)
            n = len(data)
            view[got:got + n] = data
        if not n:
            break
        got += n
    return got


def read_snapshot(src: Union[str, BinaryIO], backend="auto", device: Optional[int] = None) -> Dhla:
    fh, own = _open(src, "rb")
    try:
        head = _parse_header(fh.read(HEADER_BYTES))
        try:
            params = DhgParams(**{f: head[f] for f in ("r", "g", "k", "alpha", "key_width", "seed_dh0", "seed_h1")})
        except ConfigError as exc:
            raise DataError(f"invalid parameters in snapshot header (offset 6): {exc}") from exc
        sketch = Dhla(params, backend=backend, window_id=head["window_id"], device=device)
        lib, total = _cabi.lib(), params.sketch_bytes
        chunk = bytearray(min(CHUNK_BYTES, total))
        ptr = (C.c_uint8 * len(chunk)).from_buffer(chunk)
        view = memoryview(chunk)
        for lo in range(0, total, len(chunk)):      # file -> chunk -> device
            want = min(len(chunk), total - lo)
            got = _read_into(fh, view[:want])
            if got < want:
                raise DataError(f"snapshot payload truncated at offset {HEADER_BYTES + lo + got}: "
                                f"expected {total} payload bytes")
            _cabi.check(lib.dhsa_upload_range(sketch._h, lo, want, ptr))
        if fh.read(1):
            raise DataError(f"trailing data after snapshot payload at offset {HEADER_BYTES + total}")
        return sketch
    finally:
        if own:
            fh.close()
