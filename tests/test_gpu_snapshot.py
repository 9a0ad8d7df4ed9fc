"""Row N2: .dhla snapshots of device sketches, byte-compatible with the reference's."""
import hashlib
import io

import numpy as np
import pytest

import paper_1803_11449_b200 as P
from oracle import oracle as O

from helpers import load_json

pytestmark = pytest.mark.gpu


def _filled():
    sk = P.Dhla(P.DhgParams())
    sk.update_batch(*O.distinct_pairs(50_000, 19))
    sk.window_id = 77
    return sk


def test_snapshot_file_is_byte_identical_to_the_references():
    case = load_json("snapshot_case.json")
    buf = io.BytesIO()
    P.write_snapshot(_filled(), buf)
    blob = buf.getvalue()
    assert len(blob) == case["size"] == 42 + 10_485_760        # pkg/tests/test_dhla.py:362-366
    assert blob[:42].hex() == case["header_hex"]
    assert hashlib.sha256(blob).hexdigest() == case["file_sha256"]


def test_snapshot_round_trip_and_merge_of_loaded_sketches(tmp_path):
    # pkg/tests/test_dhla.py:350-359 and the `dhsa merge` flow (cli.py:264-275)
    a = _filled()
    path = str(tmp_path / "a.dhla")
    P.write_snapshot(a, path)
    loaded = P.read_snapshot(path)
    assert loaded.params == a.params and loaded.window_id == 77
    assert np.array_equal(loaded.bits, a.bits)
    b = P.Dhla(P.DhgParams())
    b.update_batch(*O.plant_pairs(0xC63A1B02, 2048, 10))
    merged = P.merge(loaded, b)
    ora = O.OracleSketch()
    ora.update_batch(*O.distinct_pairs(50_000, 19))
    ora.update_batch(*O.plant_pairs(0xC63A1B02, 2048, 10))
    assert np.array_equal(merged.bits, ora.bits)
    assert [r.host for r in merged.restore_superpoints(1024)] == [0xC63A1B02]


def test_snapshot_parse_errors_match_the_reference(tmp_path):
    # pkg/tests/test_dhla.py:369-391
    path = tmp_path / "w.dhla"
    P.write_snapshot(P.Dhla(P.DhgParams()), str(path))
    raw = path.read_bytes()
    clipped = tmp_path / "clipped.dhla"
    clipped.write_bytes(raw[: len(raw) // 2])
    with pytest.raises(P.DataError, match="offset"):
        P.read_snapshot(str(clipped))
    bad = tmp_path / "bad.dhla"
    bad.write_bytes(b"NOPE" + b"\x00" * 64)
    with pytest.raises(P.DataError, match="magic"):
        P.read_snapshot(str(bad))
    path.write_bytes(raw + b"\x00")
    with pytest.raises(P.DataError, match="trailing"):
        P.read_snapshot(str(path))
    with pytest.raises(P.DataError, match="header truncated"):
        P.read_snapshot(io.BytesIO(raw[:10]))
    broken = bytearray(raw)
    broken[6] = 2   # r = 2: invalid parameters
    with pytest.raises(P.DataError, match="invalid parameters"):
        P.read_snapshot(io.BytesIO(bytes(broken)))
