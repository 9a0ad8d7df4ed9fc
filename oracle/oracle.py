"""ctypes front end of the CPU oracle (oracle/dhsa_oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Import this only from tests/, from
``__graft_entry__.smoke()`` and from bench.py's cpu_baseline / ``--impl
reference`` legs.  ``paper_1803_11449_b200`` never imports it.

Parity status: PINNED -- see tests/test_oracle_golden.py (reference constants
and fixtures generated from the live reference by tests/golden/make_golden.py).

Two checkers live here:

* :class:`OracleSketch` -- the C restatement, a numpy ``bits`` array plus the
  read-out chain, shaped like the reference's ``dhsa.dhla.Dhla``
  (/root/reference/pkg/src/dhsa/dhla.py:57-196).
* :func:`load_ref_core` -- the reference's own compiled hot loops
  (``update_batch`` / ``zero_counts`` of pkg/src/dhsa/_core.pyx), built by
  ``make -C oracle ref`` into oracle/_ref/ when /root/reference is present.
"""

from __future__ import annotations

import ctypes as C
import glob
import importlib.machinery
import importlib.util
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdhsa_oracle.so")

DH0_TAG = 0x9E3779B97F4A7C15  # pkg/src/dhsa/dhg.py:29
H1_TAG = 0xD1B54A32D192ED03  # pkg/src/dhsa/dhg.py:30
DEFAULT_SEED_DH0 = 0x243F6A8885A308D3  # pkg/src/dhsa/dhg.py:32
DEFAULT_SEED_H1 = 0x13198A2E03707344  # pkg/src/dhsa/dhg.py:33


class _Params(C.Structure):
    _fields_ = [
        ("r", C.c_int32), ("g", C.c_int32), ("k", C.c_int32), ("alpha", C.c_int32),
        ("key_width", C.c_int32), ("pad_", C.c_int32),
        ("state_dh0", C.c_uint64), ("state_h1", C.c_uint64),
    ]


def build(force: bool = False) -> str:
    """Compile the C restatement (and oracle/_ref when the reference is here)."""
    src = os.path.join(_HERE, "dhsa_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-B", "libdhsa_oracle.so"], check=True,
                       stdout=subprocess.DEVNULL)
    if os.path.exists("/root/reference/pkg/src/dhsa/_core.pyx") and (force or not _ref_so()):
        subprocess.run(["make", "-C", _HERE, "ref"], check=False, stdout=subprocess.DEVNULL,
                       stderr=subprocess.DEVNULL)
    return _LIB_PATH


def _ref_so() -> Optional[str]:
    hits = sorted(glob.glob(os.path.join(_HERE, "_ref", "dhsa_ref_core*.so")))
    return hits[0] if hits else None


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P = C.POINTER(_Params)
        vp = C.c_void_p
        L.oracle_mix64.restype = C.c_uint64
        L.oracle_mix64.argtypes = [C.c_uint64]
        L.oracle_states.argtypes = [C.c_uint64, C.c_uint64, vp, vp]
        L.oracle_forward.argtypes = [P, C.c_uint64, vp]
        L.oracle_h1.restype = C.c_uint64
        L.oracle_h1.argtypes = [P, C.c_uint64]
        L.oracle_reconstruct_key.restype = C.c_int
        L.oracle_reconstruct_key.argtypes = [P, vp, vp]
        L.oracle_sketch_bytes.restype = C.c_size_t
        L.oracle_sketch_bytes.argtypes = [P]
        L.oracle_update_batch.argtypes = [P, vp, vp, vp, C.c_size_t]
        L.oracle_update_batch_mt.restype = C.c_int
        L.oracle_update_batch_mt.argtypes = [P, vp, vp, vp, C.c_size_t, C.c_int]
        L.oracle_zero_counts.argtypes = [P, vp, vp]
        L.oracle_hot_threshold.restype = C.c_double
        L.oracle_hot_threshold.argtypes = [C.c_int32, C.c_double]
        L.oracle_hot_sets.argtypes = [P, vp, C.c_double, vp, vp]
        L.oracle_zero_totals.argtypes = [P, vp, vp]
        L.oracle_flow_count.restype = C.c_double
        L.oracle_flow_count.argtypes = [P, vp, vp]
        L.oracle_bit_set_probability.restype = C.c_double
        L.oracle_bit_set_probability.argtypes = [P, C.c_double]
        L.oracle_candidate_hosts.restype = C.c_int
        L.oracle_candidate_hosts.argtypes = [P, vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp, vp, vp]
        L.oracle_shared_zero_counts.argtypes = [P, vp, vp, C.c_size_t, vp]
        L.oracle_corrected_estimate.restype = C.c_double
        L.oracle_corrected_estimate.argtypes = [P, C.c_int64, C.c_double, vp]
        L.oracle_restore_superpoints.restype = C.c_int
        L.oracle_restore_superpoints.argtypes = [P, vp, C.c_double, C.c_uint64, vp, vp, vp, vp, vp, vp]
        L.oracle_merge.argtypes = [vp, vp, vp, C.c_size_t]
        _lib = L
    return _lib


def mix64(x: int) -> int:
    return int(lib().oracle_mix64(x & (2 ** 64 - 1)))


def mix64_many(x: np.ndarray) -> np.ndarray:
    """Vector form for building test inputs (pkg/src/dhsa/dhg.py:47-56)."""
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint64(30)
        x *= np.uint64(0xBF58476D1CE4E5B9)
        x ^= x >> np.uint64(27)
        x *= np.uint64(0x94D049BB133111EB)
        x ^= x >> np.uint64(31)
    return x


def distinct_pairs(n: int, seed: int):
    """The reference test-suite's pair fixture (pkg/tests/conftest.py:25-34)."""
    mixed = mix64_many(np.arange(n, dtype=np.uint64) ^ np.uint64(seed << 34))
    return ((mixed >> np.uint64(32)).astype(np.uint32),
            (mixed & np.uint64(0xFFFFFFFF)).astype(np.uint32))


def plant_pairs(host: int, fanout: int, seed: int = 0):
    """`fanout` distinct opposites of one host (pkg/tests/test_dhla.py:30-37)."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 2 ** 32, dtype=np.uint64)
    opp = ((base + np.arange(fanout, dtype=np.uint64)) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return np.full(fanout, host, dtype=np.uint32), opp


class OracleCapacityError(Exception):
    def __init__(self, stage: int, count: int, max_candidates: int):
        self.stage, self.count, self.max_candidates = stage, count, max_candidates
        # text of pkg/src/dhsa/dhla.py:270-273
        super().__init__(f"restore stage {stage} produced {count} partial keys "
                         f"(max_candidates={max_candidates})")


@dataclass(frozen=True)
class OracleReport:
    host: int
    estimate: float
    saturated: bool


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


class OracleSketch:
    """CPU sketch with the reference's read-out chain, for checking the GPU path."""

    def __init__(self, r=5, g=1024, k=14, alpha=6, key_width=32,
                 seed_dh0=DEFAULT_SEED_DH0, seed_h1=DEFAULT_SEED_H1):
        self.r, self.g, self.k, self.alpha, self.key_width = r, g, k, alpha, key_width
        self.seed_dh0, self.seed_h1 = seed_dh0, seed_h1
        s0, s1 = C.c_uint64(), C.c_uint64()
        lib().oracle_states(seed_dh0, seed_h1, C.byref(s0), C.byref(s1))
        self.state_dh0, self.state_h1 = s0.value, s1.value
        self._p = _Params(r, g, k, alpha, key_width, 0, self.state_dh0, self.state_h1)
        self.bits = np.zeros((r, 1 << k, g // 8), dtype=np.uint8)
        assert self.bits.nbytes == lib().oracle_sketch_bytes(C.byref(self._p))

    @classmethod
    def from_params(cls, p) -> "OracleSketch":
        """From any object with the reference's DhgParams field names."""
        return cls(p.r, p.g, p.k, p.alpha, p.key_width, p.seed_dh0, p.seed_h1)

    # -- hashing ---------------------------------------------------------
    def forward(self, host: int) -> tuple:
        out = np.empty(self.r, dtype=np.uint64)
        lib().oracle_forward(C.byref(self._p), host, _ptr(out))
        return tuple(int(v) for v in out)

    def h1(self, opposite: int) -> int:
        return int(lib().oracle_h1(C.byref(self._p), opposite))

    def reconstruct_key(self, indices) -> Optional[int]:
        idx = np.asarray(indices, dtype=np.uint64)
        key = C.c_uint64()
        ok = lib().oracle_reconstruct_key(C.byref(self._p), _ptr(idx), C.byref(key))
        return int(key.value) if ok else None

    # -- scan --------------------------------------------------------------
    def update_batch(self, cand, opp, threads: int = 1) -> None:
        cand = np.ascontiguousarray(cand, dtype=np.uint32)
        opp = np.ascontiguousarray(opp, dtype=np.uint32)
        if len(cand) != len(opp):
            raise ValueError("candidate and opposite arrays differ in length")
        if threads > 1:
            lib().oracle_update_batch_mt(C.byref(self._p), _ptr(self.bits), _ptr(cand), _ptr(opp),
                                         len(cand), threads)
        else:
            lib().oracle_update_batch(C.byref(self._p), _ptr(self.bits), _ptr(cand), _ptr(opp),
                                      len(cand))

    def update(self, candidate: int, opposite: int) -> None:
        self.update_batch(np.array([candidate], np.uint32), np.array([opposite], np.uint32))

    # -- read-out ------------------------------------------------------------
    def zero_counts(self) -> np.ndarray:
        out = np.empty((self.r, 1 << self.k), dtype=np.int64)
        lib().oracle_zero_counts(C.byref(self._p), _ptr(self.bits), _ptr(out))
        return out

    def hot_sets(self, theta, zero_counts=None) -> list:
        zc = self.zero_counts() if zero_counts is None else np.ascontiguousarray(zero_counts, np.int64)
        lists = np.empty((self.r, 1 << self.k), dtype=np.uint64)
        counts = np.empty(self.r, dtype=np.uint64)
        lib().oracle_hot_sets(C.byref(self._p), _ptr(zc), float(theta), _ptr(lists), _ptr(counts))
        return [lists[i, : int(counts[i])].copy() for i in range(self.r)]

    def zero_totals(self, zero_counts=None) -> np.ndarray:
        zc = self.zero_counts() if zero_counts is None else zero_counts
        zr = np.empty(self.r, dtype=np.int64)
        lib().oracle_zero_totals(C.byref(self._p), _ptr(zc), _ptr(zr))
        return zr

    def estimate_flow_count(self, zero_counts=None):
        zr = self.zero_totals(zero_counts)
        sat = C.c_int()
        v = lib().oracle_flow_count(C.byref(self._p), _ptr(zr), C.byref(sat))
        return float(v), bool(sat.value)

    def bit_set_probability(self, flow_count: float) -> float:
        return float(lib().oracle_bit_set_probability(C.byref(self._p), flow_count))

    def candidate_hosts(self, theta, max_candidates=1 << 20, return_stage_counts=False):
        hot = self.hot_sets(theta)
        m = 1 << self.k
        lists = np.zeros((self.r, m), dtype=np.uint64)
        counts = np.zeros(self.r, dtype=np.uint64)
        for i, h in enumerate(hot):
            lists[i, : len(h)] = h
            counts[i] = len(h)
        out = np.empty(max(1, min(max_candidates, 1 << 24)), dtype=np.uint64)
        n = C.c_uint64()
        fs, fc = C.c_int32(), C.c_uint64()
        sc = np.zeros(self.r - 2, dtype=np.uint64)
        rc = lib().oracle_candidate_hosts(C.byref(self._p), _ptr(lists), _ptr(counts), max_candidates,
                                          _ptr(out), len(out), C.byref(n), C.byref(fs), C.byref(fc), _ptr(sc))
        if rc == 4:
            raise OracleCapacityError(fs.value, fc.value, max_candidates)
        if rc != 0:
            raise MemoryError("oracle_candidate_hosts")
        hosts = out[: n.value].copy()
        return (hosts, [int(v) for v in sc]) if return_stage_counts else hosts

    def shared_zero_counts(self, hosts) -> np.ndarray:
        hosts = np.ascontiguousarray(hosts, dtype=np.uint64)
        sz = np.empty(len(hosts), dtype=np.int64)
        lib().oracle_shared_zero_counts(C.byref(self._p), _ptr(self.bits), _ptr(hosts), len(hosts),
                                        _ptr(sz))
        return sz

    def corrected_estimate(self, sz: int, psi: float):
        sat = C.c_int()
        v = lib().oracle_corrected_estimate(C.byref(self._p), int(sz), float(psi), C.byref(sat))
        return float(v), bool(sat.value)

    def restore_superpoints(self, theta, max_candidates=1 << 20) -> list:
        cap = max(1, max_candidates)
        hosts = np.empty(cap, dtype=np.uint64)
        est = np.empty(cap, dtype=np.float64)
        sat = np.empty(cap, dtype=np.uint8)
        n = C.c_uint64()
        fs, fc = C.c_int32(), C.c_uint64()
        rc = lib().oracle_restore_superpoints(C.byref(self._p), _ptr(self.bits), float(theta),
                                              max_candidates, _ptr(hosts), _ptr(est), _ptr(sat),
                                              C.byref(n), C.byref(fs), C.byref(fc))
        if rc == 4:
            raise OracleCapacityError(fs.value, fc.value, max_candidates)
        if rc != 0:
            raise MemoryError("oracle_restore_superpoints")
        return [OracleReport(int(hosts[t]), float(est[t]), bool(sat[t])) for t in range(n.value)]

    def merged_with(self, other: "OracleSketch") -> "OracleSketch":
        out = OracleSketch(self.r, self.g, self.k, self.alpha, self.key_width,
                           self.seed_dh0, self.seed_h1)
        lib().oracle_merge(_ptr(out.bits), _ptr(self.bits), _ptr(other.bits), self.bits.nbytes)
        return out


# ---------------------------------------------------------------------------
# Window engine restatement (numpy; small cases).
# ---------------------------------------------------------------------------

TRACE_DTYPE = np.dtype([("ts", "<u4"), ("src", ">u4"), ("dst", ">u4")])  # pkg/src/dhsa/ingest.py:20


def run_windows(records: np.ndarray, window_seconds: int, theta, direction: str = "src",
                max_candidates: int = 1 << 20, **sketch_kw):
    """Tumbling-window detection over a record stream, as the reference's engine defines it
    (pkg/src/dhsa/engine.py:132-176; chunking there does not change the result):

      window of a record   ts // window_seconds                              engine.py:140
      arrival window       running maximum of the window ids so far          engine.py:143-145
      late record          window < arrival window: dropped, counted in the  engine.py:148,154
                           window that was open when it arrived
      direction policy     src: (src, dst); dst: (dst, src); both: both      engine.py:179-194
      a window is sealed and restored when a later one opens, or at the end  engine.py:150-152,159

    Returns [(window_id, pairs, dropped, [OracleReport])]."""
    if len(records) == 0:
        return []
    wins = records["ts"].astype(np.int64) // window_seconds
    arrival = np.maximum.accumulate(wins)
    src = records["src"].astype(np.uint32)
    dst = records["dst"].astype(np.uint32)
    out = []
    for wid in np.unique(arrival):
        span = arrival == wid
        on_time = span & (wins == arrival)
        s, d = src[on_time], dst[on_time]
        if direction == "src":
            cand, opp = s, d
        elif direction == "dst":
            cand, opp = d, s
        elif direction == "both":
            cand, opp = np.concatenate([s, d]), np.concatenate([d, s])
        else:
            raise ValueError(direction)
        sk = OracleSketch(**sketch_kw)
        sk.update_batch(cand, opp)
        out.append((int(wid), int(len(cand)), int(span.sum() - on_time.sum()),
                    sk.restore_superpoints(theta, max_candidates)))
    return out


def exact_counts(records: np.ndarray, direction: str = "src") -> dict:
    """Exact distinct-opposite count per candidate host (pkg/src/dhsa/ingest.py:159-176):
    unique 64-bit (cand << 32 | opp) keys, then a count per candidate."""
    if len(records) == 0:
        return {}
    src = records["src"].astype(np.uint64)
    dst = records["dst"].astype(np.uint64)
    if direction == "src":
        cand, opp = src, dst
    elif direction == "dst":
        cand, opp = dst, src
    elif direction == "both":
        cand, opp = np.concatenate([src, dst]), np.concatenate([dst, src])
    else:
        raise ValueError(direction)
    pairs = np.unique((cand << np.uint64(32)) | opp)
    hosts, counts = np.unique(pairs >> np.uint64(32), return_counts=True)
    return {int(h): int(c) for h, c in zip(hosts, counts)}


def _fmix32_many(x):
    x = x.astype(np.uint32, copy=True)
    with np.errstate(over="ignore"):
        x ^= x >> np.uint32(16)
        x *= np.uint32(0x85EBCA6B)
        x ^= x >> np.uint32(13)
        x *= np.uint32(0xC2B2AE35)
        x ^= x >> np.uint32(16)
    return x


def generate_trace_spec(background_hosts=0, background_max_cardinality=256, background_zipf=1.5, superpoints=0,
                        super_cardinality=(2048, 8192), duplicate_factor=1, start_ts=0, window_seconds=300, seed=0):
    """numpy restatement of the device generator's definition (paper_1803_11449_b200/traces.py,
    csrc k_generate_trace), which follows the reference generator's semantics
    (pkg/src/dhsa/ingest.py:109-153) over a counter-based random source:

      hosts[i]   fmix32(i ^ low32(mix64(seed ^ TAG_HOST)))            distinct (bijection)   ingest.py:121
      cards[i]   background: 1 + #{k : floor(2^53 P(zipf<=k)) <= u_i >> 11}, capped          ingest.py:123-126
                 super: lo + u_i mod (hi - lo + 1), u_i = mix64(i + (seed ^ TAG_CARD))       ingest.py:127-129
      dst        bases[h] + offset within the host (mod 2^32): distinct per host             ingest.py:131-137
      position p record perm(p) mod flows, perm = 4-round Feistel with cycle walking; each
                 flow exactly duplicate_factor times, shuffled                                ingest.py:139-147
      ts         start_ts + floor(p * window_seconds / total): time-ordered                   ingest.py:143-148

    Returns (records TRACE_DTYPE, truth dict)."""
    M64 = (1 << 64) - 1
    n_hosts = background_hosts + superpoints
    if n_hosts == 0:
        return np.empty(0, dtype=TRACE_DTYPE), {}
    seed64 = seed & M64
    idx = np.arange(n_hosts, dtype=np.uint64)
    host_key = mix64(seed64 ^ 0x1F83D9ABFB41BD6B) & 0xFFFFFFFF
    hosts = _fmix32_many(idx.astype(np.uint32) ^ np.uint32(host_key))
    with np.errstate(over="ignore"):
        u = mix64_many(idx + np.uint64(seed64 ^ 0x5BE0CD19137E2179))
        bases = mix64_many(idx + np.uint64(seed64 ^ 0xCBBB9D5DC1059ED8)) & np.uint64(0xFFFFFFFF)
    cards = np.empty(n_hosts, dtype=np.int64)
    if background_hosts:
        kmax, a = background_max_cardinality, background_zipf
        if kmax > 1:
            big = 1_000_000
            zeta = float(np.sum(np.arange(1, big + 1, dtype=np.float64) ** -a)) + (big + 0.5) ** (1.0 - a) / (a - 1.0)
            cdf = np.cumsum(np.arange(1, kmax, dtype=np.float64) ** -a) / zeta
            thr = np.floor(np.minimum(cdf, 1.0) * float(1 << 53)).astype(np.uint64)
        else:
            thr = np.empty(0, dtype=np.uint64)
        cards[:background_hosts] = 1 + np.searchsorted(thr, u[:background_hosts] >> np.uint64(11), side="right")
    if superpoints:
        lo, hi = super_cardinality
        cards[background_hosts:] = lo + (u[background_hosts:] % np.uint64(hi - lo + 1)).astype(np.int64)
    prefix = np.concatenate([[0], np.cumsum(cards)]).astype(np.uint64)
    flows = int(prefix[-1])
    total = flows * duplicate_factor
    bits = 2
    while (1 << bits) < total:
        bits += 1
    hb = (bits + 1) // 2
    mask = np.uint64((1 << hb) - 1)
    key = mix64(seed64 ^ 0x629A292A367CD507)
    x = np.arange(total, dtype=np.uint64)
    todo = np.ones(total, dtype=bool)
    while todo.any():
        cur = x[todo]
        l, r = (cur >> np.uint64(hb)) & mask, cur & mask
        for rnd in range(4):
            k = np.uint64(((key + rnd) * 0x9E3779B97F4A7C15) & M64)
            f = mix64_many(r ^ k) & mask
            l, r = r, l ^ f
        cur = (l << np.uint64(hb)) | r
        x[todo] = cur
        todo[todo] = cur >= np.uint64(total)
    f_idx = x % np.uint64(flows)
    h = np.searchsorted(prefix, f_idx, side="right") - 1
    rec = np.empty(total, dtype=TRACE_DTYPE)
    rec["src"] = hosts[h]
    rec["dst"] = ((bases[h] + (f_idx - prefix[h])) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    p = np.arange(total, dtype=object) if total * window_seconds >= (1 << 63) else np.arange(total, dtype=np.uint64)
    rec["ts"] = (start_ts + (p * window_seconds) // total).astype(np.uint32)
    return rec, {int(a_): int(c) for a_, c in zip(hosts.tolist(), cards.tolist())}


def engine_trace(seed: int, n_noise: int = 90_000, window_seconds: int = 300):
    """A deterministic multi-window trace with late records, built from mix64 only (no
    library RNG): three and a half windows of background pairs in time order, three hosts
    planted in windows 1, 1 and 2 with 2048..2600 destinations, 3% of records re-stamped
    up to two windows into the past (late), and one early record far in the future that
    opens window 5 before the rest of the trace ends."""
    cand, opp = distinct_pairs(n_noise, seed)
    ts = (np.arange(n_noise, dtype=np.uint64) * np.uint64(int(3.5 * window_seconds))) // np.uint64(n_noise)
    parts_c, parts_o, parts_t = [cand], [opp], [ts.astype(np.uint32)]
    for n, (host, fan, win) in enumerate(((0x0A0B0C0D, 2048, 1), (0xC0A80001, 2600, 1), (0x08080404, 2300, 2))):
        c2 = np.full(fan, host, dtype=np.uint32)
        o2 = (mix64_many(np.arange(fan, dtype=np.uint64) ^ np.uint64((seed + n + 1) << 40)) &
              np.uint64(0xFFFFFFFF)).astype(np.uint32)
        t2 = (np.uint64(win * window_seconds) +
              mix64_many(np.arange(fan, dtype=np.uint64) ^ np.uint64(77 + n)) % np.uint64(window_seconds))
        parts_c.append(c2), parts_o.append(o2), parts_t.append(t2.astype(np.uint32))
    cand, opp, ts = np.concatenate(parts_c), np.concatenate(parts_o), np.concatenate(parts_t)
    order = np.argsort(ts, kind="stable")
    cand, opp, ts = cand[order], opp[order], ts[order].astype(np.int64)
    pick = mix64_many(np.arange(len(ts), dtype=np.uint64) ^ np.uint64(seed * 1315423911))
    late = (pick % np.uint64(100)) < np.uint64(3)
    back = ((pick >> np.uint64(20)) % np.uint64(2 * window_seconds)).astype(np.int64)
    ts = np.where(late, np.maximum(ts - back, 0), ts)
    ts[len(ts) * 3 // 4] = 5 * window_seconds + 7   # a jump ahead: everything after it in windows < 5 is late
    rec = np.empty(len(ts), dtype=TRACE_DTYPE)
    rec["ts"], rec["src"], rec["dst"] = ts.astype(np.uint32), cand, opp
    return rec


# ---------------------------------------------------------------------------
# The reference's own compiled loops (oracle/_ref), when they were built.
# ---------------------------------------------------------------------------

_ref_core = None


def load_ref_core():
    """The reference's compiled `_core` module, or None if oracle/_ref is absent.

    Exposes ``update_batch(bits, state_dh0, state_h1, k, alpha, cand, opp)``,
    ``zero_counts(bits)`` and ``mix64(z)`` exactly as
    /root/reference/pkg/src/dhsa/_core.pyx:47-118 defines them.
    """
    global _ref_core
    if _ref_core is None:
        path = _ref_so()
        if path is None:
            return None
        loader = importlib.machinery.ExtensionFileLoader("dhsa_ref_core", path)
        spec = importlib.util.spec_from_loader("dhsa_ref_core", loader)
        mod = importlib.util.module_from_spec(spec)
        loader.exec_module(mod)
        _ref_core = mod
    return _ref_core
