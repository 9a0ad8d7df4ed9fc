"""Per-warp table bypass of the flow-cache scan (k_scan_flowcache): single large launches whose
keys do not repeat, repeat late, or repeat from the start.  Bits are compared with the oracle;
prints Gpps per scan mode.  tools/bypass_check.py [packets]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11449_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only)

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64_000_000


def timed(mode, cand, opp, want):
    sk = P.Dhla(P.DhgParams())
    sk.set_scan_mode(mode)
    best = None
    for rep in range(3):
        sk.reset()
        sk.seal()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.current_stream()
        e0.record(stream)
        sk.update_batch(cand, opp)
        e1.record(stream)
        sk.seal()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None or ms < best else best
    lookups, hits = sk.flow_cache_stats()
    return dict(mode=mode, ms=round(best, 3), gpps=round(len(cand) / best / 1e6, 1), used=sk.scan_mode_used,
                hit_rate=round(hits / lookups, 4) if lookups else None, bits_ok=bool(np.array_equal(sk.bits, want)))


def main():
    out = {}
    c_np, o_np = O.distinct_pairs(N, 909)
    ora = O.OracleSketch()
    ora.update_batch(c_np, o_np, threads=16)
    traces = {
        "all_distinct": (c_np, o_np),
        # no repeats in the first half, then the first half again: warps that went dry keep scanning test-first
        "distinct_then_repeat": (np.concatenate([c_np[: N // 2], c_np[: N // 2]]), np.concatenate([o_np[: N // 2], o_np[: N // 2]])),
    }
    half = O.OracleSketch()
    half.update_batch(c_np[: N // 2], o_np[: N // 2], threads=16)
    wants = {"all_distinct": ora.bits, "distinct_then_repeat": half.bits}
    for name, (c, o) in traces.items():
        cand = torch.from_numpy(c.view(np.int32)).cuda()
        opp = torch.from_numpy(o.view(np.int32)).cuda()
        out[name] = [timed(m, cand, opp, wants[name]) for m in ("test", "flow_cache", "auto")]
        for row in out[name]:
            print(name, json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))
    sys.exit(0 if all(r["bits_ok"] for rows in out.values() for r in rows) else 1)


if __name__ == "__main__":
    main()
