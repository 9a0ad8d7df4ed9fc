"""BASELINE config 3 on the hardware this build has: a 1B-packet window (config 2's flow population,
~259 packets per flow) generated on the device, scanned (a) whole on one B200 and (b) as 8 packet
shards into 8 private sketches that are OR-merged (the multi-GPU choreography, executed on one
device), then estimated and restored.  Bits, super point set and estimates are checked against the
oracle's run over the distinct flows.  Prints one JSON document."""
import hashlib
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1803_11449_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only)

THETA = 1024
SHARDS = 8


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    seed = 300
    flows_cfg = P.GeneratorConfig(background_hosts=150_000, superpoints=50, duplicate_factor=1)
    flows = P.generate_trace_device(flows_cfg, seed, fmt="pairs")
    dup = max(1, round(1_000_000_000 / flows["flows"]))
    cfg = P.GeneratorConfig(background_hosts=150_000, superpoints=50, duplicate_factor=dup)
    t0 = time.perf_counter()
    win = P.generate_trace_device(cfg, seed, fmt="pairs")
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    n = win["total"]
    cand, opp = win["cand"], win["opp"]

    ora = O.OracleSketch()
    ora.update_batch(flows["cand"].cpu().numpy().view(np.uint32), flows["opp"].cpu().numpy().view(np.uint32), threads=8)
    want = ora.restore_superpoints(THETA)

    stream = torch.cuda.Stream()
    out = {"packets": n, "distinct_flows": flows["flows"], "packets_per_flow": dup, "generate_s": gen_s, "runs": []}
    with torch.cuda.stream(stream):
        # (a) one sketch, the whole window
        sk = P.Dhla(P.DhgParams())
        sk.use_stream(stream.cuda_stream)
        for rep in range(3):
            sk.reset()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(stream)
            sk.update_batch(cand, opp)
            e[1].record(stream)
            got = sk.restore_superpoints(THETA)
            e[2].record(stream)
            torch.cuda.synchronize()
        ok_bits = sha(sk.bits) == sha(ora.bits)
        ok_sp = [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want] and \
            all(abs(a.estimate - b.estimate) <= 1e-6 * abs(b.estimate) for a, b in zip(got, want))
        ms_scan, ms_all = e[0].elapsed_time(e[1]), e[0].elapsed_time(e[2])
        out["runs"].append(dict(layout="1 sketch, whole window", scan_ms=ms_scan, window_ms=ms_all,
                                gpps_scan=n / ms_scan / 1e6, gpps_window=n / ms_all / 1e6,
                                bits_equal_oracle=bool(ok_bits), superpoints_equal_oracle=bool(ok_sp),
                                n_superpoints=len(got), flow_cache_hit_rate=sk.flow_cache_stats()[1] / n))
        # (b) 8 packet shards -> 8 private sketches -> OR merge -> restore (one device stands in for eight)
        parts = [P.Dhla(P.DhgParams()) for _ in range(SHARDS)]
        for p in parts:
            p.use_stream(stream.cuda_stream)
        cuts = [n * i // SHARDS // 4 * 4 for i in range(SHARDS)] + [n]
        for rep in range(2):
            for p in parts:
                p.reset()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(stream)
            for p, lo, hi in zip(parts, cuts[:-1], cuts[1:]):
                p.update_batch(cand[lo:hi], opp[lo:hi])
            e[1].record(stream)
            for p in parts[1:]:
                parts[0].merge_from(p)
            e[2].record(stream)
            got = parts[0].restore_superpoints(THETA)
            e[3].record(stream)
            torch.cuda.synchronize()
        ok_bits = sha(parts[0].bits) == sha(ora.bits)
        ok_sp = [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in want]
        out["runs"].append(dict(layout=f"{SHARDS} packet shards -> {SHARDS} sketches -> OR merge, on one device",
                                scan_ms=e[0].elapsed_time(e[1]), merge_ms=e[1].elapsed_time(e[2]),
                                restore_ms=e[2].elapsed_time(e[3]), window_ms=e[0].elapsed_time(e[3]),
                                gpps_window=n / e[0].elapsed_time(e[3]) / 1e6,
                                bits_equal_oracle=bool(ok_bits), superpoints_equal_oracle=bool(ok_sp)))
    # accuracy against the exact per-host truth of the generator
    m = P.evaluate(got, win["truth"], THETA)
    out["accuracy"] = m.as_dict()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
