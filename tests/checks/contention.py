"""BASELINE config 4 and the auto policy.

(1) Zipf-skewed DDoS trace -- 1M sources to 4 victims -- scanned with the victims as candidates
    (direction "dst": every packet lands in the same 5 x 4 cells) and as opposites ("src": no
    contention), per scan mode; bits are compared with the oracle in every run.
(2) `auto` must never lose to a fixed mode by more than 5%: on both directions of (1), on a
    config-2 window (flows repeat ~26 times) and on an all-distinct window (no flow repeats), fed in
    16 batches, as an engine feeds chunks, so the host policy can react inside the window, and in one
    launch, where the device decides (k_auto_decide).  Every mode
    gets one untimed window first, then three timed windows (best of three).
Prints one JSON document; exits non-zero if a bit array differs or auto loses.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1803_11449_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only: bits are compared, nothing is timed through it)

N = 100_000_000
MODES = ("red", "test", "test_agg", "flow_cache", "auto")


def as_i32(t):
    return torch.where(t >= 2 ** 31, t - 2 ** 32, t).to(torch.int32)


def ddos():
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    victims = torch.tensor([0x0A000001, 0x0A000002, 0xC0A80101, 0x08080808], dtype=torch.int64, device="cuda")
    w = torch.tensor([1.0 / (i + 1) ** 1.2 for i in range(4)], device="cuda")
    vic = victims[torch.multinomial(w, N, replacement=True, generator=g)]
    sources = torch.randint(0, 2 ** 32, (1_000_000,), device="cuda", generator=g, dtype=torch.int64)
    src = sources[torch.randint(0, 1_000_000, (N,), device="cuda", generator=g)]
    return as_i32(vic), as_i32(src)


def oracle_bits(cand, opp):
    u = torch.unique(((cand.to(torch.int64) & 0xFFFFFFFF) << 32) | (opp.to(torch.int64) & 0xFFFFFFFF))
    uc = ((u >> 32) & 0xFFFFFFFF).cpu().numpy().astype(np.uint32)
    uo = (u & 0xFFFFFFFF).cpu().numpy().astype(np.uint32)
    o = O.OracleSketch()
    o.update_batch(uc, uo, threads=8)
    return o.bits, int(len(u))


def run(name, cand, opp, want_bits, distinct, batches=1, modes=MODES):
    rows = []
    n = len(cand)
    cuts = [n * i // batches // 4 * 4 for i in range(batches)] + [n]
    for mode in modes:
        sk = P.Dhla(P.DhgParams())
        sk.set_scan_mode(mode)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            sk.use_stream(stream)
            best, used = None, None
            for rep in range(4):                      # rep 0: untimed warm-up
                sk.reset()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for lo, hi in zip(cuts[:-1], cuts[1:]):
                    sk.update_batch(cand[lo:hi], opp[lo:hi])
                    if batches > 1:
                        sk.flow_cache_stats()        # an engine's per-chunk bookkeeping: lets the async snapshot land
                e1.record(stream)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                used = sk.scan_mode_used
                ok = bool(np.array_equal(sk.bits, want_bits))
                try:
                    reps = sk.restore_superpoints(1024)
                except P.CapacityError:             # 100M distinct flows make every cell hot, as in the reference
                    reps = []
                if rep and (best is None or ms < best):
                    best = ms
        rows.append(dict(trace=name, mode=mode, kernel_used_last=used, packets=n, distinct_pairs=distinct, scan_ms=best,
                         gpps=n / (best * 1e-3) / 1e9, bits_equal_oracle=ok, reports=len(reps),
                         saturated=sum(r.saturated for r in reps)))
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    return rows


def main():
    out = []
    vic, src = ddos()
    for direction, (cand, opp) in (("ddos_dst", (vic, src)), ("ddos_src", (src, vic))):
        bits, distinct = oracle_bits(cand, opp)
        out += run(direction, cand, opp, bits, distinct)
    del vic, src
    # config 2: flows repeat
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    import bench
    c_np, o_np, fsrc, fdst, _ = bench.make_window(100, N, 0)
    cand, opp = torch.from_numpy(c_np.view(np.int32)).cuda(), torch.from_numpy(o_np.view(np.int32)).cuda()
    ora = O.OracleSketch()
    ora.update_batch(fsrc, fdst, threads=8)
    out += run("config2", cand, opp, ora.bits, len(fsrc), modes=("test_agg", "flow_cache", "auto"))
    # all distinct: no flow repeats
    c_np, o_np = O.distinct_pairs(N, 909)
    cand, opp = torch.from_numpy(c_np.view(np.int32)).cuda(), torch.from_numpy(o_np.view(np.int32)).cuda()
    ora = O.OracleSketch()
    ora.update_batch(c_np, o_np, threads=8)
    out += run("all_distinct_16_batches", cand, opp, ora.bits, N, batches=16, modes=("test", "test_agg", "flow_cache", "auto"))
    # the same window handed over in ONE launch: the host cannot react inside it, the launch is sampled and gated on the device
    out += run("all_distinct_one_launch", cand, opp, ora.bits, N, batches=1, modes=("test", "flow_cache", "auto"))
    verdict = {}
    for trace in dict.fromkeys(r["trace"] for r in out):
        rows = [r for r in out if r["trace"] == trace]
        best = max(r["gpps"] for r in rows)
        auto = next(r["gpps"] for r in rows if r["mode"] == "auto")
        verdict[trace] = dict(best_gpps=best, auto_gpps=auto, auto_over_best=auto / best)
    ok_bits = all(r["bits_equal_oracle"] for r in out)
    ok_auto = all(v["auto_over_best"] >= 0.95 for v in verdict.values())
    print(json.dumps({"runs": out, "auto_vs_best": verdict, "bits_ok": ok_bits, "auto_within_5pct": ok_auto}, indent=1))
    sys.exit(0 if ok_bits and ok_auto else 1)


if __name__ == "__main__":
    main()
