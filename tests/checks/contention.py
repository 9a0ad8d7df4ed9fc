"""BASELINE config 4: Zipf-skewed DDoS trace -- 1M sources to 4 victims -- scanned with the
victims as candidates (direction "dst": every packet lands in the same 5 x 4 cells) and as
opposites ("src": no contention), per scan mode.  Prints one JSON document."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1803_11449_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only: bits are compared, nothing is timed through it)

N = 100_000_000


def main():
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    victims = torch.tensor([0x0A000001, 0x0A000002, 0xC0A80101, 0x08080808], dtype=torch.int64, device="cuda")
    w = torch.tensor([1.0 / (i + 1) ** 1.2 for i in range(4)], device="cuda")
    vic = victims[torch.multinomial(w, N, replacement=True, generator=g)].to(torch.int32)
    sources = torch.randint(0, 2 ** 32, (1_000_000,), device="cuda", generator=g, dtype=torch.int64)
    src = (sources[torch.randint(0, 1_000_000, (N,), device="cuda", generator=g)] - (1 << 32) * (sources[0] * 0)).to(torch.int64)
    src = torch.where(src >= 2 ** 31, src - 2 ** 32, src).to(torch.int32)
    out = []
    ora = {}
    for direction, (cand, opp) in (("dst", (vic, src)), ("src", (src, vic))):
        u = torch.unique((cand.to(torch.int64) & 0xFFFFFFFF) << 32 | (opp.to(torch.int64) & 0xFFFFFFFF))
        uc = ((u >> 32) & 0xFFFFFFFF).cpu().numpy().astype(np.uint32)
        uo = (u & 0xFFFFFFFF).cpu().numpy().astype(np.uint32)
        o = O.OracleSketch()
        o.update_batch(uc, uo, threads=8)
        ora[direction] = o
        for mode in ("red", "test", "test_agg", "flow_cache", "auto"):
            sk = P.Dhla(P.DhgParams())
            sk.set_scan_mode(mode)
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sk.use_stream(stream.cuda_stream)
                sk.update_batch(cand, opp)
                sk.reset()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                sk.update_batch(cand, opp)
                e1.record(stream)
                torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            ok = bool(np.array_equal(sk.bits, o.bits))
            reps = sk.restore_superpoints(1024)
            out.append(dict(direction=direction, mode=mode, packets=N, distinct_pairs=int(len(u)), scan_ms=ms,
                            gpps=N / (ms * 1e-3) / 1e9, bits_equal_oracle=ok, reports=len(reps),
                            saturated=sum(r.saturated for r in reps)))
            print(json.dumps(out[-1]), file=sys.stderr, flush=True)
    print(json.dumps({"runs": out}, indent=1))


if __name__ == "__main__":
    main()
