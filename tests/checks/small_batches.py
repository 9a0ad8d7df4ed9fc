"""How the sketch behaves the way the reference engine drives it (engine.py:78-86): pageable host
arrays fed in batches of batch_pairs = 65536 from a thread pool onto one sketch."""
import json
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, ".")
import paper_1803_11449_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker only)

N = 20_000_000
cand, opp = O.distinct_pairs(N // 20, 5)
rng = np.random.default_rng(1)
pick = rng.integers(0, len(cand), size=N)
cand, opp = cand[pick].copy(), opp[pick].copy()          # pageable, 20 packets per flow
ora = O.OracleSketch()
ora.update_batch(cand, opp, threads=8)
out = []
for batch in (65536, 1 << 20, N):
    for workers in (1, 8):
        sk = P.Dhla(P.DhgParams())
        sk.update_batch(cand[:batch], opp[:batch])
        sk.reset()
        sk.seal()
        t0 = time.perf_counter()
        if workers == 1:
            for lo in range(0, N, batch):
                sk.update_batch(cand[lo:lo + batch], opp[lo:lo + batch])
        else:
            with ThreadPoolExecutor(workers) as pool:
                futs = [pool.submit(sk.update_batch, cand[lo:lo + batch], opp[lo:lo + batch]) for lo in range(0, N, batch)]
                for f in futs:
                    f.result()
        sk.seal()
        dt = time.perf_counter() - t0
        out.append(dict(batch_pairs=batch, workers=workers, mpps=N / dt / 1e6, bits_equal_oracle=bool(np.array_equal(sk.bits, ora.bits))))
        print(json.dumps(out[-1]), file=sys.stderr, flush=True)
print(json.dumps({"packets": N, "host_memory": "pageable numpy arrays", "runs": out}))
