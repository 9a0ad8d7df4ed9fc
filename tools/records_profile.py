"""Launch-level timing of DetectionEngine.run on raw device records (row N1): run under
ncu --metrics gpu__time_duration.sum for the launch list, or plain for wall/event timing."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1803_11449_b200 as P  # noqa: E402

cfg = P.GeneratorConfig(background_hosts=150_000, superpoints=50, duplicate_factor=26, window_seconds=600, start_ts=2100)
got = P.generate_trace_device(cfg, seed=100, fmt="records")
raw = got["records"]
n = got["total"]
eng = P.DetectionEngine(P.WindowConfig(theta=1024, window_seconds=300))
for _ in range(2):
    res = eng.run(raw)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(3):
    res = eng.run(raw)
e1.record()
torch.cuda.synchronize()
print(f"{n} records, windows {[r.window_id for r in res]}, pairs {[r.pairs for r in res]}, "
      f"{e0.elapsed_time(e1) / 3:.3f} ms per run (events), {(time.perf_counter() - t0) / 3 * 1e3:.3f} ms wall")
if len(sys.argv) > 1 and sys.argv[1] == "--cprofile":
    import cProfile
    import pstats

    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        eng.run(raw)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
