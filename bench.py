#!/usr/bin/env python
"""bench.py -- packets/s of one detection window (scan + estimate + restore + filter).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2|3]

Workload (BASELINE.json configs[1]): default DDH parameters (r=5, g=1024, k=14,
alpha=6), theta 1024, a 100M-packet window per GPU: 150k uniform-address
background hosts with Zipf(1.5) cardinalities capped at 256 plus 50 injected
scanners with 2048..8192 destinations (~3.8M distinct flows), every packet a
uniform draw from the flow table (so ~26 packets per flow, shuffled).  A "step"
is one whole window: reset the sketch, scan every packet, (N > 1: OR-merge the
per-GPU sketches), estimate, restore and threshold-filter the super points.
Both arms build the window with the same numpy code from the same seed
(make_window), so they time the same packets.

One JSON line on rank 0 (see the keys below).  `value` is device-resident
throughput, windows pipelined the way a live detector runs them (window k's
read-out is enqueued, window k+1's reset and scan are queued behind it, then
window k's reports are collected; --no-pipeline waits per window instead); `e2e` pushes the same window from pinned HOST arrays through the
public API (`Dhla.update_batch(numpy)` -> C ABI), host<->device copies inside
the timed region; `e2e_dropin` feeds it the way the reference engine does --
ordinary pageable numpy arrays, 65,536-pair batches, 1 and 8 feeder threads --
through the reference's own unmodified WindowSession (baseline/_ref) holding the
CUDA sketch.  `--impl reference` times the unmodified reference package on the
host cores exactly as its own `dhsa bench` does (pkg/src/dhsa/cli.py:368-382:
WindowSession(cfg, 0, "compiled", pool).feed_batch + seal, then restore).

--config 3 (BASELINE.json configs[2]): ONE 1B-packet window split over the ranks
by packet_slice, each rank generating only its slice on the device; strong
scaling.  The default run is config 2, weak scaling at 100M packets per GPU.
"""
from __future__ import annotations

import argparse
import concurrent.futures
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

THETA = 1024
READBACK_BYTES = 1640 + 256 * 24   # sizeof(dhsa::Readback): control block with the window counters + the first 256 report rows
WORKLOAD = ("config2: 100M-packet window per GPU, default DDH (r5 g1024 k14 a6), 150k uniform background hosts "
            "(Zipf1.5 cardinality<=256) + 50 scanners (2048-8192), ~3.8M distinct flows, theta 1024")


# ------------------------------------------------------------------ workload --

def make_flows(seed: int, background_hosts: int = 150_000, scanners: int = 50):
    """Distinct (src, dst) flows of the window: the reference generator's population shape
    (/root/reference/pkg/src/dhsa/ingest.py:109-131) at config-2 scale."""
    rng = np.random.default_rng(seed)
    n_hosts = background_hosts + scanners
    hosts = np.unique(rng.integers(0, 2 ** 32, size=n_hosts + n_hosts // 32 + 64, dtype=np.uint64))
    rng.shuffle(hosts)
    hosts = hosts[:n_hosts]
    cards = np.empty(n_hosts, dtype=np.int64)
    cards[:background_hosts] = np.minimum(rng.zipf(1.5, size=background_hosts), 256)
    cards[background_hosts:] = rng.integers(2048, 8193, size=scanners)
    src = np.repeat(hosts, cards)
    bases = rng.integers(0, 2 ** 32, size=n_hosts, dtype=np.uint64)
    starts = np.repeat(np.cumsum(cards) - cards, cards).astype(np.uint64)
    dst = (np.repeat(bases, cards) + np.arange(len(src), dtype=np.uint64) - starts) & np.uint64(0xFFFFFFFF)
    return src.astype(np.uint32), dst.astype(np.uint32), hosts[background_hosts:].astype(np.uint32)


def make_window(seed: int, n: int, rank: int = 0):
    """(cand, opp, src, dst, scanners): the packets of one window -- n uniform draws from the flow
    table, every flow at least once when n allows -- and the distinct flows they were drawn from.
    Pure numpy from (seed, rank): the GPU arm and the reference arm time the same packets."""
    src, dst, scanners = make_flows(seed)
    flows = len(src)
    rng = np.random.default_rng(seed * 1000 + rank + 1)
    pick = rng.integers(0, flows, size=n, dtype=np.int64)
    if rank == 0 and n >= flows:
        pick[np.arange(flows, dtype=np.int64) * (n // flows)] = rng.permutation(flows)
    return src[pick], dst[pick], src, dst, scanners


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# -------------------------------------------------------------------- clocks --

class ClockSampler:
    """Samples SM clock and throttle reasons while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for row in self.rows:
            try:
                sm.append(float(row[0]))
                mx.append(float(row[1]))
            except (ValueError, IndexError):
                continue
            for name, cell in zip(names, row[3:7]):
                if cell.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU baseline --

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """The installed, unmodified reference package (baseline/install_reference.sh), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "dhsa")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import dhsa
        import dhsa.engine  # noqa: F401
        from dhsa._kernels import available_backends
        return dhsa if "compiled" in available_backends() else None
    except Exception:
        return None


def reference_window(dhsa, cand: np.ndarray, opp: np.ndarray, threads: int):
    """One window through the stock reference, as `dhsa bench` times it
    (/root/reference/pkg/src/dhsa/cli.py:368-382): WindowSession(cfg, 0, "compiled", pool),
    feed_batch (65,536-pair batches submitted to the pool) + seal, then restore (pure Python)."""
    from dhsa.engine import WindowConfig, WindowSession

    cfg = WindowConfig(workers=threads, theta=THETA)
    pool = concurrent.futures.ThreadPoolExecutor(max_workers=threads) if threads > 1 else None
    session = WindowSession(cfg, 0, "compiled", pool)
    t0 = time.perf_counter()
    session.feed_batch(cand, opp)
    session.seal()
    t_scan = time.perf_counter() - t0
    if pool is not None:
        pool.shutdown()
    t1 = time.perf_counter()
    reports = session.restore()
    t_restore = time.perf_counter() - t1
    return t_scan, t_scan + t_restore, reports


def port_window(cand: np.ndarray, opp: np.ndarray, threads: int):
    """Fallback when baseline/_ref did not travel: the oracle's C port of the same path."""
    from oracle import oracle as O

    ora = O.OracleSketch()
    t0 = time.perf_counter()
    ora.update_batch(cand, opp, threads=threads)
    t_scan = time.perf_counter() - t0
    reports = ora.restore_superpoints(THETA)
    return t_scan, time.perf_counter() - t0, reports


def cpu_window(cand, opp, threads):
    dhsa = load_reference()
    if dhsa is not None:
        return ("reference",) + reference_window(dhsa, cand, opp, threads)
    return ("port",) + port_window(cand, opp, threads)


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    n = args.packets
    cand, opp, src, _, _ = make_window(args.seed, n, 0)
    threads = os.cpu_count() or 1
    times, kind, reports = [], "port", []
    for it in range(args.warmup + args.steps):
        kind, _, t_all, reports = cpu_window(cand, opp, threads)
        if it >= args.warmup:
            times.append(t_all)
    total = sum(times)
    mpps = n * len(times) / total / 1e6
    sample = (f"the whole window: {n} packets over {len(src)} flows (the GPU arm's rank-0 window, same seed), "
              f"{threads} threads, batches of 65536, "
              + ("unmodified reference package from baseline/_ref: WindowSession.feed_batch + seal + restore"
                 if kind == "reference" else "oracle C port (baseline/_ref absent)"))
    print(json.dumps({
        "impl": "reference", "metric": "packets/sec per detection window (scan+estimate+restore)",
        "value": mpps, "unit": "Mpps", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32/u64 integer hashing + f64 estimates", "data": "synthetic",
        "config": {"workload": WORKLOAD, "packets_per_gpu": n, "distinct_flows": len(src), "theta": THETA},
        "n_superpoints": len(reports),
        "cpu_baseline": {"value": mpps, "unit": "Mpps", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": mpps, "unit": "Mpps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------- GPU arm --

_T0 = time.perf_counter()


def log(msg: str) -> None:
    """Progress on stderr (stdout carries only the JSON line)."""
    print(f"[bench +{time.perf_counter() - _T0:6.1f}s] {msg}", file=sys.stderr, flush=True)


def run_ours(args, rank: int, local_rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist

    import paper_1803_11449_b200 as P
    from paper_1803_11449_b200 import _cabi
    from paper_1803_11449_b200.multi import ShardedWindow

    # DHSA_BENCH_SAME_DEVICE=1: every rank on cuda:0 with gloo for the rendezvous -- a way to run the
    # N > 1 code path (slicing, barriers, peer-mapped OR merge over CUDA IPC) on a one-GPU box; not a measurement
    same_device = os.environ.get("DHSA_BENCH_SAME_DEVICE") == "1"
    if same_device:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if same_device:
            dist.init_process_group("gloo")
        else:
            # NCCL's communicator lines stay on (stderr: stdout carries the JSON line), so a reader of the
            # log can count the ranks that really joined
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    if args.config == 3:
        # BASELINE config 3: ONE window of ~1B packets split over the ranks; each rank generates only
        # its own packet slice, on the device (k_generate_trace), from the shared flow population
        from paper_1803_11449_b200.multi import packet_slice
        from paper_1803_11449_b200.traces import trace_population

        base = P.GeneratorConfig(background_hosts=150_000, superpoints=50, duplicate_factor=1)
        hosts, cards, bases = trace_population(base, args.seed)
        src = np.repeat(hosts, cards)
        ramp = (np.arange(len(src), dtype=np.int64) - np.repeat(np.cumsum(cards) - cards, cards)).astype(np.uint32)
        dst = np.repeat(bases, cards) + ramp
        scanners = hosts[cards >= 2048]
        flows = len(src)
        dup = max(1, round(args.window_packets / flows))
        cfg3 = P.GeneratorConfig(background_hosts=150_000, superpoints=50, duplicate_factor=dup)
        n_total = flows * dup
        lo, hi = packet_slice(n_total, rank, world)
        tr = P.generate_trace_device(cfg3, args.seed, device=local_rank, fmt="pairs", lo=lo, hi=hi)
        cand_d, opp_d = tr["cand"], tr["opp"]
        n = hi - lo
        del tr
    else:
        n = args.packets
        cand_np, opp_np, src, dst, scanners = make_window(args.seed, n, rank)
        flows = len(src)
        n_total = world * n
        cand_d = torch.from_numpy(cand_np.view(np.int32)).to(dev)
        opp_d = torch.from_numpy(opp_np.view(np.int32)).to(dev)
        del cand_np, opp_np
    torch.cuda.synchronize()

    log(f"window generated: {n} packets over {flows} flows")
    win = ShardedWindow(P.DhgParams(), theta=THETA, device=local_rank, merge=args.merge)
    sk = win.sketch
    sk.set_scan_mode(args.scan_mode)
    sk.set_flow_cache((args.flow_cache_mib << 20) // 32)
    stream = torch.cuda.Stream(dev)   # one stream for torch ops, the sketch's kernels and the timing events
    torch.cuda.set_stream(stream)
    sk.use_stream(stream)

    # -- roofline inputs measured here: random-address L2 rates (rank 0, N = 1 only)
    l2 = None
    if rank == 0 and world == 1 and not args.no_probe:
        import ctypes as C
        rates = {}
        for kind, name in ((0, "red"), (1, "ld")):
            out = C.c_double()
            _cabi.check(_cabi.lib().dhsa_probe_l2(local_rank, kind, 16 << 20, 1 << 28, C.byref(out)))
            rates[name] = out.value / 1e9
        l2 = {"buffer_mib": 16, "red_gops": rates["red"], "ld_gops": rates["ld"]}

    def step_device(events=None):
        if events:
            events[0].record(stream)
        win.reset()
        if events:
            events[3].record(stream)
        win.scan(cand_d, opp_d)
        if events:
            events[1].record(stream)
        win.merge()
        reports = win.restore()
        if events:
            events[2].record(stream)
        return reports

    # -- warm-up, then parity of what the timed steps compute (not timed)
    for _ in range(args.warmup):
        reports = step_device()
    parity = None
    if rank == 0 and not args.no_parity:
        # the CPU leg as checker (never timed here, never on the product path): the oracle scans the
        # window's distinct flows on the host and the GPU's bits / reports must equal its
        from oracle import oracle as O
        ora = O.OracleSketch()
        ora.update_batch(src, dst, threads=os.cpu_count() or 1)
        want = ora.restore_superpoints(THETA)
        if win.merged_with == "partition":   # the merged bits stay with their owners: this rank checks its own range and
            from paper_1803_11449_b200.multi import partition_ranges   # the gathered zero counts of every cell
            blo, bhi = partition_ranges(win.ops, world)[rank]
            bits_ok = (n * world >= flows) and sha(sk.bits.reshape(-1)[blo:bhi]) == sha(ora.bits.reshape(-1)[blo:bhi]) \
                and bool(np.array_equal(sk.zero_counts(), ora.zero_counts()))
        else:
            bits_ok = (n * world >= flows) and sha(sk.bits) == sha(ora.bits)
        sp_ok = [(r.host, r.saturated) for r in reports] == [(r.host, r.saturated) for r in want] and \
            all(abs(a.estimate - b.estimate) <= 1e-6 * abs(b.estimate) for a, b in zip(reports, want))
        parity = {"bits_equal_oracle": bool(bits_ok), "superpoints_equal_oracle": bool(sp_ok),
                  "n_superpoints": len(reports),
                  "scanners_found": int(len(set(scanners.tolist()) & {r.host for r in reports}))}

    log("warm-up and parity done")
    # -- timed: device-resident window
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    t_begin, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = sk.launch_count
    # clocks and throttle reasons are sampled (nvidia-smi, every 20 ms) from here to the end of the last timed
    # leg: the device-resident region alone lasts a few milliseconds, the e2e and record legs ~0.2 s
    clocks = ClockSampler(local_rank)
    clocks.__enter__()
    barrier()
    t_begin.record(stream)
    # Windows are pipelined the way a live detector runs them: the read-out of window k is
    # enqueued (dhsa_restore_begin), window k + 1's reset and scan are queued behind it, and only
    # then are window k's reports collected (dhsa_restore_end) -- the device never waits for the host.
    collected = []
    for k in range(args.steps):
        if args.no_pipeline:                                  # every window waits for its own reports
            collected.append(step_device(evs[k]))
            continue
        ev = evs[k]
        ev[0].record(stream)
        win.reset()
        ev[3].record(stream)
        win.scan(cand_d, opp_d)
        ev[1].record(stream)
        if k:
            collected.append(win.restore_end())          # window k - 1
        win.merge()
        win.restore_begin()
        ev[2].record(stream)
    if not args.no_pipeline:
        collected.append(win.restore_end())
    t_end.record(stream)
    barrier()
    if args.warmup == 0:
        reports = collected[0]
    same = all([(r.host, r.estimate, r.saturated) for r in c] == [(r.host, r.estimate, r.saturated) for r in reports]
               for c in collected)
    if parity is not None:
        parity["timed_windows_equal_warmup_reports"] = bool(same and len(collected) == args.steps)
    launches = sk.launch_count - launches0
    fc_lookups, fc_hits = sk.flow_cache_stats()
    ms_total = t_begin.elapsed_time(t_end)
    scan_ms = float(np.mean([e[3].elapsed_time(e[1]) for e in evs]))      # the scan kernel's launch alone
    reset_ms = float(np.mean([e[0].elapsed_time(e[3]) for e in evs]))     # window reset: sketch + flow cache cleared
    readout_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))

    log(f"device-resident timing done: {ms_total / args.steps:.3f} ms per window")
    # -- timed: end to end from pinned host arrays through the public API
    e2e = None
    if not args.no_e2e and n <= 200_000_000:
        cand_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
        opp_h = torch.empty(n, dtype=torch.int32, pin_memory=True)
        cand_h.copy_(cand_d)
        opp_h.copy_(opp_d)
        torch.cuda.synchronize()
        cand_np, opp_np = cand_h.numpy().view(np.uint32), opp_h.numpy().view(np.uint32)

        def step_host():
            win.reset()
            win.scan(cand_np, opp_np)   # Dhla.update_batch(numpy): chunked H2D overlapped with the scan
            win.merge()
            return win.restore()        # reports come back to host memory

        for _ in range(max(1, min(args.warmup, 2))):
            step_host()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            reports_h = step_host()
        e1.record(stream)
        barrier()
        e2e_ms = e0.elapsed_time(e1)
        e2e = (e2e_ms, len(reports_h))
        del cand_h, opp_h

    # -- timed: the drop-in path.  The reference's own, unmodified WindowSession (baseline/_ref) with the
    #    CUDA sketch in its seam, fed the way `dhsa bench` feeds it: ordinary
    #    pageable numpy arrays, feed_batch cutting them into 65,536-pair batches that 1 or 8 pool
    #    threads hand to update_batch, then seal and restore.  Wall clock around the whole window
    #    (the device is idle before and drained after).
    dropin = None
    if world == 1 and not args.no_e2e and not args.no_dropin and n <= 200_000_000:
        dhsa = load_reference()
        cand_pg = cand_d.cpu().numpy().view(np.uint32).copy()      # pageable
        opp_pg = opp_d.cpu().numpy().view(np.uint32).copy()
        runs = []
        for workers in (1, 8):
            if dhsa is not None:
                from dhsa.engine import WindowConfig as RefConfig, WindowSession as RefSession
                import dhsa.engine as ref_engine
                stock = ref_engine.Dhla
                ref_engine.Dhla = lambda params, backend="auto", window_id=0: P.Dhla(params, backend="cuda",
                                                                                     window_id=window_id, device=local_rank)
                make = lambda pool: RefSession(RefConfig(workers=workers, theta=THETA), 0, "auto", pool)
                engine = "reference WindowSession (baseline/_ref), unmodified"
            else:
                stock = None
                make = lambda pool: P.WindowSession(P.WindowConfig(workers=workers, theta=THETA), 0, device=local_rank)
                engine = "this package's WindowSession (baseline/_ref absent)"
            try:
                best, got = None, None
                reps = max(3, min(2 * args.steps, 10))     # + one untimed window; the host settles over the first few
                times = []
                for rep in range(1 + reps):
                    pool = concurrent.futures.ThreadPoolExecutor(max_workers=workers) if workers > 1 else None
                    session = make(pool)
                    session.sketch.set_scan_mode(args.scan_mode)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    if dhsa is not None or workers == 1:
                        session.feed_batch(cand_pg, opp_pg)
                    else:       # this package's session does not split: do what the reference's feed_batch does
                        futs = [pool.submit(session.sketch.update_batch, cand_pg[q:q + 65536], opp_pg[q:q + 65536])
                                for q in range(0, n, 65536)]
                        for f in futs:
                            f.result()
                    session.seal()
                    got = session.restore()
                    dt = time.perf_counter() - t0
                    if pool is not None:
                        pool.shutdown()
                    if rep:
                        times.append(dt)
                        if best is None or dt < best:
                            best = dt
                ok = [(r.host, r.saturated) for r in got] == [(r.host, r.saturated) for r in reports]
                runs.append({"feeder_threads": workers, "mpps": n / best / 1e6, "ms_per_window": best * 1e3,
                             "statistic": f"best of {len(times)} windows", "median_mpps": n / float(np.median(times)) / 1e6,
                             "reports_equal_device_run": bool(ok)})
            finally:
                if stock is not None:
                    ref_engine.Dhla = stock
        # what the engine's own hand-off costs with nothing behind it: the same number of pool.submit calls of
        # a function that returns at once (CPython's executor + GIL; the library is not involved)
        with concurrent.futures.ThreadPoolExecutor(max_workers=8) as pool:
            t0 = time.perf_counter()
            futs = [pool.submit(len, cand_pg[q:q + 65536]) for q in range(0, n, 65536)]
            for f in futs:
                f.result()
            floor = time.perf_counter() - t0
        dropin = {"engine": engine, "host_memory": "pageable numpy", "batch_pairs": 65536, "unit": "Mpps",
                  "h2d_bytes_per_step": 8 * n, "runs": runs,
                  "python_executor_floor_8_threads": {"us_per_batch": floor / len(futs) * 1e6, "mpps": n / floor / 1e6}}
        del cand_pg, opp_pg
    log("end-to-end timing done")
    # -- row N1: the same window as raw 12-byte trace records through DetectionEngine (record decode,
    #    windowing, late drop and direction split fused into the scan).  Two windows, 1% late records.
    rec_stats = None
    if world == 1 and not args.no_records and args.config == 2:
        wsec = 300
        half = n // 2
        gen2 = torch.Generator(device=dev)
        gen2.manual_seed(args.seed + 7)
        ts = torch.randint(7 * wsec, 8 * wsec, (n,), device=dev, generator=gen2, dtype=torch.int32)
        ts[half:] += wsec
        late = torch.rand(n - half, device=dev, generator=gen2) < 0.01
        ts[half:][late] -= wsec                      # stamped in window 7 but arriving during window 8: dropped

        def bswap(x):                                # host order -> network order, as captures deliver addresses
            x = x.to(torch.int64) & 0xFFFFFFFF
            y = ((x & 0xFF) << 24) | ((x & 0xFF00) << 8) | ((x >> 8) & 0xFF00) | ((x >> 24) & 0xFF)
            return (y - ((y >> 31) << 32)).to(torch.int32)

        rec_dev = torch.empty((n, 3), dtype=torch.int32, device=dev)
        rec_dev[:, 0] = ts
        rec_dev[:, 1] = bswap(cand_d)
        rec_dev[:, 2] = bswap(opp_d)
        n_late = int(late.sum().item())
        del ts, late
        raw_dev = rec_dev.view(torch.uint8).reshape(-1)
        eng = P.DetectionEngine(P.WindowConfig(theta=THETA, window_seconds=wsec), device=local_rank)
        for _ in range(2):
            res = eng.run(raw_dev)
        ok = [r.window_id for r in res] == [7, 8] and res[0].pairs == half and \
            res[1].pairs == n - half - n_late and res[1].dropped == n_late
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        r0.record(stream)
        for _ in range(args.steps):
            res = eng.run(raw_dev)
        r1.record(stream)
        torch.cuda.synchronize()
        rec_ms = r0.elapsed_time(r1) / args.steps
        rec_stats = {"device_resident_mpps": n / (rec_ms * 1e-3) / 1e6, "ms_per_step": rec_ms,
                     "bytes_per_packet": 12, "windows": len(res), "late_dropped": n_late,
                     "counts_match": bool(ok), "superpoints_per_window": [len(r.reports) for r in res]}
        if not args.no_e2e and n <= 200_000_000:
            rec_h = torch.empty(n * 12, dtype=torch.uint8, pin_memory=True)
            rec_h.copy_(raw_dev)
            torch.cuda.synchronize()
            rec_np = rec_h.numpy()
            eng.run(rec_np)
            torch.cuda.synchronize()
            r0.record(stream)
            for _ in range(args.steps):
                res = eng.run(rec_np)
            r1.record(stream)
            torch.cuda.synchronize()
            ms = r0.elapsed_time(r1) / args.steps
            rec_stats["e2e_mpps"] = n / (ms * 1e-3) / 1e6
            rec_stats["e2e_ms_per_step"] = ms
            rec_stats["e2e_h2d_bytes_per_step"] = 12 * n
            del rec_h
        del rec_dev, raw_dev

    log("records path done")
    clocks.__exit__(None, None, None)
    # -- max over ranks
    stats = torch.tensor([ms_total, scan_ms, readout_ms, e2e[0] if e2e else 0.0, reset_ms],
                         device="cpu" if same_device else dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    ms_total, scan_ms, readout_ms, e2e_ms, reset_ms = (float(v) for v in stats.tolist())

    if rank == 0:
        peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(peaks_path):
            peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        else:
            peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
        achieved = 8.0 * n / (scan_ms * 1e-3) / 1e9
        kernel = "k_scan_flowcache<5>" if args.scan_mode in ("flow_cache", "auto") else \
            f"k_scan_vec4<5,{P.dhla.SCAN_MODES[args.scan_mode]}>"
        roofline = {
            "bound": "hbm", "kernel": kernel,
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": peak_src, "algorithmic_bytes_per_packet": 8,
            "launch_ms": scan_ms, "packets_per_launch": n, "scan_gpps": n / (scan_ms * 1e-3) / 1e9,
            "traffic": args.traffic_bytes,
        }
        if roofline["traffic"] is None:
            # dram__bytes_read.sum + dram__bytes_write.sum of one 100M-packet launch, from the committed ncu capture
            for tag in ("r02", "r01"):            # the newest committed capture of this kernel
                tpath = os.path.join(ROOT, "profiles", f"{tag}_traffic.json")
                if not (os.path.exists(tpath) and n == 100_000_000):
                    continue
                table = json.load(open(tpath))
                entry = table.get(kernel.split(",")[0] + (",2>" if "vec4" in kernel else ""), None) or table.get(kernel)
                if entry:
                    roofline["traffic"] = entry["dram_bytes_per_launch"]
                    roofline["traffic_source"] = f"profiles/{tag}_traffic.json (ncu --set full)"
                    break
        if l2:
            roofline["l2_probe"] = l2
        # The ceiling that actually binds (north star: the slower of HBM streaming and the sketch's L2
        # traffic).  ncu shows the scan limited by the SM's L1-miss request port -- one request per clock
        # per SM -- not by DRAM.  Requests and REDs per packet come from the committed ncu capture of this
        # kernel on this workload (profiles/r02_scan_counters.json, written by tools/ncu_counters.py from
        # lts__t_requests_srcunit_tex / lts__t_sectors_srcunit_tex_op_red / sm__cycles_elapsed), never
        # from a hand-set constant; the port rate is SMs x the SM clock sampled during this run.
        roofline["hbm_ceiling_gpps"] = peak / 8.0
        cpath = os.path.join(ROOT, "profiles", "r02_scan_counters.json")
        ctr = json.load(open(cpath)).get(kernel) if os.path.exists(cpath) else None
        clk = clocks.summary()
        if ctr and n == ctr.get("packets_per_launch") and clk.get("sm_mhz"):
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            port = sms * clk["sm_mhz"] * 1e6 / 1e9                       # G requests/s the SMs can issue
            req = ctr["l2_requests_per_packet"]
            roofline["request_port_gps"] = port
            roofline["l2_requests_per_packet"] = req
            roofline["l2_red_per_packet"] = ctr["l2_red_per_packet"]
            roofline["request_ceiling_gpps"] = port / req
            if l2 and ctr["l2_red_per_packet"] > 0:
                roofline["atomic_ceiling_gpps"] = l2["red_gops"] / ctr["l2_red_per_packet"]
            ceilings = [roofline[k] for k in ("hbm_ceiling_gpps", "request_ceiling_gpps", "atomic_ceiling_gpps")
                        if k in roofline]
            roofline["binding_ceiling_gpps"] = min(ceilings)
            roofline["frac_of_binding_ceiling"] = roofline["scan_gpps"] / roofline["binding_ceiling_gpps"]
            roofline["ncu"] = {k: ctr[k] for k in ("request_port_busy_pct", "lts_throughput_pct", "dram_throughput_pct",
                                                     "source") if k in ctr}
        value = n_total * args.steps / (ms_total * 1e-3) / 1e6
        workload = WORKLOAD if args.config == 2 else (
            f"config3: ONE {n_total}-packet window (config 2's flow population, {n_total // flows} packets per flow) "
            f"split over {world} GPU(s) by packet slices, generated on the device, OR-merged, theta 1024")
        line = {
            "metric": "packets/sec per detection window (scan+estimate+restore)",
            "value": value, "unit": "Mpps", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_total / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.config == 2 else "strong",
            "vs_baseline": None, "dtype": "u32/u64 integer hashing + f64 estimates", "data": "synthetic",
            "config": {"workload": workload, "packets_per_gpu": n, "window_packets": n_total if args.config == 3 else n,
                       "distinct_flows": flows, "theta": THETA,
                       "scan_mode": args.scan_mode, "scan_kernel_used": sk.scan_mode_used, "merge": win.merged_with,
                       "pipeline": ("none: every window waits for its reports (--no-pipeline)" if args.no_pipeline else
                                    "reports of window k collected after window k+1's reset+scan are queued "
                                    "(restore_begin/_end); every window's reports are read back"),
                       "flow_cache": ({"mib": args.flow_cache_mib,
                                       "hit_rate": (fc_hits / fc_lookups) if fc_lookups else None}
                                      if args.scan_mode in ("flow_cache", "auto") else None),
                       "l2": f"inputs ({8 * n / 1e6:.0f} MB per GPU) larger than L2; sketch (10 MiB) L2-resident by design"},
            "phase_ms": {"reset": reset_ms, "scan": scan_ms, "merge+estimate+restore+filter": readout_ms},
            "roofline": roofline,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        if parity:
            line["parity"] = parity
        if rec_stats:
            line["records_path"] = rec_stats
        if e2e:
            # one copy per read-out: control block + window counters + the first 256 report rows
            reports_bytes = READBACK_BYTES
            line["e2e"] = {"value": n_total * args.steps / (e2e_ms * 1e-3) / 1e6, "unit": "Mpps",
                           "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": reports_bytes,
                           "ms_per_step": e2e_ms / args.steps}
        if dropin:
            line["e2e_dropin"] = dropin
        if world == 1 and not args.no_cpu_baseline:
            m = min(n, args.cpu_sample)
            cand_s = cand_d[:m].cpu().numpy().view(np.uint32)
            opp_s = opp_d[:m].cpu().numpy().view(np.uint32)
            threads = os.cpu_count() or 1
            cpu_window(cand_s[: m // 8], opp_s[: m // 8], threads)  # page in, spin up the pool
            kind, t_scan, t_all, cpu_reports = cpu_window(cand_s, opp_s, threads)
            log("cpu baseline done")
            line["cpu_baseline"] = {
                "value": m / t_all / 1e6, "unit": "Mpps", "cores": threads, "kind": kind,
                "scan_only_mpps": m / t_scan / 1e6, "restore_ms": (t_all - t_scan) * 1e3,
                "sample": (f"{'the whole window' if m == n else 'first ' + str(m) + ' packets of the window'}, {threads} threads "
                           f"sharing one sketch, batches of 65536; "
                           + ("unmodified reference package (baseline/_ref): WindowSession.feed_batch + seal + restore, "
                              "as pkg/src/dhsa/cli.py:368-382" if kind == "reference" else "oracle C port (baseline/_ref absent)")),
                "reports_equal_gpu": [(r.host, r.saturated) for r in cpu_reports] == [(r.host, r.saturated) for r in reports]
                if m == n else None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--packets", type=int, default=100_000_000, help="packets per GPU per window")
    ap.add_argument("--seed", type=int, default=100)
    ap.add_argument("--scan-mode", default="auto", choices=["red", "test", "test_agg", "flow_cache", "auto"])
    ap.add_argument("--flow-cache-mib", type=int, default=32, help="flow cache size; flow_cache mode only")
    ap.add_argument("--merge", default="auto", choices=["auto", "p2p", "partition", "allgather"])
    ap.add_argument("--cpu-sample", type=int, default=100_000_000,
                    help="packets of the window the in-run CPU baseline scans (default: the whole config-2 window)")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3],
                    help="2: 100M packets per GPU, weak scaling (default); 3: one ~1B-packet window split over the ranks")
    ap.add_argument("--window-packets", type=int, default=1_000_000_000, help="config 3: packets of the whole window")
    ap.add_argument("--no-dropin", action="store_true", help="skip the reference-engine (pageable, 65,536-pair batches) leg")
    ap.add_argument("--traffic-bytes", type=float, default=None,
                    help="dram bytes per scan launch from the committed ncu capture (profiles/)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--no-records", action="store_true", help="skip the raw-record (DetectionEngine) leg")
    ap.add_argument("--no-pipeline", action="store_true",
                    help="collect every window's reports before the next window is queued (default: one window later)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world != args.gpus and world == 1 and args.gpus > 1:
        print(json.dumps({"error": f"--gpus {args.gpus} needs torchrun with {args.gpus} ranks"}), flush=True)
        sys.exit(2)
    run_ours(args, rank, local_rank, world)


if __name__ == "__main__":
    main()
