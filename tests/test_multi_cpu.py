"""world_size-2 (and 3) gloo runs of the multi-GPU merge choreography on CPU.

The collective code under test is the product's own (paper_1803_11449_b200.multi:
byte_ranges, packet_slice, merge_p2p, merge_allgather).  Only the per-sketch
primitives are stood in for: host sketches from the oracle, with "peer memory"
as np.memmap files, so the handle exchange, range arithmetic, barrier order and
the reduce-scatter + all-gather structure run exactly as on GPUs.
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_11449_b200 import ConfigError
from paper_1803_11449_b200.multi import (byte_ranges, merge_allgather, merge_p2p, merge_partitioned, packet_slice,
                                         partition_ranges)

from oracle import oracle as O

TOY = dict(r=4, g=64, k=8, alpha=4, key_width=16)


def test_byte_ranges_cover_exactly_once_and_align():
    for nbytes in (16, 8192, 10_485_760, 48):
        for world in (1, 2, 3, 4, 8):
            rs = byte_ranges(nbytes, world)
            assert len(rs) == world and rs[0][0] == 0 and rs[-1][1] == nbytes
            for (lo, hi), (lo2, _) in zip(rs[:-1], rs[1:]):
                assert hi == lo2
            assert all(lo % 16 == 0 and hi % 16 == 0 and lo <= hi for lo, hi in rs)
    with pytest.raises(ConfigError):
        byte_ranges(100, 2)
    with pytest.raises(ConfigError):
        byte_ranges(64, 0)


def test_packet_slices_partition_the_window():
    for n in (0, 1, 5, 1000, 100_000_001):
        for world in (1, 2, 4, 8):
            cuts = [packet_slice(n, r, world) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == n
            for (lo, hi), (lo2, _) in zip(cuts[:-1], cuts[1:]):
                assert hi == lo2 and lo % 4 == 0
    with pytest.raises(ConfigError):
        packet_slice(10, 2, 2)


class HostOps:
    """Host stand-in for CudaMergeOps: same methods, numpy memory."""

    COUNTERS = 256   # the device layout: [bits | window counters | zero counts] in one mapped allocation

    def __init__(self, sketch: O.OracleSketch, path: str):
        self.sketch, self.path = sketch, path
        n = sketch.bits.nbytes
        self.alloc_bytes = (n + 15) & ~15
        self.cell_bytes = sketch.bits.shape[2]
        self.ncell = sketch.bits.shape[0] * sketch.bits.shape[1]
        self.zc = np.full(self.ncell, -1, dtype=np.int32)      # -1: never counted nor gathered
        self.mem_bytes = self.alloc_bytes + self.COUNTERS + 4 * self.ncell
        self.mem = np.memmap(path, dtype=np.uint8, mode="w+", shape=(self.mem_bytes,))
        self.opened = []
        self.owners = None

    def seal(self):
        self.mem[: self.sketch.bits.nbytes] = self.sketch.bits.reshape(-1)
        self.mem[self.alloc_bytes + self.COUNTERS:] = self.zc.view(np.uint8)
        self.mem.flush()

    def _load(self):
        self.sketch.bits[:] = np.asarray(self.mem[: self.sketch.bits.nbytes]).reshape(self.sketch.bits.shape)

    def export_handle(self) -> bytes:
        return self.path.encode().ljust(64, b"\0")

    def open_handle(self, handle: bytes):
        m = np.memmap(handle.rstrip(b"\0").decode(), dtype=np.uint8, mode="r", shape=(self.mem_bytes,))
        self.opened.append(m)
        return m

    def close_handles(self):
        self.opened = []

    def or_from_peers(self, peers, lo, hi):
        flat = self.sketch.bits.reshape(-1)
        hi = min(hi, flat.size)
        for m in peers:
            flat[lo:hi] |= np.asarray(m[lo:hi])

    def copy_from_peer(self, peer, lo, hi):
        flat = self.sketch.bits.reshape(-1)
        hi = min(hi, flat.size)
        flat[lo:hi] = np.asarray(peer[lo:hi])

    # partitioned read-out
    def own_pointer(self):
        return None   # "this rank's own bits"

    def zero_counts_range(self, lo, hi):
        hi = min(hi, self.sketch.bits.nbytes)
        assert lo % self.cell_bytes == 0 and hi % self.cell_bytes == 0
        cells = self.sketch.bits.reshape(self.ncell, self.cell_bytes)[lo // self.cell_bytes: hi // self.cell_bytes]
        self.zc[lo // self.cell_bytes: hi // self.cell_bytes] = 8 * self.cell_bytes - np.unpackbits(cells, axis=1).sum(axis=1)

    def gather_zero_counts(self, peer, lo, hi):
        hi = min(hi, self.sketch.bits.nbytes)
        theirs = np.asarray(peer[self.alloc_bytes + self.COUNTERS:]).view(np.int32)
        self.zc[lo // self.cell_bytes: hi // self.cell_bytes] = theirs[lo // self.cell_bytes: hi // self.cell_bytes]

    def set_cell_owners(self, bases, cuts):
        self.owners = (list(bases), list(cuts))

    def merged_view(self) -> O.OracleSketch:
        """What a partitioned read-out sees: every cell from the rank that owns it."""
        bases, cuts = self.owners
        flat = np.empty(self.sketch.bits.nbytes, dtype=np.uint8)
        for q, base in enumerate(bases):
            lo, hi = cuts[q], min(cuts[q + 1], flat.size)
            flat[lo:hi] = self.sketch.bits.reshape(-1)[lo:hi] if base is None else np.asarray(base[lo:hi])
        return flat.reshape(self.sketch.bits.shape)

    def bits_tensor(self):
        return torch.from_numpy(self.sketch.bits.reshape(-1))

    def new_gather_buffer(self, world):
        return torch.empty((world, self.sketch.bits.nbytes), dtype=torch.uint8)

    def or_from_buffer(self, row):
        self.sketch.bits.reshape(-1)[:] |= row.numpy()


def _worker(rank, world, port, tmpdir, mode, kw, n_packets):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cand, opp = O.distinct_pairs(n_packets, 71)
        if kw.get("key_width", 32) < 32:
            cand = cand & np.uint32((1 << kw["key_width"]) - 1)
        theta = 32 if kw else 1024
        for host, fan, seed in ((0x1234, 200, 1), (0xBEEF, 150, 2)) if kw else ((0xC63A1B02, 2048, 10),):
            c2, o2 = O.plant_pairs(host, fan, seed)
            cand, opp = np.concatenate([cand, c2]), np.concatenate([opp, o2])
        order = np.random.default_rng(5).permutation(len(cand))
        cand, opp, n_packets = cand[order], opp[order], len(cand)
        lo, hi = packet_slice(n_packets, rank, world)
        sk = O.OracleSketch(**kw)
        sk.update_batch(cand[lo:hi], opp[lo:hi])
        ops = HostOps(sk, os.path.join(tmpdir, f"rank{rank}.bits"))
        if mode == "p2p":
            merge_p2p(ops, dist)
            # a second window on the same sketches: peers stay mapped (no second handle exchange)
            opened = len(ops.opened)
            extra_c, extra_o = O.distinct_pairs(500, 72 + rank)
            if kw.get("key_width", 32) < 32:
                extra_c = extra_c & np.uint32((1 << kw["key_width"]) - 1)
            sk.update_batch(extra_c, extra_o)
            merge_p2p(ops, dist)
            assert len(ops.opened) == opened == world - 1
            for q in range(world):
                ec, eo = O.distinct_pairs(500, 72 + q)
                if kw.get("key_width", 32) < 32:
                    ec = ec & np.uint32((1 << kw["key_width"]) - 1)
                cand, opp = np.concatenate([cand, ec]), np.concatenate([opp, eo])
        elif mode == "partition":
            merge_partitioned(ops, dist)
            blo, bhi = partition_ranges(ops, world)[rank]
            assert blo % ops.cell_bytes == 0 and (bhi % ops.cell_bytes == 0 or bhi == ops.alloc_bytes)
            whole = O.OracleSketch(**kw)
            whole.update_batch(cand, opp)
            # own range merged, counts of every cell gathered, cells of every range reachable through its owner
            mine = np.array_equal(sk.bits.reshape(-1)[blo:bhi], whole.bits.reshape(-1)[blo:bhi])
            counts = np.array_equal(ops.zc.reshape(whole.zero_counts().shape), whole.zero_counts())
            seen = np.array_equal(ops.merged_view(), whole.bits)
            dist.barrier()        # (ShardedWindow.restore puts this barrier behind the read-out)
            sk.bits[:] = ops.merged_view()
            assert mine and counts and seen, f"rank {rank}: partitioned merge differs ({mine}, {counts}, {seen})"
        else:
            merge_allgather(ops, dist)
        whole = O.OracleSketch(**kw)
        whole.update_batch(cand, opp)
        ok = np.array_equal(sk.bits, whole.bits)
        got = [(r.host, r.estimate) for r in sk.restore_superpoints(theta)]
        want = [(r.host, r.estimate) for r in whole.restore_superpoints(theta)]
        flags = [None] * world
        dist.all_gather_object(flags, bool(ok and got == want))
        assert all(flags), f"rank {rank}: merged sketch differs ({flags})"
        assert len(want) >= 1
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["p2p", "allgather", "partition"])
@pytest.mark.parametrize("world, kw", [(2, TOY), (3, TOY), (2, dict())])
def test_sharded_scan_and_merge_equals_single_scan(mode, world, kw):
    port = 29500 + (os.getpid() + hash((mode, world, bool(kw)))) % 2000
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, port, tmp, mode, kw, 3000 if kw else 40_000),
                 nprocs=world, join=True)
