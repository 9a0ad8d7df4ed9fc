"""One detection window sharded over the GPUs of a node, one process per GPU.

The sketch is a pure function of the window's distinct pair set and merging is a
bitwise OR (/root/reference/pkg/src/dhsa/dhla.py:305-318), so the
window shards by packets with no data-path collective during the scan:

    rank p scans packets [p*N/P, (p+1)*N/P) into a private sketch
    merge:  reduce-scatter with OR  -- rank p ORs byte range p of every peer's
            sketch into its own, reading peers over NVLink through CUDA-IPC-mapped
            pointers (csrc k_or_merge; NCCL has no OR reduction)
            all-gather             -- rank p copies the merged range q from peer q
    restore runs on the merged sketch (microseconds; every rank holds the result)

or, with ``merge="partition"`` (the north star's "estimation and restore are partitioned by cell
range"): the all-gather of merged bits is replaced by

    rank p counts the zeros of ITS merged range (K2 over its own cells)
    all-gather of the zero counts   -- 4 bytes per cell instead of g/8: 327 KB instead of 10 MiB
    restore                         -- the stage chain works from the counts alone; the r cells of
                                       each surviving candidate are read from the ranks that own
                                       them, over the same peer-mapped pointers

``torch.distributed`` is plumbing only: rendezvous, the 64-byte IPC handle
exchange and barriers.  If peer mapping is unavailable the merge falls back to
``all_gather_into_tensor`` of whole sketches over NCCL followed by the local OR
kernel -- still the CUDA path, never a CPU one.

The collective choreography is written against a small ops interface so the
world_size-2 gloo tests can drive exactly this code with host buffers.
"""

from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _cabi
from .dhla import DEFAULT_MAX_CANDIDATES, Dhla
from .errors import ConfigError


def byte_ranges(nbytes: int, world: int, align: int = 16) -> List[Tuple[int, int]]:
    """Cut [0, nbytes) into `world` contiguous ranges on `align`-byte boundaries.

    nbytes is the padded allocation size (a multiple of `align`); ranges differ
    by at most one alignment unit and cover everything exactly once."""
    if world < 1:
        raise ConfigError(f"world size must be positive (got {world})")
    if nbytes % align:
        raise ConfigError(f"sketch allocation {nbytes} is not a multiple of {align} bytes")
    units = nbytes // align
    cuts = [(units * p) // world * align for p in range(world + 1)]
    return list(zip(cuts[:-1], cuts[1:]))


def packet_slice(n_packets: int, rank: int, world: int, align: int = 4) -> Tuple[int, int]:
    """Contiguous slice of a window's packets owned by `rank` (4-packet aligned so
    every rank's slice starts on a 16-byte boundary of the uint32 arrays)."""
    if not 0 <= rank < world:
        raise ConfigError(f"rank {rank} outside world of {world}")
    units = (n_packets + align - 1) // align
    lo = min(n_packets, (units * rank) // world * align)
    hi = min(n_packets, (units * (rank + 1)) // world * align)
    return lo, hi


class CudaMergeOps:
    """Merge primitives of a device sketch (the product implementation)."""

    def __init__(self, sketch: Dhla):
        self.sketch = sketch
        self._lib = _cabi.lib()
        self._opened: List[int] = []

    @property
    def alloc_bytes(self) -> int:
        return (self.sketch.memory_bytes + 15) & ~15

    def seal(self) -> None:
        self.sketch.seal()

    def stream_context(self):
        """Context manager under which torch (and NCCL, which orders its collectives with torch's
        *current* stream) works on the sketch's launch stream, so a collective is ordered behind the
        kernels already queued there and the kernels queued after it wait for it."""
        import torch

        handle = self.sketch.stream_handle
        device = f"cuda:{self.sketch.device}"
        if handle == 0:   # CUDA's legacy default stream is torch's default stream
            return torch.cuda.stream(torch.cuda.default_stream(device))
        return torch.cuda.stream(torch.cuda.ExternalStream(handle, device=device))

    def device_barrier(self, dist, group=None) -> bool:
        """Barrier across the ranks that never stops the host: a one-element NCCL all-reduce
        enqueued behind the sketch's kernels on the sketch's stream.  It completes on a rank only
        when every rank has reached it -- i.e. finished the kernels queued before it -- and the
        kernels queued after it wait for it.  False (and nothing enqueued) when the process group
        is not NCCL; the caller then falls back to seal() + dist.barrier()."""
        import torch

        if dist.get_backend(group) != "nccl":
            return False
        if getattr(self, "_token", None) is None:
            self._token = torch.zeros(1, dtype=torch.int32, device=f"cuda:{self.sketch.device}")
        with self.stream_context():
            dist.all_reduce(self._token, group=group)
        return True

    def export_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        _cabi.check(self._lib.dhsa_ipc_export(self.sketch._h, buf))
        return bytes(buf)

    def open_handle(self, handle: bytes) -> int:
        ptr = C.c_void_p()
        buf = (C.c_uint8 * 64).from_buffer_copy(handle)
        _cabi.check(self._lib.dhsa_ipc_open(self.sketch.device, buf, C.byref(ptr)))
        self._opened.append(int(ptr.value))
        return int(ptr.value)

    def close_handles(self) -> None:
        if self.sketch._h:   # the owner table points into the mappings that go away below
            self._lib.dhsa_set_cell_owners(self.sketch._h, None, None, 0)
        for ptr in self._opened:
            self._lib.dhsa_ipc_close(self.sketch.device, C.c_void_p(ptr))
        self._opened = []

    def or_from_peers(self, peer_ptrs: Sequence[int], lo: int, hi: int) -> None:
        arr = (C.c_void_p * len(peer_ptrs))(*peer_ptrs)
        _cabi.check(self._lib.dhsa_or_merge_peers(self.sketch._h, arr, len(peer_ptrs), lo, hi))

    def copy_from_peer(self, peer_ptr: int, lo: int, hi: int) -> None:
        _cabi.check(self._lib.dhsa_copy_slice_from_peer(self.sketch._h, C.c_void_p(peer_ptr), lo, hi))

    # partitioned read-out
    @property
    def cell_bytes(self) -> int:
        return self.sketch.params.g // 8

    def own_pointer(self) -> int:
        return self.sketch.bits_device_ptr

    def zero_counts_range(self, lo: int, hi: int) -> None:
        _cabi.check(self._lib.dhsa_zero_counts_range(self.sketch._h, lo, hi))

    def gather_zero_counts(self, peer_ptr: int, lo: int, hi: int) -> None:
        _cabi.check(self._lib.dhsa_gather_zero_counts_from_peer(self.sketch._h, C.c_void_p(peer_ptr), lo, hi))

    def set_cell_owners(self, ptrs: Sequence[int], cuts: Sequence[int]) -> None:
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        cut = (C.c_uint64 * len(cuts))(*cuts)
        _cabi.check(self._lib.dhsa_set_cell_owners(self.sketch._h, arr, cut, len(ptrs)))

    # all-gather fallback: whole sketch images as torch tensors on this device
    def bits_tensor(self):
        import torch

        class _View:
            pass

        v = _View()
        v.__cuda_array_interface__ = {
            "shape": (self.sketch.memory_bytes,), "typestr": "|u1",
            "data": (self.sketch.bits_device_ptr, False), "version": 2,
        }
        return torch.as_tensor(v, device=f"cuda:{self.sketch.device}")

    def new_gather_buffer(self, world: int):
        import torch

        return torch.empty((world, self.sketch.memory_bytes), dtype=torch.uint8,
                           device=f"cuda:{self.sketch.device}")

    def or_from_buffer(self, row) -> None:
        _cabi.check(self._lib.dhsa_or_merge_buffer(self.sketch._h, C.c_void_p(row.data_ptr()),
                                                   self.sketch.memory_bytes))


def peer_pointers(ops, dist, group=None) -> dict:
    """{rank: mapped sketch} of every peer.  The handle exchange and the mapping (hundreds of
    microseconds per peer) happen once per sketch -- its allocation never moves -- and are kept
    on the ops object; collective on the first call only."""
    cache = getattr(ops, "_peer_ptrs", None)
    if cache is None:
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        handles: List[Optional[bytes]] = [None] * world
        try:
            mine = ops.export_handle()
        except Exception:
            mine = None                    # still take part in the exchange: it is a collective
        dist.all_gather_object(handles, mine, group=group)
        if any(h is None for h in handles):
            raise ConfigError("a rank could not export its sketch for peer mapping")
        cache = {q: ops.open_handle(handles[q]) for q in range(world) if q != rank}
        ops._peer_ptrs = cache
    return cache


def release_peers(ops) -> None:
    ops.close_handles()
    ops._peer_ptrs = None


def _barrier(ops, dist, group=None) -> None:
    """All ranks' queued work is done before anything queued after this runs: stream-ordered on
    the device when the ops object offers it, else drain the stream and meet on the host."""
    fn = getattr(ops, "device_barrier", None)
    if fn is not None and fn(dist, group):
        return
    ops.seal()
    dist.barrier(group)


def merge_p2p(ops, dist, group=None) -> None:
    """Reduce-scatter(OR) + all-gather over peer-mapped sketches.  Collective.  With NCCL the
    three barriers are stream-ordered all-reduces, so the whole merge is enqueued without a single
    host synchronisation: [barrier][k_or_merge][barrier][k_copy_slice x (P-1)][barrier]."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world == 1:
        return
    ranges = byte_ranges(ops.alloc_bytes, world)
    ptrs = peer_pointers(ops, dist, group)
    _barrier(ops, dist, group)    # my scan has landed, and so has everyone's
    lo, hi = ranges[rank]
    ops.or_from_peers([ptrs[q] for q in sorted(ptrs)], lo, hi)
    _barrier(ops, dist, group)    # every owner's range is final
    for q in sorted(ptrs):
        ops.copy_from_peer(ptrs[q], *ranges[q])
    _barrier(ops, dist, group)    # nobody resets while a peer still reads


def partition_ranges(ops, world: int) -> List[Tuple[int, int]]:
    """Byte ranges of a partitioned read-out: as byte_ranges, cut on cell boundaries."""
    return byte_ranges(ops.alloc_bytes, world, align=max(16, ops.cell_bytes))


def merge_partitioned(ops, dist, group=None) -> None:
    """Reduce-scatter(OR), then zero counts per owner and an all-gather of the COUNTS; the merged
    bits stay where they were reduced and the read-out reads candidate cells from their owners.
    Collective.  [barrier][k_or_merge][k_zero_counts over the own range][barrier][k_copy_words x (P-1)];
    the caller puts a barrier behind the read-out (ShardedWindow.restore), because peers read this
    rank's cells until their read-out is done."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world == 1:
        return
    ranges = partition_ranges(ops, world)
    ptrs = peer_pointers(ops, dist, group)
    _barrier(ops, dist, group)    # my scan has landed, and so has everyone's
    lo, hi = ranges[rank]
    ops.or_from_peers([ptrs[q] for q in sorted(ptrs)], lo, hi)
    ops.zero_counts_range(lo, hi)
    _barrier(ops, dist, group)    # every owner's range and its counts are final
    for q in sorted(ptrs):
        ops.gather_zero_counts(ptrs[q], *ranges[q])
    bases = [ops.own_pointer() if q == rank else ptrs[q] for q in range(world)]
    ops.set_cell_owners(bases, [ranges[0][0]] + [r[1] for r in ranges])


def merge_allgather(ops, dist, group=None) -> None:
    """Fallback: NCCL all-gather of whole sketches, then the local OR kernel.  Collective.

    The collective and the gather buffer live on the sketch's launch stream (``stream_context``):
    NCCL orders a collective with the stream that is current when it is issued and nothing else, so
    issued on any other stream the OR kernels -- which run on the sketch's stream -- could read the
    buffer before NCCL has filled it."""
    import contextlib

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if world == 1:
        return
    ops.seal()
    ctx = getattr(ops, "stream_context", None)
    with (ctx() if ctx is not None else contextlib.nullcontext()):
        buf = ops.new_gather_buffer(world)
        dist.all_gather_into_tensor(buf.view(-1), ops.bits_tensor(), group=group)
        for q in range(world):
            if q != rank:
                ops.or_from_buffer(buf[q])
        ops.seal()   # the buffer goes back to the allocator only after the OR kernels have read it


class ShardedWindow:
    """A window whose packets are split over the ranks of a process group."""

    def __init__(self, params, theta: int = 1024, device: Optional[int] = None, group=None,
                 max_candidates: int = DEFAULT_MAX_CANDIDATES, merge: str = "auto"):
        import torch.distributed as dist

        if merge not in ("auto", "p2p", "partition", "allgather"):
            raise ConfigError(f"merge must be auto, p2p, partition or allgather (got {merge!r})")
        self._dist = dist
        self.group = group
        self.theta = theta
        self.max_candidates = max_candidates
        self.merge_mode = merge
        self.sketch = Dhla(params, device=device)
        self.ops = CudaMergeOps(self.sketch)
        self.merged_with = None
        self._p2p_ok: Optional[bool] = None

    @property
    def world(self) -> int:
        return self._dist.get_world_size(self.group) if self._dist.is_initialized() else 1

    def reset(self) -> None:
        self.sketch.reset()

    def scan(self, candidates, opposites) -> None:
        """This rank's slice of the window (numpy or torch CUDA tensors)."""
        self.sketch.update_batch(candidates, opposites)

    def merge(self) -> str:
        """After this every rank's sketch is the union over all ranks."""
        if self.world == 1:
            self.merged_with = "none"
            return self.merged_with
        mode = self.merge_mode
        if mode in ("auto", "p2p", "partition"):
            ok = self._try_p2p(partition=mode == "partition")
            if ok:
                self.merged_with = "partition" if mode == "partition" else "p2p"
                return self.merged_with
            if mode != "auto":
                raise ConfigError("peer-mapped merge requested but CUDA IPC mapping failed on some rank")
        merge_allgather(self.ops, self._dist, self.group)
        self.merged_with = "allgather"
        return self.merged_with

    def _try_p2p(self, partition: bool = False) -> bool:
        import torch

        dist = self._dist
        if self._p2p_ok is None:
            # Agreed once (the topology does not change between windows): every rank exchanges its
            # handle and tries to map every peer; one rank that cannot (no peer access, IPC refused
            # by the container) sends everybody to the all-gather merge.
            can = 1
            try:
                for q in range(torch.cuda.device_count()):
                    if q != self.sketch.device and not torch.cuda.can_device_access_peer(self.sketch.device, q):
                        can = 0
            except Exception:
                can = 0
            try:
                peer_pointers(self.ops, dist, self.group)      # collective exchange, local mapping
            except Exception:
                can = 0
            on_gpu = dist.get_backend(self.group) == "nccl"   # gloo rendezvous (tests) reduces on the host
            flag = torch.tensor([can], dtype=torch.int32,
                                device=f"cuda:{self.sketch.device}" if on_gpu else "cpu")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=self.group)
            self._p2p_ok = int(flag.item()) != 0
            if not self._p2p_ok:
                try:
                    release_peers(self.ops)
                except Exception:
                    pass
        if self._p2p_ok:
            (merge_partitioned if partition else merge_p2p)(self.ops, dist, self.group)
        return self._p2p_ok

    def close(self) -> None:
        """Unmap the peers' sketches (kept mapped across windows)."""
        release_peers(self.ops)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _after_readout(self) -> None:
        """Partitioned read-out: peers read this rank's cells until their read-out is done, so nobody
        goes on to the next window's reset before everybody's is queued behind a barrier."""
        if self.merged_with == "partition":
            _barrier(self.ops, self._dist, self.group)

    def restore(self):
        try:
            return self.sketch.restore_superpoints(self.theta, max_candidates=self.max_candidates)
        finally:
            self._after_readout()

    def restore_begin(self) -> None:
        """Enqueue the read-out; the next window's reset() + scan() may follow before restore_end()."""
        self.sketch.restore_superpoints_begin(self.theta, max_candidates=self.max_candidates)
        self._after_readout()

    def restore_end(self):
        return self.sketch.restore_superpoints_end()
