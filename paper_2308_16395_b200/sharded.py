"""One streamed update split across GPUs, one process per GPU.

The reference has no distributed mode; its ``stream_update``
(streaming.hpp:63, streaming.cpp:157-233) is a sequential chain over the
non-streaming modes. Sharding one slice along its LAST spatial mode
``s = d-2`` keeps every rank's slab contiguous and makes the one exchange the
compressed tensor:

* rank g holds rows ``[bounds[g], bounds[g+1])`` of mode s of every slice and
  projects modes ``0 .. s-1`` of its slab locally (``tsg_shard_begin``);
* one allgather (NCCL over NVLink / NVSwitch; gloo on CPU) moves
  ``[partial norm pairs | R_0..R_{s-1} x N_s/G local compressed tensor]`` per
  rank — for C3 (512^3, ranks 32) that is 4.2 MB in total, the same bytes as
  the allreduce of partial mode-s projections SURVEY §8(e) proposes;
* every rank assembles the identical full input of mode s from the identical
  gathered bytes and runs mode s onward, the decision and the insertion
  redundantly (``tsg_shard_continue``). All reductions over ranks run in rank
  order on those bytes, so all ranks stay bitwise identical and no factor is
  ever broadcast. Basis growth at a local mode (rare) requests one more
  allgather of that mode's input and grows redundantly.

``ShardedStreamingState`` drives the protocol over any ``comm`` with an
``allgather(send, recv)`` method; ``TorchComm`` wraps torch.distributed
(NCCL for device buffers, gloo for host buffers). ``LoopbackGroup`` runs G
virtual ranks in one process on one GPU (the exchange is a device copy), so
the sharded arithmetic can be checked on a single B200 without ranks that
wait on one another.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import streaming as S


def shard_bounds(n: int, world: int) -> list[int]:
    """Even split of n rows over `world` ranks (the first n % world get one more)."""
    if world < 1 or world > n:
        raise S.InvalidArgument(1, f"cannot split {n} rows over {world} ranks")
    base, extra = divmod(n, world)
    b = [0]
    for g in range(world):
        b.append(b[-1] + base + (1 if g < extra else 0))
    return b


def slab_of(slice_flat, slice_dims, bounds, rank):
    """Rank `rank`'s slab of a flat colexicographic slice: rows
    [bounds[rank], bounds[rank+1]) of the last spatial mode (a contiguous
    chunk; works for numpy arrays and torch tensors alike)."""
    inner = int(np.prod(slice_dims[:-1]))
    return slice_flat[bounds[rank] * inner: bounds[rank + 1] * inner]


def device_view(ptr: int, n: int, device: int):
    """Zero-copy torch view of n float64 at a device pointer owned by libtsg."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                    "data": (int(ptr), False), "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device=torch.device("cuda", device))


class TorchComm:
    """Rank-ordered allgather over torch.distributed: NCCL on CUDA tensors
    (over NVLink / NVSwitch), gloo on CPU tensors."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def allgather(self, send, recv, stream=None) -> None:
        outs = list(recv.view(self.world, -1).unbind(0))
        if stream is not None:
            import torch
            with torch.cuda.stream(stream):
                self.dist.all_gather(outs, send, group=self.group)
        else:
            self.dist.all_gather(outs, send, group=self.group)


class ShardedStreamingState(S.StreamingState):
    """A StreamingState whose updates are split over G ranks (tsg_shard_*).

    Every rank initialises with the same full batch (``init_flat``), then
    calls ``setup(rank, world)``; per slice, ``stream_update_slab(slab, comm)``
    with its slab (``slab_of``). Exported states are identical on all ranks.
    """

    def __init__(self, device: int = 0, **kw):
        kw.pop("asynchronous", None)
        super().__init__(device=device, asynchronous=False, **kw)
        self.device = device
        self.exchanges = 0
        self.exchanged_doubles = 0

    def setup(self, rank: int, world: int, bounds=None):
        if bounds is None:
            bounds = shard_bounds(self.query()["slice_dims"][-1], world)
        b = np.asarray(bounds, dtype=np.int64)
        self._check(self.L.tsg_shard_setup(self.h, rank, world, b.ctypes.data_as(S._i64p)))
        self.rank, self.world, self.bounds = rank, world, [int(v) for v in b]
        return self.bounds

    # -- protocol steps (also used by LoopbackGroup) --
    def begin(self, slab) -> S.TsgExchange:
        ex = S.TsgExchange()
        ptr, kind = S._pointer(slab)
        self._check(self.L.tsg_shard_begin(self.h, ptr, kind, C.byref(ex)))
        return ex

    def cont(self, ex: S.TsgExchange) -> S.TsgExchange:
        self._check(self.L.tsg_shard_continue(self.h, C.byref(ex)))
        return ex

    def exchange_tensors(self, ex: S.TsgExchange):
        return (device_view(ex.send, ex.count, self.device),
                device_view(ex.recv, ex.count * self.world, self.device))

    def stream_update_slab(self, slab, comm) -> None:
        """One sharded stream_update: local pass, allgather(s), redundant finish.
        The collective is enqueued on the engine's stream."""
        import torch
        stream = torch.cuda.ExternalStream(self.cuda_stream(), device=self.device)
        n, dbl = drive(self, slab, comm, stream=stream)
        self.exchanges += n
        self.exchanged_doubles += dbl


def drive(engine, slab, comm, stream=None) -> tuple[int, int]:
    """The per-slice protocol of include/tsg.h over any engine exposing
    begin / exchange_tensors / cont and any comm exposing allgather.
    Returns (exchanges, doubles gathered per rank x world)."""
    ex = engine.begin(slab)
    n = dbl = 0
    while ex.pending:
        send, recv = engine.exchange_tensors(ex)
        comm.allgather(send, recv, stream=stream)
        n += 1
        dbl += int(ex.count) * engine.world
        ex = engine.cont(ex)
    return n, dbl


class LoopbackGroup:
    """G virtual ranks in one process (each its own handle and full state on
    the same device). Each protocol step runs on every rank before the next
    one starts, and the allgather is a device copy, so no kernel ever waits
    on another rank's kernel."""

    def __init__(self, states: list):
        self.states = states

    def stream_update(self, slabs) -> None:
        import torch
        exs = [st.begin(sl) for st, sl in zip(self.states, slabs)]
        while True:
            pend = [bool(e.pending) for e in exs]
            if not any(pend):
                return
            if not all(pend) or len({int(e.count) for e in exs}) != 1:
                raise RuntimeError(f"ranks diverged: pending {pend}, counts {[e.count for e in exs]}")
            torch.cuda.synchronize()  # the local passes run on the engines' streams
            views = [st.exchange_tensors(e) for st, e in zip(self.states, exs)]
            cnt = int(exs[0].count)
            for _, recv in views:
                for g, (send, _) in enumerate(views):
                    recv[g * cnt:(g + 1) * cnt].copy_(send)
            torch.cuda.synchronize()
            exs = [st.cont(e) for st, e in zip(self.states, exs)]
