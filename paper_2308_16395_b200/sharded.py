"""One streamed update split across GPUs, one process per GPU.

The reference has no distributed mode; its ``stream_update``
(streaming.hpp:63, streaming.cpp:157-233) is a sequential chain over the
non-streaming modes. Each slice is sharded along ONE spatial mode ``s`` — by
default the largest (the last one on ties, so the slab is a contiguous chunk
and the exchange the smallest), or the one the caller names (BASELINE
configs[2]: mode 1):

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
  ever broadcast;
* basis growth at a local mode k < s: every rank forms the N_k x N_k Gram of
  its part of the residual, ONE all-reduce sums them (N_k^2 doubles), the
  eigensolve runs redundantly, ``K = W^T E`` and the remaining local modes
  stay local, and the slice continues with a fresh compressed-tensor gather
  (sthosvd.cpp:45-59, streaming.cpp:142-151 split over the ranks).

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


def default_shard_mode(slice_dims) -> int:
    """The largest spatial mode, the last one on ties (tsg_shard_setup)."""
    m = 0
    for k, n in enumerate(slice_dims):
        if n >= slice_dims[m]:
            m = k
    return m


def slab_of(slice_flat, slice_dims, bounds, rank, mode=None):
    """Rank `rank`'s slab of a flat colexicographic slice: rows
    [bounds[rank], bounds[rank+1]) of spatial mode `mode` (default: the
    default shard mode) as a flat colexicographic dense tensor. A contiguous
    view when `mode` is the last spatial mode, a copy otherwise; works for
    numpy arrays and torch tensors alike."""
    nd = len(slice_dims)
    if mode is None:
        mode = default_shard_mode(slice_dims)
    lo, hi = bounds[rank], bounds[rank + 1]
    if mode == nd - 1:
        inner = int(np.prod(slice_dims[:-1]))
        return slice_flat[lo * inner: hi * inner]
    t = slice_flat.reshape(tuple(slice_dims)[::-1])  # row-major view of the colex tensor
    ax = nd - 1 - mode
    if isinstance(slice_flat, np.ndarray):
        return np.ascontiguousarray(np.take(t, np.arange(lo, hi), axis=ax)).reshape(-1)
    return t.narrow(ax, lo, hi - lo).contiguous().reshape(-1)


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

    def allreduce(self, send, recv, stream=None) -> None:
        """recv = sum over ranks of send — the same bytes on every rank (NCCL
        and gloo all-reduce both distribute one reduced value per element)."""
        def run():
            recv.copy_(send)
            self.dist.all_reduce(recv, op=self.dist.ReduceOp.SUM, group=self.group)
        if stream is not None:
            import torch
            with torch.cuda.stream(stream):
                run()
        else:
            run()


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

    def setup(self, rank: int, world: int, bounds=None, mode=None):
        """Split mode `mode` (default: the largest spatial mode, the last one on
        ties) over `world` ranks; `bounds` defaults to an even split."""
        dims = self.query()["slice_dims"]
        if mode is None:
            mode = default_shard_mode(dims)
        if bounds is None:
            bounds = shard_bounds(dims[mode], world)
        b = np.asarray(bounds, dtype=np.int64)
        self._check(self.L.tsg_shard_setup_mode(self.h, rank, world, mode, b.ctypes.data_as(S._i64p)))
        self.rank, self.world, self.bounds, self.mode = rank, world, [int(v) for v in b], mode
        self.exchange_log = []  # (op, doubles per rank) of every exchange
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
        nrecv = ex.count if ex.op == S.XCHG_ALLREDUCE_SUM else ex.count * self.world
        if hasattr(self, "exchange_log"):
            self.exchange_log.append((int(ex.op), int(ex.count)))
        return (device_view(ex.send, ex.count, self.device),
                device_view(ex.recv, nrecv, self.device))

    def sync_exchange(self) -> None:
        """Drain the engine's stream and the device's current torch stream: used
        by drive() around a collective that is not ordered on the engine's stream."""
        import torch
        torch.cuda.ExternalStream(self.cuda_stream(), device=self.device).synchronize()
        torch.cuda.current_stream(self.device).synchronize()

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
    Returns (exchanges, doubles gathered per rank x world).

    tsg_shard_begin / tsg_shard_continue return as soon as the local pass is
    ENQUEUED on the engine's stream, so the send buffer is only valid in that
    stream's order. With ``stream`` (the engine's stream) the collective is
    ordered behind it; without one (a host-staging comm: gloo, MPI) the
    engine's stream is drained before every exchange and the collective is
    complete before the engine continues."""
    ex = engine.begin(slab)
    n = dbl = 0
    while ex.pending:
        send, recv = engine.exchange_tensors(ex)
        if stream is None:
            engine.sync_exchange()
        if getattr(ex, "op", S.XCHG_ALLGATHER) == S.XCHG_ALLREDUCE_SUM:
            comm.allreduce(send, recv, stream=stream)
        else:
            comm.allgather(send, recv, stream=stream)
        if stream is None:
            engine.sync_exchange()
        n += 1
        dbl += int(ex.count) * (1 if getattr(ex, "op", 0) == S.XCHG_ALLREDUCE_SUM else engine.world)
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
            if not all(pend) or len({(int(e.count), int(e.op)) for e in exs}) != 1:
                raise RuntimeError(f"ranks diverged: pending {pend}, "
                                   f"requests {[(e.count, e.op) for e in exs]}")
            torch.cuda.synchronize()  # the local passes run on the engines' streams
            views = [st.exchange_tensors(e) for st, e in zip(self.states, exs)]
            cnt = int(exs[0].count)
            if int(exs[0].op) == S.XCHG_ALLREDUCE_SUM:
                total = views[0][0].clone()
                for send, _ in views[1:]:   # rank order: one sum, the same bytes to every rank
                    total += send
                for _, recv in views:
                    recv.copy_(total)
            else:
                for _, recv in views:
                    for g, (send, _) in enumerate(views):
                        recv[g * cnt:(g + 1) * cnt].copy_(send)
            torch.cuda.synchronize()
            exs = [st.cont(e) for st, e in zip(self.states, exs)]
