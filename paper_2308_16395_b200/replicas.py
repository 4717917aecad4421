"""Multi-GPU plumbing for the streamed update: independent replicas.

This is the `--mode replicas` alternative to the sharded single stream
(`sharded.py`): each rank (one process per GPU, launched by
torchrun) owns its own stream — its own seeded slice sequence — and no
data-path collective exists. The only collectives are the benchmark's barrier
and the max/sum reductions of its timing, which this module wraps so the same
code runs over NCCL on GPUs and over gloo on CPU (tests/test_replicas.py,
world_size 2). The default multi-GPU mode is the sharded one, where a single
stream's slices are split along a spatial mode with one exchange per slice.
"""
from __future__ import annotations

import dataclasses
import os


@dataclasses.dataclass
class Group:
    world: int
    rank: int
    local: int
    backend: str | None

    @property
    def device(self) -> str:
        return "cuda" if self.backend == "nccl" else "cpu"


def init(backend: str = "nccl") -> Group:
    """Read RANK / LOCAL_RANK / WORLD_SIZE (torchrun) and join the group."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        if not dist.is_initialized():
            dist.init_process_group(backend=backend)
        return Group(world, rank, local, backend)
    return Group(1, 0, local, None)


def barrier(g: Group) -> None:
    if g.world > 1:
        import torch.distributed as dist
        dist.barrier()


def _reduce(g: Group, v: float, op: str) -> float:
    if g.world == 1:
        return float(v)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64, device=g.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def reduce_max(g: Group, v: float) -> float:
    return _reduce(g, v, "max")


def reduce_sum(g: Group, v: float) -> float:
    return _reduce(g, v, "sum")


def job_rate(g: Group, units: float, seconds: float) -> tuple[float, float]:
    """Whole-job rate: units summed over ranks / the slowest rank's time.
    Returns (rate, max_seconds)."""
    total = reduce_sum(g, units)
    tmax = reduce_max(g, seconds)
    return (total / tmax if tmax > 0 else 0.0), tmax


def stream_config(cfg, rank: int):
    """Replica `rank`'s stream: the same workload shape, its own seed."""
    return dataclasses.replace(cfg, seed=cfg.seed + 7919 * rank) if rank else cfg


def close(g: Group) -> None:
    if g.world > 1:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
