"""View-sharded data parallelism.

Every rank holds a full float64 parameter replica; the views of a training step are
split into contiguous shards, each rank accumulates sum_v g_v / V_total over its shard
into the flat gradient buffer, and one all-reduce(sum) -- NCCL over NVLink on the GPU
box -- leaves the mean gradient on every rank.  Adam then runs replicated, so the
parameters stay bit-identical across ranks.  The render sweep (config 3) shards
frames the same way with no collective at all.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Contiguous, balanced shard of view indices for ``rank`` (sizes differ by <= 1)."""
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside world {world}")
    base, extra = divmod(n_views, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return list(range(lo, hi))


def allreduce_gradients(grads: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the flat gradient buffer across ranks in place (no-op for one rank)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)
    return grads


def init_from_env(backend: str = "nccl") -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from torchrun's environment; initialises the
    default process group when world_size > 1."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def local_device(local: int, backend: str = "nccl") -> int:
    """CUDA ordinal for this rank.  NCCL needs one GPU per rank; the gloo plumbing check
    (host-side collectives, no kernel waits on another rank) may fold ranks onto fewer GPUs."""
    n = torch.cuda.device_count()
    if local < n:
        return local
    if backend == "nccl":
        raise RuntimeError(f"local rank {local} but only {n} GPU(s): NCCL needs one GPU per rank")
    return local % n
