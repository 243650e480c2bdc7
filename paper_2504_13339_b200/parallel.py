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


class GradientExchange:
    """The step gradient's cross-rank exchange, bucketed and pipelined.

    The flat buffer's 19 units (class-major: one parameter component of all n Gaussians
    each) are cut into ``buckets`` contiguous ranges.  Per bucket, on the caller's stream:
    ``vegs_grad_pack`` sums the lanes' partial buffers (the Adam kernel's fixed order) into
    the payload -- the float64 step buffer itself, or a float32 copy (``payload="f32"``: half
    the NVLink bytes; the gradient is rounded once, well inside the float32 blend's own
    1e-4 tolerance) -- and an asynchronous all-reduce(sum) of that bucket is queued (NCCL
    runs it on its own stream, ordered after the pack).  Adam on bucket b
    (``vegs_adam_step_range``) waits only for bucket b's collective, so the packing of later
    buckets and Adam on earlier ones overlap the transfers.  Every rank adds the same
    all-reduced values and runs the same Adam: replicas stay bitwise identical.

    Not overlapped with the last view's backward: its projection/shading chain writes all
    19 components of every kept Gaussian, so no bucket is final before it ends."""

    def __init__(self, n: int, device, group=None, payload: str = "f64", buckets: int = 4):
        if payload not in ("f64", "f32"):
            raise ValueError(f"payload must be 'f64' or 'f32', got {payload!r}")
        self.n = int(n)
        self.group = group
        self.payload = payload
        b = max(1, min(int(buckets), 19))
        self.bounds = [(19 * k // b, 19 * (k + 1) // b) for k in range(b)]
        self.pay32 = torch.empty(19 * self.n, dtype=torch.float32, device=device) if payload == "f32" else None
        self.launches = 0
        self.collectives = 0

    def step(self, params, grads, extra, m, v, hyper, nonfinite, skip=None) -> None:
        """Pack, all-reduce and Adam, bucket by bucket (``extra``: at most 3 more lane
        buffers, added to ``grads`` in order)."""
        from .device import adam_step_range_device, grad_pack_device

        n, works = self.n, []
        for u0, u1 in self.bounds:
            grad_pack_device(grads, extra, self.pay32, n, u0, u1 - u0)
            self.launches += 1 if (self.pay32 is not None or extra) else 0
            buf = (self.pay32 if self.pay32 is not None else grads)[u0 * n:u1 * n]
            works.append(_all_reduce_async(buf, self.group))
            self.collectives += works[-1] is not None
        for (u0, u1), work in zip(self.bounds, works):
            if work is not None:
                work.wait()  # the caller's stream waits for this bucket's collective only
            adam_step_range_device(params, grads, self.pay32, m, v, n, u0, u1 - u0, hyper, nonfinite, skip)
            self.launches += 1


def _all_reduce_async(buf: torch.Tensor, group):
    if dist.is_available() and dist.is_initialized():
        return dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group, async_op=True)
    return None


def init_from_env(backend: str = "nccl") -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from torchrun's environment; initialises the
    default process group when world_size > 1."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if backend == "nccl":
            # NCCL's init lines (communicator, nranks, transport) stay in the job log unless
            # the user chose a level -- on stderr, so rank 0's JSON line stays the last line
            # of stdout
            if "NCCL_DEBUG" not in os.environ:
                os.environ["NCCL_DEBUG"] = "INFO"
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
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
