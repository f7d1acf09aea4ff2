"""Multi-GPU plumbing for the sharded path.

Every (sequence, layer, KV head) tile is independent at allocate, pack and
decode time (allocate_model index = l*H_kv+h, pipeline.cpp:199-205; decode per
cache, trizone.cpp:251), so N GPUs run N independent shards with no data-path
collective. The only collectives are the timing barrier and the max-over-ranks
reduction of the step time. One process per GPU, NCCL on the box; gloo on CPU
for the tests.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    """The slice of a job one rank owns."""

    rank: int
    world: int
    first: int   # first global item (sequence or unit) of this rank
    count: int   # items on this rank

    @property
    def items(self) -> range:
        return range(self.first, self.first + self.count)


def weak_shard(per_rank: int, rank: int, world: int) -> Shard:
    """Weak scaling: every rank owns `per_rank` sequences, global ids rank*per_rank + i."""
    if per_rank < 0 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    return Shard(rank, world, rank * per_rank, per_rank)


def strong_shard(total: int, rank: int, world: int) -> Shard:
    """Strong scaling: `total` items split into contiguous, balanced ranges
    (the first total % world ranks get one extra)."""
    if total < 0 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return Shard(rank, world, first, base + (1 if rank < extra else 0))


def env_world() -> tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None) -> tuple[int, int, int]:
    """Initialise the process group when WORLD_SIZE > 1 (NCCL on GPUs)."""
    import torch

    world, rank, local = env_world()
    if world > 1:
        import torch.distributed as dist

        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            # gloo: CPU tests, or several ranks sharing one GPU (NCCL refuses two
            # ranks on one device) — rank-local GPU work on device local % count
            if torch.cuda.is_available():
                torch.cuda.set_device(local % torch.cuda.device_count())
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def _device():
    import torch
    import torch.distributed as dist

    return torch.device("cuda") if dist.get_backend() == "nccl" else torch.device("cpu")


def barrier_sync(world: int) -> None:
    """Barrier across ranks, then drain this rank's GPU work."""
    import torch

    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    if torch.cuda.is_available():
        torch.cuda.synchronize()


def max_over_ranks(x: float, world: int) -> float:
    """Step times are reported as the max over ranks (the slowest GPU bounds the job)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_partials(partial, world: int):
    """All-gather every rank's decode partials [U, g, d + 2] into [world, U, g, d + 2]
    (NCCL over NVLink on the box, gloo on CPU): the one data-path collective,
    used only by the optional sequence split."""
    import torch

    if world == 1:
        return partial.unsqueeze(0)
    import torch.distributed as dist

    out = torch.empty((world * partial.shape[0],) + tuple(partial.shape[1:]), dtype=partial.dtype,
                      device=partial.device)
    dist.all_gather_into_tensor(out, partial.contiguous())
    return out.view((world,) + tuple(partial.shape))


def sequence_split_decode(model, q, world: int, rank: int, dtype=None):
    """Optional cross-GPU merge: every rank decodes its token
    chunks of every tile (each rank holds the whole packed model), the partials
    are all-gathered and merged with a log-sum-exp combine — the strong-scaling
    path for one sequence whose tiles are long."""
    from . import pipeline as P

    part = P.decode_partial(model, q, rank, world)
    parts = gather_partials(part, world)
    return P.merge_partials(parts, dtype or q.dtype)


def finalize(world: int) -> None:
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
