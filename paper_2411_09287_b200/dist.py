"""Multi-GPU plumbing: one process per GPU, torch.distributed for control.

A batch of multiplications with its batch verification is an independent
protocol object, so the element batch is sharded: each rank runs the three
parties over its contiguous shard (weak scaling) and the only data-path
collective is the final gather of the opened outputs to rank 0 (NCCL
all-gather over NVLink; gloo in the CPU tests).  Other collectives are the
benchmark's barrier and max-over-ranks timing.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str | None = None) -> tuple[int, int, int]:
    """Join the process group; one GPU per local rank (gloo runs may
    oversubscribe GPUs for testing: local ranks wrap around the devices)."""
    rank, world, local = env()
    dev = local
    if torch.cuda.is_available() and backend == "gloo":
        dev = local % torch.cuda.device_count()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(dev)
            kw["device_id"] = torch.device("cuda", dev)
        elif torch.cuda.is_available():
            torch.cuda.set_device(dev)
        dist.init_process_group(backend, **kw)
    elif torch.cuda.is_available():
        torch.cuda.set_device(dev)
    return rank, world, dev


def _device_for_collective() -> torch.device:
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(x: float) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_device_for_collective())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_device_for_collective())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier() -> None:
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def gather_outputs(t: torch.Tensor) -> torch.Tensor:
    """Concatenate every rank's equal-length opened output shard in rank
    order (the final output reconstruction / gather of the sharded batch).
    One all-gather into a preallocated buffer; world 1 returns t itself."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return t
    world = dist.get_world_size()
    src = t.reshape(-1).contiguous()
    if dist.get_backend() == "nccl":
        if not src.is_cuda:
            src = src.cuda()
    else:
        src = src.cpu()
    out = torch.empty(world * src.numel(), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src)
    return out


def session_seed(rank: int, step: int, stream: int = 0) -> int:
    """Distinct, reproducible 128-bit session seed per (stream, rank, step):
    the three fields occupy disjoint bit ranges, so no two (rank, step)
    pairs of any stream (warm-up, timed, end-to-end, side workloads) share
    pairwise seeds or masks for step, rank < 2^32."""
    if not (0 <= rank < 1 << 32 and 0 <= step < 1 << 32 and 0 <= stream < 1 << 64):
        raise ValueError("session_seed: rank/step must be < 2^32, stream < 2^64")
    return (stream << 64) | (rank << 32) | step


def shard(n_total: int, world: int, rank: int, align: int = 1) -> tuple[int, int]:
    """Contiguous [start, stop) slice of n_total units for `rank`, slice sizes
    multiples of `align` except the last (batch sizes that keep 2^R pairs
    inside one shard)."""
    per = -(-n_total // world)
    per = -(-per // align) * align
    start = min(n_total, rank * per)
    return start, min(n_total, start + per)


def finalize() -> None:
    if dist.is_initialized():
        dist.destroy_process_group()
