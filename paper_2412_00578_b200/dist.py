"""View-parallel multi-GPU plumbing.

The scene is replicated on every rank (each rank regenerates it from the seed); camera
views are dealt round-robin, v = rank (mod world).  Frames never communicate.  The only
collective is one all_reduce(SUM) of the float64 pruning-score vector per scoring pass
(Sec. 4.2.1: U~_i sums over all training views, P:384 / P:420), over NCCL on
NVLink; under gloo (CPU tests) the same code runs on CPU tensors.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def default_backend(world_size: int) -> str:
    """NCCL when every rank has a GPU of its own; gloo otherwise (CPU tests, or several ranks
    sharing one GPU -- NCCL refuses two ranks on one device; gloo all_reduces CUDA tensors
    through host memory)."""
    if torch.cuda.is_available() and torch.cuda.device_count() >= world_size:
        return "nccl"
    return "gloo"


def local_device(local_rank: int) -> int:
    """CUDA device of a local rank (ranks beyond the device count share devices round-robin)."""
    return local_rank % max(1, torch.cuda.device_count())


def init(backend: str | None = None) -> tuple[int, int, int]:
    rank, ws, lr = world()
    if ws > 1 and not dist.is_initialized():
        if backend is None:
            backend = default_backend(ws)
        if torch.cuda.is_available():
            torch.cuda.set_device(local_device(lr))
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        kw = {"device_id": torch.device("cuda", local_device(lr))} if backend == "nccl" else {}
        dist.init_process_group(backend=backend, rank=rank, world_size=ws, **kw)
    return rank, ws, lr


def backend() -> str | None:
    return dist.get_backend() if dist.is_available() and dist.is_initialized() else None


def views_for_rank(n_views: int, rank: int, world_size: int) -> list[int]:
    """Round-robin view shard: interleaves orbit positions so per-rank cost balances."""
    return list(range(rank, n_views, world_size))


def allreduce_scores(score: torch.Tensor) -> torch.Tensor:
    """Sum the per-rank float64 score vectors in place (the one collective of the path).
    Runs whenever a process group exists (at world size 1 too: the collective is then a copy,
    but the NCCL path is the one that executes); without one it is a no-op."""
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(score, op=dist.ReduceOp.SUM)
    return score


def accumulate_scores(score_view, n_views: int, n: int, device, rank: int | None = None,
                      world_size: int | None = None) -> torch.Tensor:
    """Score over all views: this rank's shard via score_view(v, score) (adds view v's
    U~ into score), then the all_reduce.  Every rank ends with the identical vector."""
    if rank is None or world_size is None:
        r, w, _ = world()
        rank = r if rank is None else rank
        world_size = w if world_size is None else world_size
    score = torch.zeros(n, dtype=torch.float64, device=device)
    for v in views_for_rank(n_views, rank, world_size):
        score_view(v, score)
    return allreduce_scores(score)


def max_over_ranks(x: float) -> float:
    """Max of a host float over ranks (timing: the job is as slow as its slowest rank)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return x


def barrier() -> None:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
