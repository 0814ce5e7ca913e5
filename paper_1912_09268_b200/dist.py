"""torch.distributed plumbing for one-process-per-GPU runs.

Rendezvous always on 127.0.0.1 (the container hostname may not resolve).
`agree_plan` is paper Algorithm 2 line 8 (Bcast(m)): every
rank solves the plan deterministically on its host and the ranks verify
they hold the identical plan by comparing a digest, failing loudly if not.
"""
from __future__ import annotations

import hashlib
import os
from typing import Optional, Tuple

import torch
import torch.distributed as dist


def env_world() -> Tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init(backend: str = "nccl", device: Optional[int] = None) -> Tuple[int, int, int]:
    rank, world, local = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        kwargs = {}
        if backend == "nccl":
            torch.cuda.set_device(local if device is None else device)
            kwargs["device_id"] = torch.device("cuda", local if device is None else device)
        dist.init_process_group(backend, rank=rank, world_size=world, **kwargs)
    return rank, world, local


def barrier() -> None:
    if dist.is_initialized():
        dist.barrier()


def max_over_ranks(x: float, device=None) -> float:
    if not dist.is_initialized():
        return x
    if device is None and dist.get_backend() == "nccl":
        device = torch.device("cuda", torch.cuda.current_device())
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def plan_digest(tags) -> str:
    return hashlib.sha256(bytes(int(t) for t in tags)).hexdigest()


def agree_plan(tags, group=None) -> str:
    """All ranks must hold the same merge plan; returns its digest."""
    digest = plan_digest(tags)
    if dist.is_initialized():
        world = dist.get_world_size(group)
        got = [None] * world
        dist.all_gather_object(got, digest, group=group)
        if any(g != digest for g in got):
            raise RuntimeError(f"merge plans differ across ranks: {got}")
    return digest
