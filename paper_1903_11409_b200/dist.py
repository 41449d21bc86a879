"""Multi-GPU plumbing for the batch-sharded hot path (hot-path row a-7).

Graphs are independent (C is block diagonal), so ranks split the batch into
contiguous ranges with bspmm_partition (nnz*k balanced) and run bspmm_csr on
their own device with no collective on the data path.  torch.distributed is
used only for timing (max over ranks) and bookkeeping (sums).  Host logic is
backend-agnostic, so it is tested with gloo on CPU (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import os
from typing import Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import partition


def env_world() -> Tuple[int, int, int]:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init(backend: str = "nccl", device: torch.device | None = None) -> Tuple[int, int]:
    rank, world, _ = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend=backend, rank=rank, world_size=world, **kw)
    return rank, world


def shard_of(nnz_off: np.ndarray, k: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous graph range [i0, i1) of `rank` (identical on every rank: integer rule)."""
    split = partition(nnz_off, k, world)
    return int(split[rank]), int(split[rank + 1])


def _reduce(x: float, op, device) -> float:
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(x: float, device=None) -> float:
    return _reduce(x, dist.ReduceOp.MAX if dist.is_available() else None, device)


def sum_over_ranks(x: float, device=None) -> float:
    return _reduce(x, dist.ReduceOp.SUM if dist.is_available() else None, device)


def barrier(device=None):
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        if device is not None and device.type == "cuda":
            dist.barrier(device_ids=[device.index])
        else:
            dist.barrier()
