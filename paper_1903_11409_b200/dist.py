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


def finalize() -> None:
    """Tear down the process group (multi-rank runs) before exit."""
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


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


# ---- optional reassembly of the full C on every rank (SURVEY §8(e), NEXT-4b) ----
# Off the hot path.  Two implementations: the NCCL baseline (one broadcast per
# rank, in place) and the product, the multicast store fused into the SpMM
# (Handle.csr_multicast into a team buffer built by mc_team_buffer).

def row_bounds(row_off_all: np.ndarray, split: np.ndarray) -> np.ndarray:
    """Global row range of every rank: rows [b[r], b[r+1]) (contiguous shards)."""
    return np.asarray(row_off_all, dtype=np.int64)[np.asarray(split, dtype=np.int64)]


def allgather_rows(C_full: torch.Tensor, bounds, group=None) -> None:
    """NCCL/gloo baseline all-gather-v: rank r owns rows [bounds[r], bounds[r+1])
    of C_full (already computed in place); afterwards every rank holds all rows."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return
    for r in range(dist.get_world_size(group)):
        lo, hi = int(bounds[r]), int(bounds[r + 1])
        if hi > lo:
            dist.broadcast(C_full[lo:hi], src=r, group=group)


_fd_calls = [0]


def share_fd(fd: int | None, tag: str = "bspmm") -> int:
    """Pass a file descriptor from rank 0 to every local rank (SCM_RIGHTS over an
    abstract Unix socket named after MASTER_PORT).  Rank 0 passes its fd and gets
    it back; the others pass None and receive their own duplicate."""
    import socket
    import time
    rank = dist.get_rank()
    world = dist.get_world_size()
    _fd_calls[0] += 1
    name = f"\0{tag}-{os.environ.get('MASTER_ADDR', '')}-{os.environ.get('MASTER_PORT', '0')}-{_fd_calls[0]}"
    if rank == 0:
        assert fd is not None
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name)
        srv.listen(world)
        barrier()
        for _ in range(world - 1):
            conn, _ = srv.accept()
            socket.send_fds(conn, [b"f"], [fd])
            conn.close()
        srv.close()
        barrier()
        return fd
    barrier()
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    for attempt in range(200):
        try:
            cli.connect(name)
            break
        except OSError:
            time.sleep(0.01)
    _, fds, _, _ = socket.recv_fds(cli, 1, 1)
    cli.close()
    barrier()
    return fds[0]


def mc_team_buffer(shape, device: torch.device):
    """A multicast team buffer spanning every rank's GPU (one process per GPU):
    rank 0 creates and exports, the others import; all join before any binds."""
    from . import McBuffer
    world = dist.get_world_size() if (dist.is_available() and dist.is_initialized()) else 1
    if world == 1:
        return McBuffer(shape, device)
    rank = dist.get_rank()
    if rank == 0:
        buf = McBuffer(shape, device, num_devices=world, export=True, bind=False)
        share_fd(buf.fd)
    else:
        fd = share_fd(None)
        buf = McBuffer(shape, device, num_devices=world, fd=fd, bind=False)
        os.close(fd)
    barrier(device)        # every device joined the team
    buf.bind()
    barrier(device)        # every device bound before the first multicast store
    return buf


def team_barrier(device: torch.device) -> None:
    """Stream-ordered barrier after multicast stores: once it returns on every
    rank's stream, every rank's shard is visible in its own copy."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.zeros(1, device=device)
        dist.all_reduce(t)
