"""N>1 host path on CPU (gloo, world_size 2): every rank derives the same
nnz*k split (bspmm_partition), regenerates only its own graphs from per-graph
seeds, and the per-rank results reassemble into the single-process result;
max/sum-over-ranks reductions used by bench.py timing work.  The per-rank
compute here is the CPU oracle standing in for the GPU kernel (no GPU on this
box); the GPU side of sharding is covered by test_gpu_parity's shard
emulation."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cid, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    from paper_1903_11409_b200 import dist as bdist

    r, w = bdist.init("gloo")
    assert (r, w) == (rank, world)
    c = synth.CONFIGS[cid]
    n_all, z_all = synth.counts(c["kind"], c["params"], synth.BASE_SEED + cid, 0, c["batch"])
    nnz_off = np.concatenate([[0], np.cumsum(z_all)]).astype(np.int64)
    i0, i1 = bdist.shard_of(nnz_off, c["k"], rank, world)
    # every rank must agree on the split
    mine = torch.tensor([i0, i1], dtype=torch.int64)
    allr = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allr, mine)
    bounds = [tuple(int(x) for x in t) for t in allr]
    assert bounds[0][0] == 0 and bounds[-1][1] == c["batch"]
    assert all(bounds[q][1] == bounds[q + 1][0] for q in range(world - 1))
    b = synth.config(cid, i0=i0, i1=i1)
    C, _ = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    np.save(os.path.join(out_dir, f"C_{rank}.npy"), C)
    # timing reductions used by bench.py
    assert bdist.max_over_ranks(float(rank + 1)) == float(world)
    assert bdist.sum_over_ranks(1.0) == float(world)
    bdist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cid", [2, 3])
def test_two_rank_shards_reassemble(tmp_path, cid):
    import oracle
    import synth
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), cid, str(tmp_path)), nprocs=world, join=True)
    parts = [np.load(tmp_path / f"C_{r}.npy") for r in range(world)]
    full = synth.config(cid)
    C, _ = oracle.spmm(full.k, full.row_off, None, full.row_ptr, full.col, full.vals, full.B)
    assert np.array_equal(np.concatenate(parts), C)


def _reassemble_worker(rank, world, port, out_dir):
    """Optional reassembly helpers: the broadcast all-gather-v of
    C rows, and the fd hand-off used to build the multicast team buffer."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import synth
    from paper_1903_11409_b200 import dist as bdist, partition

    bdist.init("gloo")
    cid = 3
    c = synth.CONFIGS[cid]
    n_all, z_all = synth.counts(c["kind"], c["params"], synth.BASE_SEED + cid, 0, c["batch"])
    nnz_off = np.concatenate([[0], np.cumsum(z_all)]).astype(np.int64)
    row_off = np.concatenate([[0], np.cumsum(n_all)]).astype(np.int64)
    split = partition(nnz_off, c["k"], world)
    bounds = bdist.row_bounds(row_off, split)
    i0, i1 = int(split[rank]), int(split[rank + 1])
    b = synth.config(cid, i0=i0, i1=i1)
    C_full = torch.full((int(row_off[-1]), c["k"]), float("nan"))
    C_full[bounds[rank]:bounds[rank + 1]] = torch.from_numpy(
        oracle.spmm_f32(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B))
    bdist.allgather_rows(C_full, bounds)
    np.save(os.path.join(out_dir, f"full_{rank}.npy"), C_full.numpy())
    # fd hand-off: rank 0 shares a pipe's read end, writes a marker; rank 1 reads it
    if rank == 0:
        r_fd, w_fd = os.pipe()
        got = bdist.share_fd(r_fd)
        assert got == r_fd
        os.write(w_fd, b"bspmm-fd-ok")
        os.close(w_fd)
        bdist.barrier()
        os.close(r_fd)
    else:
        fd = bdist.share_fd(None)
        bdist.barrier()
        assert os.read(fd, 64) == b"bspmm-fd-ok"
        os.close(fd)
    bdist.barrier()
    dist.destroy_process_group()


def test_two_rank_reassembly_and_fd_share(tmp_path):
    import oracle
    import synth
    world = 2
    mp.spawn(_reassemble_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    full = synth.config(3)
    C = oracle.spmm_f32(full.k, full.row_off, None, full.row_ptr, full.col, full.vals, full.B)
    for r in range(world):
        got = np.load(tmp_path / f"full_{r}.npy")
        assert np.array_equal(got.view(np.uint32), C.view(np.uint32))
