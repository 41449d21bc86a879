"""bench.py's multi-rank logic end to end on CPU (gloo, world_size 2 and 4).

Every rank builds bench.ShardPlan (row a-7: the nnz*k split of BASELINE config
N, identical on every rank; or the weak-scaling ranges), regenerates only its
own graphs, runs its shard (the CPU oracle stands in for the GPU kernel: there
is no GPU here), and the timings go through bench.job_timing with the gloo
max-over-ranks reduction; rank 0 assembles the JSON line with
bench.make_report.  The checks: the report's totals equal the single-rank
report's (strong) or world x the batch (weak), the ranks' graphs tile the job
exactly once, the per-rank results reassemble into the single-process result,
and the whole-job value is total flops / max-over-ranks time.  No collective
touches the data path; only timings and counts are reduced."""
import json
import os
import socket
import sys
import time

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cid, scaling, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    import oracle
    from paper_1903_11409_b200 import dist as bdist, partition

    bdist.init("gloo")
    sp = bench.ShardPlan(cid, world, rank, scaling, partition)
    b = sp.rank_batch()
    t = time.perf_counter()
    C = oracle.spmm_f32(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    ms_rank = (time.perf_counter() - t) * 1e3 + 1.0 + rank      # distinct per rank
    ms, spmm_ms = bench.job_timing(ms_rank, 0.5 * ms_rank, bdist.max_over_ranks)
    nnz_sum = bdist.sum_over_ranks(float(b.n_nnz))
    rows_sum = bdist.sum_over_ranks(float(b.n_rows))
    np.save(os.path.join(out_dir, f"C_{rank}.npy"), C)
    info = {"rank": rank, "i0": sp.i0, "i1": sp.i1, "ms_rank": ms_rank, "ms": ms, "spmm_ms": spmm_ms,
            "nnz_sum": nnz_sum, "rows_sum": rows_sum, "n_nnz": b.n_nnz, "batch": b.batch,
            "split": [int(x) for x in sp.split]}
    if rank == 0:
        info["report"] = bench.make_report(sp, ms, 1, 0, 6554.6, gpu_launches=1)
    json.dump(info, open(os.path.join(out_dir, f"info_{rank}.json"), "w"))
    bdist.barrier()
    dist.destroy_process_group()


def _single_report(cid, scaling, world):
    sys.path.insert(0, ROOT)
    import bench
    from paper_1903_11409_b200 import partition
    return bench.ShardPlan(cid, 1 if scaling == "strong" else world, 0, scaling, partition)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("scaling", ["strong", "weak"])
@pytest.mark.parametrize("cid", [2, 3])
def test_bench_rank_logic(tmp_path, world, scaling, cid):
    sys.path.insert(0, ROOT)
    import oracle
    import synth

    mp.spawn(_worker, args=(world, _free_port(), cid, scaling, str(tmp_path)), nprocs=world, join=True)
    infos = [json.load(open(tmp_path / f"info_{r}.json")) for r in range(world)]
    rep = infos[0]["report"]
    c = synth.CONFIGS[cid]
    # every rank agreed on the split; the ranges tile the job's graphs once
    assert all(i["split"] == infos[0]["split"] for i in infos)
    assert infos[0]["i0"] == 0 and all(infos[r]["i1"] == infos[r + 1]["i0"] for r in range(world - 1))
    gbatch = c["batch"] * (world if scaling == "weak" else 1)
    assert infos[-1]["i1"] == gbatch and rep["config"]["global_batch"] == gbatch
    if scaling == "weak":
        assert all(i["batch"] == c["batch"] for i in infos)
    # totals: the whole job, equal to the single-rank view of the same job
    ref = _single_report(cid, scaling, world)
    assert rep["config"]["nnz"] == ref.nnz_total == int(infos[0]["nnz_sum"])
    assert rep["config"]["rows"] == ref.n_total == int(infos[0]["rows_sum"])
    assert rep["n_gpus"] == world and rep["scaling"] == scaling
    # timing: max over ranks; value = all ranks' flops / that time
    ms = max(i["ms_rank"] for i in infos)
    assert all(abs(i["ms"] - ms) < 1e-9 for i in infos)
    assert abs(rep["ms_per_step"] - ms) < 1e-9
    assert abs(rep["value"] - 2.0 * ref.nnz_total * c["k"] / (ms / 1e3) / 1e9) < 1e-9 * rep["value"]
    # the per-rank results reassemble into the single-process result
    full = synth.generate(c["kind"], c["params"], gbatch, c["k"], synth.BASE_SEED + cid)
    Cref = oracle.spmm_f32(full.k, full.row_off, None, full.row_ptr, full.col, full.vals, full.B)
    parts = np.concatenate([np.load(tmp_path / f"C_{r}.npy") for r in range(world)])
    assert np.array_equal(parts.view(np.uint32), Cref.view(np.uint32))
