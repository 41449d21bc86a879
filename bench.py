#!/usr/bin/env python
"""bench.py — Batched SpMM (arXiv 1903.11409) on B200: GFLOP/s (2*nnz*k,
PAPER.md:341) and effective HBM GB/s for BASELINE.json config 5 (batch 65536
molecule-like graphs, k=256), sharded by nnz*k over N GPUs.

A step = one pass of the whole hot path over the batch: the device
batch-offset builder (row a-1, the look-back scan kernel -- what bspmm_csr
with sizes only runs for a batch this large) + the batched CSR SpMM kernel
(rows a-3..a-6); the partition (row a-7) is computed once per job on the host.  Inputs (5.4 GB at N=1) are far
larger than the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "Batched SpMM GFLOP/s & effective HBM GB/s (% of B200 peak) at 1/2/4/8 GPUs"
FALLBACK_HBM_GBS = 6650.0


def alg_bytes(n_rows: int, nnz: int, k: int, batch: int) -> int:
    """Algorithmic HBM bytes of one SpMM launch: every node row
    costs 8k + 4 + 8d bytes (B row read once, C row written once, one row pointer,
    d (col, val) pairs) plus 8 B of row offset per matrix."""
    return 8 * k * n_rows + 4 * (n_rows + 1) + 8 * nnz + 8 * (batch + 1)


def offsets_bytes(batch: int) -> int:
    return 4 * batch + 8 * (batch + 1)


def pcie_roofline_ms(bytes_in: int, bytes_out: int, dev) -> float:
    """Best of 3: one pinned H2D copy of bytes_in and one D2H of bytes_out on two
    streams at once (the floor for an end-to-end step moving those bytes)."""
    import torch
    hin = torch.empty(bytes_in // 4 + 1, dtype=torch.float32).pin_memory()
    hout = torch.empty(bytes_out // 4 + 1, dtype=torch.float32).pin_memory()
    din = torch.empty_like(hin, device=dev)
    dout = torch.empty_like(hout, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    best = float("inf")
    for _ in range(3):
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        with torch.cuda.stream(s1):
            din.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)
        torch.cuda.synchronize(dev)
        best = min(best, time.perf_counter() - t)
    del hin, hout, din, dout
    torch.cuda.empty_cache()
    return best * 1e3


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class Clocks:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    (the device found by its UUID, then by index), else an `nvidia-smi -lms`
    subprocess on the same GPU."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock"}

    def __init__(self, index: int, period: float = 0.002):
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        self.source = None
        self.uuid = None
        try:
            import torch
            self.uuid = "GPU-" + str(torch.cuda.get_device_properties(index).uuid)
        except Exception:
            pass
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            dev = None
            if self.uuid:
                try:
                    dev = pynvml.nvmlDeviceGetHandleByUUID(self.uuid)
                except Exception:
                    dev = None
            if dev is None:
                dev = pynvml.nvmlDeviceGetHandleByIndex(index if pynvml.nvmlDeviceGetCount() > index else 0)
            self.dev = dev
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.dev, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self.source = "nvml"
        except Exception as e:
            print(f"bench: NVML clock sampling unavailable ({type(e).__name__}: {e}); trying nvidia-smi",
                  file=sys.stderr)
            self.ok = self._smi_probe()
        self.period = period
        self._stop = threading.Event()
        # samples are kept only while `active` is set (the timed region); the
        # thread starts before the warm-up so the sampler's first-call latency
        # is paid outside the region
        self.active = threading.Event()

    def _smi_cmd(self, extra):
        sel = ["-i", self.uuid] if self.uuid else []
        return ["nvidia-smi", *sel, "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                "--format=csv,noheader,nounits", *extra]

    def _smi_probe(self) -> bool:
        try:
            out = subprocess.run(self._smi_cmd([]), capture_output=True, text=True, timeout=20).stdout.strip()
            self.max_mhz = int(float(out.splitlines()[0].split(",")[1]))
            self.source = "nvidia-smi"
            return True
        except Exception:
            return False

    def _run(self):
        if self.source == "nvidia-smi":
            proc = subprocess.Popen(self._smi_cmd(["-lms", "20"]), stdout=subprocess.PIPE, text=True)
            try:
                for line in proc.stdout:
                    if self._stop.is_set():
                        break
                    if self.active.is_set():
                        try:
                            f = [x.strip() for x in line.split(",")]
                            self.samples.append(float(f[0]))
                            self.reasons |= int(f[2], 16)
                        except Exception:
                            pass
            finally:
                proc.kill()
            return
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.dev, nv.NVML_CLOCK_SM)
                why = int(get_r(self.dev))
                if self.active.is_set():
                    self.samples.append(mhz)
                    self.reasons |= why
            except Exception as e:
                if not getattr(self, "_warned", False):
                    print(f"bench: NVML sample failed ({type(e).__name__}: {e})", file=sys.stderr)
                    self._warned = True
            time.sleep(self.period)

    def sample_now(self):
        """One synchronous sample from the calling thread (the timed region's own
        poll loop: it does not depend on the sampler thread being scheduled)."""
        if not self.ok or self.source != "nvml" or not self.active.is_set():
            return
        try:
            nv = self.nv
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            mhz = nv.nvmlDeviceGetClockInfo(self.dev, nv.NVML_CLOCK_SM)
            why = int(get_r(self.dev))
            self.samples.append(mhz)
            self.reasons |= why
        except Exception:
            pass

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join(timeout=5)

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["clock-sampling-unavailable"],
                    "samples": 0, "source": self.source}
        names = [v for b, v in self.REASONS.items() if self.reasons & b and b != 0x1]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples), "source": self.source}


def cpu_baseline(b, budget_s: float = 12.0):
    """The oracle (oracle/, fp64 loops, OpenMP across matrices) as it stands, on a
    bounded prefix of this rank's graphs, on the host cores."""
    import oracle
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    ncal = min(b.batch, 512)
    def run(nb):
        g1 = int(b.row_off[nb])
        z1 = int(b.row_ptr[g1])
        t0 = time.perf_counter()
        oracle.spmm(b.k, b.row_off[:nb + 1], None, b.row_ptr[:g1 + 1], b.col[:z1], b.vals[:z1], b.B[:g1])
        return time.perf_counter() - t0, 2.0 * z1 * b.k
    dt, _ = run(ncal)
    nb = int(min(b.batch, max(ncal, ncal * budget_s / max(dt, 1e-6))))
    # repeat the bounded sample until ~budget_s of CPU work has been timed
    tot, fl_tot, reps = 0.0, 0.0, 0
    while tot < budget_s and reps < 100:
        dt, fl = run(nb)
        tot += dt
        fl_tot += fl
        reps += 1
    return {"value": fl_tot / tot / 1e9, "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"first {nb} of {b.batch} graphs of the rank-0 shard (config 5) x {reps} runs, "
                      f"fp64 oracle.spmm (OpenMP over matrices), {tot:.1f} s",
            "cpu_model": cpu_model(), "runs": reps,
            "one_thread_configs_1_4": oracle_one_thread()}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


_ONE_THREAD = r"""
import json, sys, time
import numpy as np
sys.path.insert(0, sys.argv[1])
import oracle, synth
out = {}
for cid in (1, 2, 3, 4):
    b = synth.config(cid)
    ts = []
    for _ in range(int(sys.argv[2])):
        t = time.perf_counter()
        oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
        ts.append(time.perf_counter() - t)
    fl = 2.0 * b.n_nnz * b.k
    out["c%d" % cid] = {"mean_ms": 1e3 * float(np.mean(ts)), "median_ms": 1e3 * float(np.median(ts)),
                        "runs": len(ts), "gflops_mean": fl / float(np.mean(ts)) / 1e9}
print(json.dumps(out))
"""


def oracle_one_thread(runs: int = 10) -> dict:
    """The oracle on ONE host thread (OMP_NUM_THREADS=1, a fresh process) over the
    full configs 1-4: mean and median of `runs` executions each (the paper's
    protocol is the mean of 10)."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    try:
        r = subprocess.run([sys.executable, "-c", _ONE_THREAD, ROOT, str(runs)], env=env, capture_output=True,
                           text=True, timeout=300)
        return json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as e:  # reported, never fatal for the bench line
        return {"error": f"{type(e).__name__}: {e}"}


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    cid = args.config
    c = synth.CONFIGS[cid]
    cores = len(os.sched_getaffinity(0))
    # bounded sample per step: a fixed prefix of the batch, ~0.25 s of oracle work
    b = synth.config(cid, i0=0, i1=min(c["batch"], 2048))
    nb = b.batch
    def step():
        oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    t0 = time.perf_counter()
    step()
    one = time.perf_counter() - t0
    if one > 0:
        nb = max(16, min(b.batch, int(b.batch * 0.25 / one)))
    g1 = int(b.row_off[nb]); z1 = int(b.row_ptr[g1])
    ro, rp, col, vals, B = b.row_off[:nb + 1], b.row_ptr[:g1 + 1], b.col[:z1], b.vals[:z1], b.B[:g1]
    def step():
        oracle.spmm(b.k, ro, None, rp, col, vals, B)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    flops = 2.0 * z1 * b.k
    val = flops / dt / 1e9
    sample = f"first {nb} graphs of config {cid} per step (fp64 oracle.spmm, OpenMP over matrices)"
    out = {"metric": METRIC, "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": {"workload": synth.CONFIG_NAMES[cid], "global_batch": c["batch"], "k": c["k"],
                      "parallelism": "cpu-oracle"},
           "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": sample,
                            "cpu_model": cpu_model()},
           "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def load_traffic(cid: int):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            e = d.get(f"c{cid}")
            if e and e.get("dram_bytes_per_launch"):
                return float(e["dram_bytes_per_launch"]), e.get("source", p)
        except Exception:
            pass
    return None, None


class ShardPlan:
    """Row a-7 for one rank: the job's graphs, their split and this rank's range.

    strong scaling: the config's batch is split into contiguous nnz*k-balanced
    ranges (bspmm_partition, identical on every rank); weak: rank r owns graphs
    [r*batch, (r+1)*batch) of the seeded stream (the job has world*batch graphs)."""

    def __init__(self, cid: int, world: int, rank: int, scaling: str, partition_fn):
        c = synth.CONFIGS[cid]
        self.cid, self.world, self.rank, self.scaling = cid, world, rank, scaling
        self.kind, self.params, self.k = c["kind"], c["params"], c["k"]
        self.seed = synth.BASE_SEED + cid
        self.gbatch = c["batch"] * (world if scaling == "weak" else 1)
        n_all, z_all = synth.counts(self.kind, self.params, self.seed, 0, self.gbatch)
        self.nnz_off_all = np.zeros(self.gbatch + 1, np.int64)
        np.cumsum(z_all, out=self.nnz_off_all[1:])
        self.row_off_all = np.zeros(self.gbatch + 1, np.int64)
        np.cumsum(n_all, out=self.row_off_all[1:])
        if scaling == "weak":
            self.split = np.arange(world + 1, dtype=np.int64) * c["batch"]
        else:
            self.split = np.asarray(partition_fn(self.nnz_off_all, self.k, world), dtype=np.int64)
        self.i0, self.i1 = int(self.split[rank]), int(self.split[rank + 1])
        self.n_total = int(self.row_off_all[-1])
        self.nnz_total = int(self.nnz_off_all[-1])

    def rank_batch(self):
        """This rank's graphs, regenerated alone from their per-graph seeds."""
        return synth.generate(self.kind, self.params, self.gbatch, self.k, self.seed, i0=self.i0, i1=self.i1)

    def row_bounds(self) -> np.ndarray:
        return self.row_off_all[self.split]

    def flops(self) -> float:
        return 2.0 * self.nnz_total * self.k

    def step_bytes(self) -> int:
        return alg_bytes(self.n_total, self.nnz_total, self.k, self.gbatch) + offsets_bytes(self.gbatch)


def job_timing(ms_rank: float, spmm_ms_rank: float, max_fn):
    """Whole-job step time and SpMM time: the max over ranks (the slowest rank
    finishes the job)."""
    return max_fn(ms_rank), max_fn(spmm_ms_rank)


def make_report(sp: ShardPlan, ms: float, steps: int, warmup: int, peak: float, **extra) -> dict:
    """The bench JSON line (rank 0): whole-job GFLOP/s over all ranks' graphs."""
    value = sp.flops() / (ms / 1e3) / 1e9
    hbm_gbs = sp.step_bytes() / (ms / 1e3) / 1e9
    out = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": sp.world, "steps": steps,
        "warmup": warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": sp.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded G-mol graphs, U[-1,1) values)",
        "config": {"workload": synth.CONFIG_NAMES[sp.cid], "global_batch": sp.gbatch, "k": sp.k,
                   "rows": sp.n_total, "nnz": sp.nnz_total,
                   "parallelism": (f"batch-sharded x{sp.world} (nnz*k split)" if sp.scaling == "strong"
                                   else f"x{sp.world} independent batches"),
                   "l2": "inputs larger than L2 (no flush needed)"},
        "hbm_gbs": hbm_gbs, "hbm_frac_of_measured": hbm_gbs / peak,
    }
    cfg_extra = extra.pop("config_extra", {})
    out["config"].update(cfg_extra)
    out.update(extra)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="bspmm", choices=["bspmm", "reference"])
    ap.add_argument("--config", type=int, default=5, help="BASELINE.json config id (bench line: 5)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--kt", type=int, default=0)
    ap.add_argument("--warps", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--chunks", type=int, default=0)
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the config's batch is sharded over the N GPUs (BASELINE config 5); "
                         "weak: every rank runs a full batch of its own graphs")
    ap.add_argument("--allgather", choices=["none", "nccl", "multicast"], default="none",
                    help="optional reassembly of the full C on every GPU inside the step (off the hot path): "
                         "NCCL broadcasts, or the multimem store fused into the SpMM (NEXT-4b)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_1903_11409_b200 as bs
    from paper_1903_11409_b200 import dist as bdist

    rank, world, local = bdist.env_world()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    bdist.init("nccl", dev)
    assert world == args.gpus or world == 1, "--gpus must match WORLD_SIZE"

    cid = args.config
    # a-7: every rank computes the same split from the per-graph nnz counts
    sp = ShardPlan(cid, world, rank, args.scaling, bs.partition)
    b = sp.rank_batch()
    k = b.k
    gbatch = sp.gbatch
    h = bs.Handle(dev)
    h.set_hints(int(b.sizes.max()) if b.batch else 0, int(b.nnz.max()) if b.batch else 0)
    if args.kt or args.warps or args.ctas or args.chunks:
        h.set_tuning(args.kt, args.warps, args.ctas, args.chunks)

    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    sizes, row_ptr, col, vals, B = T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B)
    ro = torch.empty(b.batch + 1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    bounds = sp.row_bounds()
    row_base = int(bounds[rank])
    mcbuf, C_full = None, None
    if args.allgather == "multicast":
        mcbuf = bdist.mc_team_buffer((sp.n_total, k), dev)
        C = mcbuf.uc[row_base:row_base + b.n_rows]
    elif args.allgather == "nccl":
        C_full = torch.empty((sp.n_total, k), dtype=torch.float32, device=dev)
        C = C_full[row_base:row_base + b.n_rows]
    else:
        C = torch.empty((b.n_rows, k), dtype=torch.float32, device=dev)

    def step(ev=None):
        # what bspmm_csr(row_off=NULL, sizes) does for a batch this large, as two
        # calls so that the SpMM kernel alone can be bracketed by events
        h.build_offsets(sizes, out=ro)                    # a-1 (look-back scan kernel)
        if ev is not None:
            ev[0].record(stream)
        if mcbuf is not None:                             # a-3..a-6, C stored to every GPU
            h.csr_multicast(ro, None, row_ptr, col, vals, B, mcbuf, row_base=row_base)
        else:
            h.csr(ro, None, row_ptr, col, vals, B, C)     # a-3..a-6
        if ev is not None:
            ev[1].record(stream)
        if mcbuf is not None:
            bdist.team_barrier(dev)
        elif C_full is not None:
            bdist.allgather_rows(C_full, bounds)

    clk = Clocks(dev.index).__enter__()
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize(dev)
    plan = h.last_plan()
    K = args.steps
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = h.launch_count()
    bdist.barrier(dev)
    torch.cuda.synchronize(dev)
    clk.active.set()
    t0.record(stream)
    for s in range(K):
        step(kev[s])
    t1.record(stream)
    while not t1.query():  # the GPU is still in the timed region: sample its clocks here too
        clk.sample_now()
        time.sleep(0.002)
    torch.cuda.synchronize(dev)
    clk.active.clear()
    clk.__exit__()
    bdist.barrier(dev)
    launches = h.launch_count() - launches0
    ms_rank = t0.elapsed_time(t1) / K
    spmm_ms_rank = float(np.mean([a.elapsed_time(e) for a, e in kev]))
    ms, spmm_ms = job_timing(ms_rank, spmm_ms_rank, lambda x: bdist.max_over_ranks(x, dev))
    flops = sp.flops()
    peak, peak_src = peaks()
    # roofline of the dominant kernel on this rank (the SpMM), per launch
    spmm_bytes = alg_bytes(b.n_rows, b.n_nnz, k, b.batch)
    achieved = spmm_bytes / (spmm_ms_rank / 1e3) / 1e9
    traffic, tsrc = load_traffic(cid) if world == 1 else (None, None)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "spmm_csr_kernel", "alg_bytes_per_launch": spmm_bytes,
            "launch_ms": spmm_ms_rank, "peak_source": peak_src, "traffic_source": tsrc,
            "share_of_step": spmm_ms_rank / ms_rank}

    # e2e through the public API on HOST buffers (pinned): H2D inputs + D2H C inside the region
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hs, hrp, hc, hv, hB = pin(b.sizes), pin(b.row_ptr), pin(b.col), pin(b.vals), pin(b.B)
        hC = torch.empty((b.n_rows, k), dtype=torch.float32).pin_memory()
        del C, B, C_full
        if mcbuf is not None:
            mcbuf.close()
        torch.cuda.empty_cache()
        h.csr_host(hs, hrp, hc, hv, hB, hC)              # warm-up (allocates the device mirror)
        bdist.barrier(dev)
        t = time.perf_counter()
        for _ in range(args.e2e_steps):
            h.csr_host(hs, hrp, hc, hv, hB, hC)
        e2e_s = (time.perf_counter() - t) / args.e2e_steps
        e2e_s = bdist.max_over_ranks(e2e_s, dev)
        h2d = bdist.sum_over_ranks(hs.numel() * 4 + hrp.numel() * 4 + hc.numel() * 4 + hv.numel() * 4 +
                                   hB.numel() * 4, dev)
        d2h = bdist.sum_over_ranks(hC.numel() * 4, dev)
        e2e = {"value": flops / e2e_s / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_s * 1e3,
               "path": "bspmm_csr_host (pinned host buffers, chunked H2D/compute/D2H overlap)"}
        # PCIe roofline of this leg: the same bytes as raw pinned copies, both directions at once
        pc = pcie_roofline_ms(hs.numel() * 4 + hrp.numel() * 4 + hc.numel() * 4 + hv.numel() * 4 + hB.numel() * 4,
                              hC.numel() * 4, dev)
        e2e["pcie_roofline_ms"] = pc
        e2e["frac_of_pcie_roofline"] = pc / (e2e_s * 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(b)

    if rank == 0:
        out = make_report(sp, ms, K, args.warmup, peak, roofline=roof, cpu_baseline=cpu, e2e=e2e,
                          gpu_launches=int(launches), clocks=clk.summary(),
                          config_extra={"allgather": args.allgather, "plan": plan})
        print(json.dumps(out), flush=True)
    bdist.barrier(dev)
    bdist.finalize()


if __name__ == "__main__":
    main()
