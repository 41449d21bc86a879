#!/usr/bin/env python
"""Summarise ncu captures into profiles/ (runs here, no GPU needed: `ncu -i`).

  python tools/ncu_summary.py full <report.ncu-rep> <label> [--alg-bytes N]   -> JSON on stdout
  python tools/ncu_summary.py launches <launches.csv>                         -> per-kernel table

`full` reads one `--set full` report (first kernel in it) and prints the
counters the roofline needs (duration, DRAM bytes, throughput %, hit rates,
occupancy, registers, bank conflicts).  `launches` reads a
`--metrics gpu__time_duration.sum --csv` launch list and prints the share of
each kernel in the listed time.
"""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "dram__cycles_elapsed.avg.per_second": "dram_clock_hz",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1, "second": 1, "Ghz": 1e9, "Mhz": 1e6, "hz": 1,
         "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}


def full(rep, label, alg_bytes=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"label": label, "report": rep, "kernel": vals[hdr.index("Kernel Name")]}
    for m, k in WANT.items():
        if m in hdr:
            i = hdr.index(m)
            v = vals[i].replace(",", "")
            try:
                x = float(v) * SCALE.get(units[i], 1.0)
            except ValueError:
                x = v
            res[k] = x
    if isinstance(res.get("duration"), float):
        d = res["duration"]
        rd, wr = res.get("dram_read", 0.0), res.get("dram_write", 0.0)
        res["dram_bytes_per_launch"] = rd + wr
        res["dram_gbs"] = (rd + wr) / d / 1e9
        if alg_bytes:
            res["alg_bytes_per_launch"] = alg_bytes
            res["alg_gbs_cold"] = alg_bytes / d / 1e9
            res["traffic_over_alg"] = (rd + wr) / alg_bytes
    return res


def launches(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    kn, val, unit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    mn = hdr.index("Metric Name")
    agg, dram = {}, {}
    for r in rows[1:]:
        if len(r) <= val:
            continue
        name = r[kn].split("(")[0].replace("void ", "")
        v = float(r[val].replace(",", ""))
        if r[mn] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):  # other metrics of the same launches
            dram[name] = dram.get(name, 0.0) + v * SCALE.get(r[unit], 1)
            continue
        if r[mn] != "gpu__time_duration.sum":
            continue
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * SCALE.get(r[unit], 1e-9)
    tot = sum(v[1] for v in agg.values())
    out = {k: {"launches": n, "total_us": s * 1e6, "mean_us": s / n * 1e6, "share": s / tot}
           for k, (n, s) in agg.items()}
    for k, b in dram.items():
        if k in out:
            out[k]["dram_bytes_per_launch"] = b / out[k]["launches"]
    return {"total_s": tot, "kernels": out}


if __name__ == "__main__":
    if sys.argv[1] == "full":
        ab = None
        if "--alg-bytes" in sys.argv:
            ab = float(sys.argv[sys.argv.index("--alg-bytes") + 1])
        print(json.dumps(full(sys.argv[2], sys.argv[3], ab), indent=1))
    else:
        print(json.dumps(launches(sys.argv[2]), indent=1))
