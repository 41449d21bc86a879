#!/bin/bash
# Round profile capture (run under gpurun on ONE B200):
#   gpurun -- 'bash tools/profile_round.sh'
# Writes gpurun_out/prof/: bench JSON, ncu launch lists, ncu --set full reports.
# Summarise here with tools/ncu_summary.py into profiles/rNN/.
set -u
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
# 1. the bench line itself (not under a profiler)
timeout 400 python bench.py --steps 100 --warmup 5 > $O/bench.json 2> $O/bench.err
# 2. launch list of the same command (cold-cache, serialised: compare shares)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_bench_c5.csv python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
  > $O/ncu_launch.log 2>&1
# 3. one full capture of the dominant kernel (and the offsets kernel) in the bench launch configuration
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_csr_kernel -s 5 -c 1 \
  -o $O/full_c5_spmm python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:offsets_kernel -s 5 -c 1 \
  -o $O/full_c5_offsets python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c5o.log 2>&1
# 4. the other configs: full capture of C4, launch lists with DRAM bytes for C2..C5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_csr_kernel -s 3 -c 1 \
  -o $O/full_c4_spmm python tools/kbench.py --configs 4 --ncu-mode > $O/ncu_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches_c2345.csv python tools/kbench.py --configs 2,3,4,5 --ncu-mode > $O/ncu_cfg.log 2>&1
# 5. steady-state kernel timings (CUDA graph, replicas > 2x L2; with the backward breakdown) and phase traces
timeout 400 python tools/kbench.py --configs 2,3,4,5 --backward --copy-baseline > $O/kbench.jsonl 2>&1
# 6. backward (NEXT-2) on C5: launch list with DRAM bytes, one full capture of the SDDMM
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches_bwd_c5.csv python tools/probe/bwd_once.py 5 > $O/ncu_bwd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sddmm_staged_kernel -s 1 -c 1 \
  -o $O/full_c5_sddmm python tools/probe/bwd_once.py 5 > $O/ncu_sddmm.log 2>&1
(for c in 2 3 4 5; do timeout 60 python tools/trace.py --config $c; done) > $O/trace.jsonl 2>&1
echo done
