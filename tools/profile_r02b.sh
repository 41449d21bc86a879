#!/bin/bash
# Round-2 (second session) profile capture (one B200): gpurun -- 'bash tools/profile_r02b.sh'
# -> gpurun_out/prof3/ ; summarised into profiles/r02/ with tools/ncu_summary.py.
# What changed since profile_r02.sh: the tile kernel stages B by cp.async (C4),
# the fused COO kernel has converter warps (C3 COO).
set -u
O=gpurun_out/prof3
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 400 python bench.py --steps 100 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_bench_c5.csv python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_csr_kernel -s 9 -c 1 \
  -o $O/full_c3_coo python tools/kbench.py --configs 3 --ncu-mode --ncu-coo > $O/ncu_c3coo.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tile_kernel -s 3 -c 1 \
  -o $O/full_c4_tile python tools/kbench.py --configs 4 --ncu-mode > $O/ncu_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches_c2345.csv python tools/kbench.py --configs 2,3,4,5 --ncu-mode --ncu-coo > $O/ncu_cfg.log 2>&1
timeout 600 python tools/kbench.py --configs 2,3,4,5 --backward --copy-baseline > $O/kbench.jsonl 2>&1
(for c in 2 3 4 5; do timeout 60 python tools/trace.py --config $c; done; timeout 60 python tools/trace.py --config 3 --coo) > $O/trace.jsonl 2>&1
echo done
