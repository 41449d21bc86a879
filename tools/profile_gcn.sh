#!/bin/bash
# GCN layer (NEXT-1) profile capture with the final kernel: gpurun -- 'bash tools/profile_gcn.sh'
set -u
O=gpurun_out/profgcn
mkdir -p $O
timeout 900 python tools/gcn_bench.py > $O/gcn_bench.jsonl 2> $O/gcn_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gcn_fused_kernel -s 1 -c 1 \
  -o $O/full_gcn_reaction100 python tools/gcn_once.py reaction100 > $O/ncu_gcn.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:gcn_fused_kernel -s 1 -c 1 \
  -o $O/full_gcn_big python tools/gcn_once.py big >> $O/ncu_gcn.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_gcn.csv \
  python tools/gcn_once.py big > $O/ncu_launch.log 2>&1
echo done
