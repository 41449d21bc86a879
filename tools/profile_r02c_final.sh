#!/bin/bash
# Round-2 (third session) capture on one B200: gpurun -- 'bash tools/profile_r02c_final.sh'
# -> gpurun_out/prof5/ ; summarised into profiles/r02/ (files *_c).
# What changed since profile_r02b.sh: the structure-staged SDDMM for streaming
# batches, the pre-wait L2 prefetch of the tile and pipeline kernels.
set -u
O=gpurun_out/prof5
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 400 python bench.py --steps 100 --warmup 5 > $O/bench.json 2> $O/bench.err; echo bench rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_bench_c5.csv python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sddmm_struct_kernel -s 2 -c 1 \
  -o $O/full_c5_sddmm python tools/probe/sddmm_once.py > $O/ncu_sddmm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tile_kernel -s 3 -c 1 \
  -o $O/full_c4_tile python tools/kbench.py --configs 4 --ncu-mode > $O/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_csr_kernel -s 3 -c 1 \
  -o $O/full_c3_spmm python tools/kbench.py --configs 3 --ncu-mode > $O/ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_csr_kernel -s 9 -c 1 \
  -o $O/full_c3_coo python tools/kbench.py --configs 3 --ncu-mode --ncu-coo > $O/ncu_c3coo.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches_bwd_c5.csv python tools/probe/bwd_once.py 5 > $O/ncu_bwd.log 2>&1
timeout 900 python tools/kbench.py --configs 2,3,4,5 --backward --copy-baseline --coo-dbg 16777216 \
  --sddmm-dbg 134217728 --dbg 0,16777216 > $O/kbench.jsonl 2>&1
(for c in 2 3 4 5; do timeout 60 python tools/trace.py --config $c; done; timeout 60 python tools/trace.py --config 3 --coo) > $O/trace.jsonl 2>&1
bash tools/gpu_sanitize.sh
mkdir -p $O/san && cp gpurun_out/san/*.log $O/san/ 2>/dev/null
echo done
