#!/bin/bash
# End-of-round-2 verification and capture on one B200:
#   gpurun -- 'bash tools/profile_r02_final.sh'  -> gpurun_out/final/
set -u
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.txt 2>&1; tail -1 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -1 $O/smoke.txt
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err; echo "torchrun rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err; echo "reference rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_bench_c5.csv python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_tile_kernel -s 3 -c 1 \
  -o $O/full_c4_tile_tma python tools/kbench.py --configs 4 --ncu-mode > $O/ncu_c4.log 2>&1
timeout 900 python tools/kbench.py --configs 2,3,4,5 --backward --copy-baseline --dbg 0,16777216 --coo-dbg 16777216 \
  --bwd-dbg 536870912 > $O/kbench.jsonl 2> $O/kbench.err; echo "kbench rc=$?"
(for c in 2 3 4 5; do timeout 60 python tools/trace.py --config $c; done; timeout 60 python tools/trace.py --config 3 --coo) > $O/trace.jsonl 2>&1
bash tools/gpu_checked.sh final
echo done
