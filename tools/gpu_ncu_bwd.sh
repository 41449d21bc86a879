# ncu --set full of the fused backward at C5 (tools/probe/bwd_once.py): gpurun -- "bash tools/gpu_ncu_bwd.sh <tag>"
set -u
O=gpurun_out/nbw${1:-1}; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:backward_fused -s 1 -c 1 \
  -o $O/full_c5_bwd_fused python tools/probe/bwd_once.py 5 > $O/ncu.log 2>&1; tail -2 $O/ncu.log
