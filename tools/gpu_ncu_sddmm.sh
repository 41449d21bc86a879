# ncu --set full of the standalone SDDMM at C5 (tools/probe/sddmm_once.py): gpurun -- "bash tools/gpu_ncu_sddmm.sh <tag> [dbg]"
set -u
O=gpurun_out/nsd${1:-1}; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sddmm -s 2 -c 1 \
  -o $O/full_c5_sddmm python tools/probe/sddmm_once.py --dbg ${2:-0} > $O/ncu.log 2>&1; tail -3 $O/ncu.log
