# SDDMM A/B at C5 (kbench, steady state) + the backward parity tests
set -u
O=gpurun_out/sd${1:-1}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_backward.py -x -q > $O/pytest_bwd.txt 2>&1; tail -2 $O/pytest_bwd.txt
timeout 600 python tools/kbench.py --configs 5 --backward --sddmm-dbg ${2:-134217728,268435456} > $O/kbench.jsonl 2> $O/kbench.err
tail -1 $O/kbench.jsonl
