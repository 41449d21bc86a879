set -u
O=gpurun_out/r2p; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_backward.py -q -x > $O/pytest_bwd.log 2>&1
tail -n 5 $O/pytest_bwd.log
timeout 600 python tools/kbench.py --configs 5 --backward --sddmm-dbg 4194304 > $O/kbench.jsonl 2>&1
tail -n 3 $O/kbench.jsonl
