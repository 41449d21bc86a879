set -u
O=gpurun_out/r2c; mkdir -p $O
timeout 300 python tools/kbench.py --configs 2,4 --dbg 0,65536,16384 > $O/kbench.jsonl 2> $O/kbench.err
(timeout 60 python tools/trace.py --config 4; timeout 60 python tools/trace.py --config 4 --dbg 65536) > $O/trace.jsonl 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -n 8 $O/pytest_gpu.log
