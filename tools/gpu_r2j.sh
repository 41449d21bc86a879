set -u
O=gpurun_out/r2j; mkdir -p $O
timeout 300 python tools/kbench.py --configs 2,3,4,5 > $O/kbench.jsonl 2>&1
(timeout 60 python tools/trace.py --config 3 --coo) > $O/trace_c3.jsonl 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
tail -n 5 $O/pytest_gpu.log
