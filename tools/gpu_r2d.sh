set -u
O=gpurun_out/r2d; mkdir -p $O
timeout 300 python tools/kbench.py --configs 2,3,4,5 --dbg 0,16,16384 > $O/kbench.jsonl 2> $O/kbench.err
(timeout 60 python tools/trace.py --config 4) > $O/trace.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.log 2>&1
tail -n 3 $O/pytest_parity.log
