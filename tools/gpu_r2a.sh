set -u
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 400 python tools/kbench.py --configs 2,3,4 --dbg 0,16384 --copy-baseline > $O/kbench.jsonl 2> $O/kbench.err
(for c in 2 3 4; do timeout 60 python tools/trace.py --config $c; done) > $O/trace.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
tail -n 5 $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench.log 2>&1; tail -n 2 $O/bench.log
