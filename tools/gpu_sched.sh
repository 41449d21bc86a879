# balanced static schedule A/B (kbench C2-C4, default vs plain static) + GPU parity suite
set -u
O=gpurun_out/sch${1:-1}; mkdir -p $O
timeout 300 python tools/kbench.py --configs 3,2,4 --dbg 0,16777216 --coo-dbg 16777216 > $O/kbench.jsonl 2> $O/kbench.err
cat $O/kbench.jsonl | cut -c1-420
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.txt 2>&1; tail -3 $O/pytest_gpu.txt
