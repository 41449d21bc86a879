set -u
O=gpurun_out/r2e; mkdir -p $O
timeout -s KILL 600 python -m pytest tests/test_gpu_gcn.py -x -q > $O/pytest_gcn.log 2>&1
tail -n 30 $O/pytest_gcn.log
timeout -s KILL 600 python tools/gcn_bench.py > $O/gcn_bench.jsonl 2> $O/gcn_bench.err
tail -n 5 $O/gcn_bench.jsonl $O/gcn_bench.err
