set -u
O=gpurun_out/r2f; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_gcn.py -q > $O/pytest_gcn.log 2>&1
tail -n 40 $O/pytest_gcn.log
timeout -s KILL 600 python tools/gcn_bench.py > $O/gcn_bench.jsonl 2> $O/gcn_bench.err
tail -n 5 $O/gcn_bench.jsonl $O/gcn_bench.err
# A/B: round-1-final library vs this one on the same box (C3, C5 pipeline regression check)
(cd _ab_old && timeout 300 python tools/kbench.py --configs 3,5 > ../$O/kbench_old.jsonl 2>&1)
timeout 300 python tools/kbench.py --configs 3,5 > $O/kbench_new.jsonl 2>&1
(cd _ab_old && timeout 300 python tools/kbench.py --configs 3,5 > ../$O/kbench_old2.jsonl 2>&1)
