set -u
O=gpurun_out/r2n; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_gcn.py -q -x > $O/pytest_gcn.log 2>&1
tail -n 15 $O/pytest_gcn.log
for d in 0 1048576 2097152 3145728; do timeout -s KILL 600 python tools/gcn_bench.py --small --dbg $d > $O/gcn_bench_$d.jsonl 2> $O/gcn_bench_$d.err; done
cat $O/gcn_bench_0.jsonl
