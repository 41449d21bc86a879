set -u
O=gpurun_out/r2m; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_gcn.py -q -x > $O/pytest_gcn.log 2>&1
tail -n 15 $O/pytest_gcn.log
for d in 0 524288 131072 262144; do timeout -s KILL 600 python tools/gcn_bench.py --dbg $d > $O/gcn_bench_$d.jsonl 2> $O/gcn_bench_$d.err; done
cat $O/gcn_bench_0.jsonl
