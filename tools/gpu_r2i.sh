set -u
O=gpurun_out/r2i; mkdir -p $O
for d in 0 131072 262144 393216; do timeout -s KILL 600 python tools/gcn_bench.py --dbg $d > $O/gcn_bench_$d.jsonl 2> $O/gcn_bench_$d.err; done
(timeout 60 python tools/trace.py --config 3 --coo; timeout 60 python tools/trace.py --config 3) > $O/trace_c3.jsonl 2>&1
timeout 300 python tools/kbench.py --configs 3 > $O/kbench.jsonl 2>&1
