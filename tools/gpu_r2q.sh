set -u
O=gpurun_out/r2q; mkdir -p $O
timeout -s KILL 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
tail -n 3 $O/pytest_gpu.log
timeout -s KILL 600 python tools/gcn_bench.py > $O/gcn_bench.jsonl 2> $O/gcn_bench.err
cat $O/gcn_bench.jsonl
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
