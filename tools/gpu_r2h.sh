set -u
O=gpurun_out/r2h; mkdir -p $O
timeout -s KILL 900 python -m pytest tests/test_gpu_gcn.py -q > $O/pytest_gcn.log 2>&1
tail -n 3 $O/pytest_gcn.log
timeout -s KILL 600 python tools/gcn_bench.py > $O/gcn_bench.jsonl 2> $O/gcn_bench.err
cat $O/gcn_bench.jsonl; tail -3 $O/gcn_bench.err
timeout -s KILL 600 ncu --set full --import-source on -k regex:gcn_fused_kernel -s 1 -c 1 -o $O/gcn_reaction100 python tools/gcn_once.py reaction100 > $O/ncu.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on -k regex:gcn_fused_kernel -s 1 -c 1 -o $O/gcn_tox21 python tools/gcn_once.py tox21 >> $O/ncu.log 2>&1
tail -3 $O/ncu.log
