set -u
O=gpurun_out/s1; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo smoke rc=$? >> $O/smoke.txt
timeout 400 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.txt 2>&1; tail -5 $O/pytest_gpu.txt
timeout 300 python tools/kbench.py --help > $O/kbench_help.txt 2>&1
