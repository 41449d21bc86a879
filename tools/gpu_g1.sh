set -u
mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1/smi.txt
timeout 300 python tools/kbench.py --configs 2,3,4 --dbg 0,16384 --copy-baseline > gpurun_out/g1/kbench.jsonl 2> gpurun_out/g1/kbench.err
(for c in 2 3 4; do timeout 60 python tools/trace.py --config $c; done) > gpurun_out/g1/trace.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/g1/pytest_parity.log 2>&1
timeout 900 python -m pytest tests/test_gpu_backward.py -x -q -k exhaustive > gpurun_out/g1/pytest_bwd.log 2>&1
tail -n 3 gpurun_out/g1/pytest_parity.log; tail -n 3 gpurun_out/g1/pytest_bwd.log
