set -u
O=gpurun_out/r3b; mkdir -p $O
CUDA_LAUNCH_BLOCKING=1 timeout 900 python -m pytest tests/test_gpu_backward.py -x -q -k "ring" > $O/pytest.txt 2>&1; tail -30 $O/pytest.txt | grep -E "passed|failed|Error|error|test_" | head
