set -u
O=gpurun_out/r2r; mkdir -p $O
python -c "import pynvml; pynvml.nvmlInit(); print(pynvml.nvmlDeviceGetCount())" > $O/nvml.txt 2>&1
nvidia-smi --query-gpu=index,uuid,clocks.sm,clocks_event_reasons.active --format=csv >> $O/nvml.txt 2>&1
timeout 400 python bench.py --no-e2e > $O/bench.json 2> $O/bench.err; tail -c 300 $O/bench.json; cat $O/bench.err | tail -3
