# fused backward: parity tests + C5 (and C3) timing against the separate kernels (debug bit 29)
set -u
O=gpurun_out/bw${1:-1}; mkdir -p $O
[ -n "${3:-}" ] && timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_streams.py -x -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
timeout 600 python tools/kbench.py --configs ${4:-5} --backward --bwd-dbg ${2:-536870912} > $O/kbench.jsonl 2> $O/kbench.err
python - "$O" <<'PY'
import json, sys
for l in open(sys.argv[1] + "/kbench.jsonl"):
    d = json.loads(l)
    print({k: round(v, 1) for k, v in d.items() if "backward" in k or "sddmm" in k or "transpose" in k})
PY
