# pre-wait prefetch A/B (kbench, default vs debug bit 24) + parity tests
set -u
O=gpurun_out/pf${1:-1}; mkdir -p $O
timeout 300 python tools/kbench.py --configs 4 --tile-cbs 8,16,32,8,16,32,8,16,32  > $O/kbench.jsonl 2> $O/kbench.err
python - "$O" <<'PY'
import json, sys
for l in open(sys.argv[1] + "/kbench.jsonl"):
    d = json.loads(l)
    if "us" in d: print(d["config"], d["dbg"], round(d["us"], 3), round(d["frac"], 3))
    else: print(d["config"], {k: round(v, 2) for k, v in d.items() if "coo_convert" in k})
PY
[ -n "${2:-}" ] && timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
