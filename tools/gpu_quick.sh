# quick A/B: kbench <configs> over debug-bit sets and tile column blocks + a short bench line:
#   gpurun -- "bash tools/gpu_quick.sh <tag> <dbg list> <tile-cb list> <configs>"
set -u
O=gpurun_out/q${1:-1}; mkdir -p $O
timeout 300 python tools/kbench.py --configs ${4:-4,2} --dbg ${2:-0,67108864} --tile-cbs ${3:-0,16} > $O/kbench.jsonl 2> $O/kbench.err
python - "$O" <<'PY'
import json, sys
for l in open(sys.argv[1] + "/kbench.jsonl"):
    d = json.loads(l)
    if "us" in d: print(d["config"], d["dbg"], d.get("tile_cb"), round(d["us"], 3), round(d["frac"], 3))
    else: print(d["config"], {k: round(v, 2) for k, v in d.items() if "coo_convert" in k})
PY
timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench.json 2> $O/bench.err
python -c "import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['clocks'])"
