# steady-state phase trace (kbench --trace) of one config with and without the pre-wait prefetch:
#   gpurun -- "bash tools/gpu_pf_trace.sh <tag> <config>"
set -u
O=gpurun_out/pft${1:-1}; mkdir -p $O
timeout 300 python tools/kbench.py --configs ${2:-4} --dbg 0,16777216 --trace > $O/kbench.jsonl 2> $O/kbench.err
python - "$O" <<'PY'
import json, sys
for l in open(sys.argv[1] + "/kbench.jsonl"):
    d = json.loads(l)
    if "us" in d: print(d["config"], d["dbg"], round(d["us"], 3), json.dumps(d.get("trace")))
PY
