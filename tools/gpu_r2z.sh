set -u
O=gpurun_out/r2z; mkdir -p $O
timeout 120 python tools/trace.py --config 3 --coo > $O/trace_coo.jsonl 2>&1
timeout 120 python tools/trace.py --config 3 > $O/trace_csr.jsonl 2>&1
python - <<'PY'
import json
for f in ("trace_coo", "trace_csr"):
    d = json.loads(open(f"gpurun_out/r2z/{f}.jsonl").read().strip().splitlines()[-1])
    print(f, {k: v for k, v in d.items() if k not in ("plan", "config", "launch", "nostore")})
PY
