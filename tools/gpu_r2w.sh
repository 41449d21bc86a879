set -u
O=gpurun_out/r2w; mkdir -p $O
timeout 300 python tools/kbench.py --configs 3 > $O/kb.jsonl 2> $O/kb.err
timeout 120 python tools/trace.py --config 3 --coo > $O/trace_coo.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "coo" > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt; tail -2 $O/kb.err; python -c "
import json
for l in open('$O/kb.jsonl'):
    d=json.loads(l); print({k:(round(v,2) if isinstance(v,float) else v) for k,v in d.items() if k in ('us','step_us','coo_convert_csr_us','coo_atomic_us','fused_step_us')})
"; cut -c 1-900 $O/trace_coo.jsonl | tail -1
