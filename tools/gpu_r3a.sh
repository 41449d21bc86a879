set -u
O=gpurun_out/r3a; mkdir -p $O
true
timeout 300 python tools/kbench.py --configs 5 --backward --sddmm-dbg 4194304,16777216,33554432 > $O/kb.jsonl 2> $O/kb.err; tail -2 $O/kb.err
python -c "
import json
for l in open('$O/kb.jsonl'):
    d=json.loads(l); print({k:(round(v,1) if isinstance(v,float) else v) for k,v in d.items() if 'us' in k})
"
