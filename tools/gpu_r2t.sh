set -u
O=gpurun_out/r2t; mkdir -p $O
timeout 300 python tools/kbench.py --configs 4 --trace --dbg 0,4194304,25165824,41943040 > $O/kb.jsonl 2> $O/kb.err
tail -3 $O/kb.err
cat $O/kb.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'us' in d: print(d['dbg'], round(d['us'],2), d['plan']['kernel'], d['plan']['grid'], json.dumps(d.get('trace')))
"
