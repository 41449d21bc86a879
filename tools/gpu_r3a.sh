set -u
O=gpurun_out/r3a; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_backward.py -x -q > $O/pytest.txt 2>&1; tail -3 $O/pytest.txt
timeout 300 python tools/kbench.py --configs 5 --backward --sddmm-dbg 4194304 > $O/kb.jsonl 2> $O/kb.err; tail -2 $O/kb.err
python -c "
import json
for l in open('$O/kb.jsonl'):
    d=json.loads(l); print({k:(round(v,1) if isinstance(v,float) else v) for k,v in d.items() if 'us' in k})
"
