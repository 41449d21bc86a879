set -u
O=gpurun_out/r2y; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "coo" > $O/pytest.txt 2>&1; tail -2 $O/pytest.txt
cat > $O/cooprobe.py <<'PY'
import sys, json, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import paper_1903_11409_b200 as bs
from kbench import setup, time_calls, coo_convert_csr
dev = torch.device("cuda", 0)
b, reps, per = setup(3, dev)
h = bs.Handle(0)
h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
for w in [int(x) for x in sys.argv[1].split(",")]:
    h.set_tuning(0, w, 0, 0)
    us = [time_calls(h, reps, 200, coo_convert_csr) * 1e3 for _ in range(3)]
    print(json.dumps({"cons_warps": w, "us": [round(u, 2) for u in us], "plan": h.last_plan()["threads"]}), flush=True)
PY
timeout 300 python $O/cooprobe.py 10,12,14,16 2>&1 | tail -8
