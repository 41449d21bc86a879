set -u
O=gpurun_out/g3; mkdir -p $O
timeout 400 python tools/kbench.py --configs 2,3,4 --dbg 0,16384 --trace > $O/kbench.jsonl 2> $O/kbench.err
for cb in 1 2 4 8 16 32; do timeout 200 python - <<PY >> $O/cbsweep.jsonl 2>>$O/kbench.err
import sys, json
sys.argv=['kbench']
sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import torch, kbench, synth
import paper_1903_11409_b200 as bs
dev=torch.device('cuda',0)
h=bs.Handle(0)
h.set_tile_cb($cb)
for cid in (2,3,4):
    b,reps,per=kbench.setup(cid,dev)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    ms=kbench.time_calls(h,reps,200,kbench.spmm_only)
    print(json.dumps({"config":cid,"cb":$cb,"us":ms*1e3,"frac":per/(ms/1e3)/1e9/6556.2,"plan":h.last_plan()}))
PY
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > $O/pytest_parity.log 2>&1
tail -n 3 $O/pytest_parity.log
