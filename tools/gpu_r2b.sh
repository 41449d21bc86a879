set -u
O=gpurun_out/r2b; mkdir -p $O
timeout 300 python tools/kbench.py --configs 2,4 --dbg 0,16384,32768 > $O/kbench.jsonl 2> $O/kbench.err
for dbg in 0 32768; do for cb in 1 2 4 8 16 32; do timeout 200 python - <<PY >> $O/cbsweep.jsonl 2>>$O/kbench.err
import sys, json
sys.argv=['kbench']
sys.path.insert(0,'tools'); sys.path.insert(0,'.')
import torch, kbench, synth
import paper_1903_11409_b200 as bs
dev=torch.device('cuda',0)
h=bs.Handle(0)
h.set_tile_cb($cb)
h.set_debug($dbg)
for cid in (2,3,4):
    b,reps,per=kbench.setup(cid,dev)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    ms=kbench.time_calls(h,reps,200,kbench.spmm_only)
    print(json.dumps({"config":cid,"cb":$cb,"dbg":$dbg,"us":ms*1e3,"frac":per/(ms/1e3)/1e9/6554.6,"plan":h.last_plan()}))
PY
done; done
(timeout 60 python tools/trace.py --config 4; timeout 60 python tools/trace.py --config 4 --dbg 32768; timeout 60 python tools/trace.py --config 2) > $O/trace.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "configs_csr or tile" > $O/pytest_parity.log 2>&1
tail -n 3 $O/pytest_parity.log
