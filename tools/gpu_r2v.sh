set -u
O=gpurun_out/r2v; mkdir -p $O
for rep in 1 2; do
for d in 0 4194304 32768 $((32768|4194304)); do timeout 120 python tools/probe/tile_balance.py --dbg $d --out $O/t_${d}_$rep.npz 2>/dev/null; done
done
