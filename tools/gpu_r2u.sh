set -u
O=gpurun_out/r2u; mkdir -p $O
for cb in 0 16 32; do timeout 120 python tools/probe/tile_balance.py --dbg 4194304 --cb $cb --out $O/tile_cb$cb.npz; done
timeout 120 python tools/probe/tile_balance.py --dbg $((4194304|32768)) --cb 8 --out $O/tile_cpa8.npz
timeout 120 python tools/probe/tile_balance.py --dbg $((4194304|32768)) --cb 32 --out $O/tile_cpa32.npz
