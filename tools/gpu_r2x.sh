set -u
O=gpurun_out/r2x; mkdir -p $O
for cb in 2 4 8 16 32; do timeout 120 python tools/probe/tile_balance.py --config 3 --cb $cb --out $O/c3_cb$cb.npz 2>/dev/null; done
for cb in 2 4 8; do timeout 120 python tools/probe/tile_balance.py --config 3 --dbg 32768 --cb $cb --out $O/c3t_cb$cb.npz 2>/dev/null; done
timeout 120 python tools/probe/tile_balance.py --config 2 --cb 4 --out $O/c2_cb4.npz 2>/dev/null
timeout 120 python tools/probe/tile_balance.py --config 2 --cb 8 --out $O/c2_cb8.npz 2>/dev/null
