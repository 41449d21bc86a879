set -u
O=gpurun_out/g2; mkdir -p $O
timeout 400 python tools/kbench.py --configs 2,3,4 --dbg 0,16384 --copy-baseline --trace > $O/kbench.jsonl 2> $O/kbench.err
echo done
