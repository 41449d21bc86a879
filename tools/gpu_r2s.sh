set -u
O=gpurun_out/r2s; mkdir -p $O
timeout 300 python tools/kbench.py --configs 4 --dbg 0,4194304,25165824,41943040 > $O/kb.jsonl 2> $O/kb.err
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "colown or configs_csr or tile_shapes or tile_fallbacks or k_sweep or leading or padded or direct_path" > $O/pytest.txt 2>&1
tail -5 $O/pytest.txt; cat $O/kb.jsonl | cut -c 1-200
