set -u
O=gpurun_out/prof4; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_csr_kernel -s 5 -c 1 \
  -o $O/full_c5_spmm python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_c5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_csr_kernel -s 3 -c 1 \
  -o $O/full_c2_spmm python tools/kbench.py --configs 2 --ncu-mode > $O/ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_csr_kernel -s 3 -c 1 \
  -o $O/full_c3_spmm python tools/kbench.py --configs 3 --ncu-mode > $O/ncu_c3.log 2>&1
echo done
