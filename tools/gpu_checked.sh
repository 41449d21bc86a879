# the bounds-checked build (make checked) under the GPU suite and the sanitizer workload
set -u
O=gpurun_out/chk${1:-1}; mkdir -p $O
BSPMM_LIB=checked timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu_checked.txt 2>&1; tail -3 $O/pytest_gpu_checked.txt
BSPMM_LIB=checked timeout 600 python tools/sanitize_run.py > $O/sanitize_run_checked.txt 2>&1; echo "sanitize_run rc=$?"; tail -1 $O/sanitize_run_checked.txt
BSPMM_LIB=checked timeout 600 python tools/probe/bwd_once.py 5 > $O/bwd_c5_checked.txt 2>&1; echo "bwd c5 rc=$?"
BSPMM_LIB=checked timeout 600 python tools/probe/sddmm_once.py > $O/sddmm_c5_checked.txt 2>&1; echo "sddmm c5 rc=$?"
BSPMM_LIB=checked python -c "import paper_1903_11409_b200._lib as L; print(\"loaded:\", L.LIB_PATH)" >> $O/pytest_gpu_checked.txt
