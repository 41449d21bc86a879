set -u
# compute-sanitizer over tools/sanitize_run.py (every kernel and entry point);
# summaries land in gpurun_out/san/ (copied to profiles/r02/ when judged)
O=gpurun_out/san; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout -s KILL 1500 $CS --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/$tool.log 2>&1
  echo "$tool rc=$?"; tail -n 3 $O/$tool.log
done
timeout -s KILL 1500 $CS --tool racecheck --racecheck-report analysis --print-limit 20 python tools/sanitize_run.py 32 > $O/racecheck.log 2>&1
echo "racecheck rc=$?"; tail -n 5 $O/racecheck.log
