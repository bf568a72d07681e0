# compute-sanitizer over scripts/sanitize_probe.py, one tool per pass
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_probe.py > gpurun_out/san_$t.log 2>&1
  echo "$t rc=$?" | tee -a gpurun_out/san_summary.txt
done
