# compute-sanitizer memcheck / racecheck / synccheck over every kernel
# (tools/sanitize_driver.py); summary lines -> gpurun_out/sanitize_<tool>.txt
for T in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_driver.py > gpurun_out/sanitize_$T.txt 2>&1
  echo "$T rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|BAD|FAILS|Error" gpurun_out/sanitize_$T.txt | tail -5 | tee -a gpurun_out/sanitize_summary.txt
done
