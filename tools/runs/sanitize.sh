# compute-sanitizer over tools/sanitize_smoke.py (every kernel incl. the TMA GEMM / wgrad at > 2,048 rows)
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t python tools/sanitize_smoke.py > gpurun_out/r02_sanitizer_$t.txt 2>&1
  echo "rc=$?" >> gpurun_out/r02_sanitizer_$t.txt
  tail -3 gpurun_out/r02_sanitizer_$t.txt
done
