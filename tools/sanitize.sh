# compute-sanitizer over tools/sanitize_driver.py with every tool
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t"; timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_driver.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|mismatches|Error|error" | head -12
done
