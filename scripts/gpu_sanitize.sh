# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on scripts/sanitize_small.py
TAG=${TAG:-r02}
out=gpurun_out/${TAG}_sanitizer.txt
echo "# compute-sanitizer on scripts/sanitize_small.py, one B200, ${TAG}" > $out
for T in memcheck racecheck synccheck initcheck; do
  echo "## $T" >> $out
  timeout 1200 compute-sanitizer --tool $T python scripts/sanitize_small.py 2>&1 | grep -E "sanitize-small|SUMMARY|Error|error|Invalid|Race|Hazard" | head -30 >> $out
done
cat $out
