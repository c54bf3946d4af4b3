#!/bin/bash
# GPU box: compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_case.py cases.
OUT=gpurun_out/${TAG:-r02}_sanitizer.txt
: > $OUT
for tool in memcheck racecheck synccheck; do
  for c in tiny n512_d64 n512_d128 st_d128 str_d64; do
    echo "=== $tool $c" >> $OUT
    timeout 300 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $c >> $OUT 2>&1
    echo "exit $?" >> $OUT
  done
done
grep -E "^===|ERROR SUMMARY|exit|Error|error" $OUT | head -80
