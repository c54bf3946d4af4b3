#!/bin/bash
# compute-sanitizer over the final build (product library), plus the one-launch residue kernel
# (diagnostics library, SPLAT_RESIDUE_1PASS=1)
mkdir -p gpurun_out
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
TAG=r02zn bash tools/sanitize_all.sh
python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || exit 1
OUT=gpurun_out/r02zn_sanitizer.txt
for tool in memcheck racecheck synccheck; do
  echo "=== $tool st_d128 one-launch (diag)" >> $OUT
  SPLAT_LIB=diag SPLAT_RESIDUE_1PASS=1 timeout 300 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py st_d128 >> $OUT 2>&1
  echo "exit $?" >> $OUT
done
grep -E "^===|ERROR SUMMARY|exit" $OUT | tail -12
