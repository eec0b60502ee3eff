#!/bin/bash
# compute-sanitizer over every kernel family at small sizes (race detection for the look-back flags).
OUT=${OUT:-gpurun_out}
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py > $OUT/sanitize_$tool.txt 2>&1
  echo "exit $?"; tail -4 $OUT/sanitize_$tool.txt
done
