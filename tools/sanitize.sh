#!/bin/bash
# compute-sanitizer over every kernel family at small sizes (race detection for the look-back flags).
OUT=${OUT:-gpurun_out}
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py > $OUT/sanitize_$tool.txt 2>&1
  echo "exit $?"; tail -4 $OUT/sanitize_$tool.txt
done
# initcheck does not model the TMA engine's bulk shared->global stores (the last passes' output windows): their
# bytes read as uninitialised on the later D2H copy although they equal the oracle.  Rerun with plain stores
# (bsg_set_bulk_stores(0)) so the rest of the check stays meaningful.
echo "== initcheck (last passes with plain stores)"
BSG_SAN_NO_BULK=1 compute-sanitizer --tool initcheck --error-exitcode 9 --print-limit 20 python tools/sanitize_run.py > $OUT/sanitize_initcheck_nobulk.txt 2>&1
echo "exit $?"; tail -4 $OUT/sanitize_initcheck_nobulk.txt
