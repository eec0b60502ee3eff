#!/bin/bash
# Captures the ncu evidence for the bench configurations (run under gpurun on one GPU).
#   PART=launch: launch lists of every bench config (each kernel with its device time; cold cache, serialised)
#   PART=c2|c2single|c3|c3rt|c3single|c4|c5: one full-set capture of that config's kernels (c3rt: the persistent
#   last pass of C3, merged into the c3 summary by tools/ncu_summary.py)
# Split into parts because gpurun returns at most 64 MiB of gpurun_out per call.
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
B="python bench.py --steps 2 --warmup 1 --no-comparators --no-cpu-baseline --e2e-steps 1"
N="ncu --set full --clock-control none --import-source on"
case ${PART:-launch} in
  launch)
    for cfg in c2 c3 c4 c5; do
      ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$cfg.csv $B --config $cfg > $OUT/launches_$cfg.log 2>&1
    done ;;
  c2) $N -k regex:"k_part1|k_part2|k_place" -s 3 -c 3 -o $OUT/prof_c2 $B --config c2 > $OUT/prof_c2.log 2>&1 ;;
  c2single) BSG_PATH=1 $N -k regex:k_pow2 -s 1 -c 1 -o $OUT/prof_c2single $B --config c2 > $OUT/prof_c2single.log 2>&1 ;;
  c3) $N -k regex:"k_part1|k_part2|k_window|k_place" -s 6 -c 6 -o $OUT/prof_c3 $B --config c3 > $OUT/prof_c3.log 2>&1 ;;
  c3rt) $N -k regex:k_place_rank_t -s 1 -c 1 -o $OUT/prof_c3rt $B --config c3 > $OUT/prof_c3rt.log 2>&1 ;;
  c3single) BSG_PATH=1 $N -k regex:k_compact -s 1 -c 1 -o $OUT/prof_c3single $B --config c3 > $OUT/prof_c3single.log 2>&1 ;;
  c4) $N -k regex:k_batched -s 1 -c 1 -o $OUT/prof_c4 $B --config c4 > $OUT/prof_c4.log 2>&1 ;;
  c5) $N -k regex:k_pow2 -s 1 -c 1 -o $OUT/prof_c5 $B --config c5 > $OUT/prof_c5.log 2>&1 ;;
esac
ls -la $OUT
