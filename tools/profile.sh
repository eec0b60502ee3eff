#!/bin/bash
# Captures the ncu evidence for the bench configurations (run under gpurun on one GPU).
#   launch lists: every kernel of a short bench run with its device time (cold cache, serialised)
#   full sets:    one capture of the dominant kernel per config
set -x
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
B="python bench.py --steps 2 --warmup 1 --no-comparators --no-cpu-baseline --e2e-steps 1"
for cfg in c2 c3 c4 c5; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$cfg.csv $B --config $cfg > $OUT/launches_$cfg.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k_part1|k_part2|k_place" -s 3 -c 3 -o $OUT/prof_c2 $B --config c2 > $OUT/prof_c2.log 2>&1
BSG_PATH=1 ncu --set full --clock-control none --import-source on -k regex:k_pow2 -s 1 -c 1 -o $OUT/prof_c2single $B --config c2 > $OUT/prof_c2single.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_part1|k_part2|k_window|k_place" -s 5 -c 5 -o $OUT/prof_c3 $B --config c3 > $OUT/prof_c3.log 2>&1
BSG_PATH=1 ncu --set full --clock-control none --import-source on -k regex:k_compact -s 1 -c 1 -o $OUT/prof_c3single $B --config c3 > $OUT/prof_c3single.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_batched -s 1 -c 1 -o $OUT/prof_c4 $B --config c4 > $OUT/prof_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pow2 -s 1 -c 1 -o $OUT/prof_c5 $B --config c5 > $OUT/prof_c5.log 2>&1
ls -la $OUT
