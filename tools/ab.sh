#!/bin/bash
# A/B per-kernel times: CFGS="c3 c3lcg" VARS="rt0" bash tools/ab.sh  (default build first, then build/var_<v>)
mkdir -p gpurun_out
for c in ${CFGS:-c2}; do
  for v in default $VARS; do
    if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
    env $L timeout 300 python tools/ktime.py $c ${REPS:-5} 2>&1 | tee -a gpurun_out/ab.txt
  done
done
