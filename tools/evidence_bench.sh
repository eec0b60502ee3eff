#!/bin/bash
# Round-end bench evidence on one B200: every configuration, the reference arm of C2/C3, and the --gpus 2 code path
# (two ranks sharing GPU 0 over gloo; not a scaling number).  Lines land in gpurun_out/b_<cfg>.json.
OUT=${OUT:-gpurun_out}
mkdir -p $OUT
for c in ${CFGS:-c2 c2lcg c3 c3lcg c4 c1 c5}; do
  extra=""; [ $c = c5 ] && extra="--steps 5"
  python bench.py --config $c $extra > $OUT/b_$c.json 2> $OUT/b_$c.err
done
for c in ${REFS:-c2 c3}; do
  python bench.py --impl reference --config $c > $OUT/b_ref_$c.json 2> $OUT/b_ref_$c.err
done
BSG_BENCH_DEVICE=0 BSG_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c2 --steps 5 --warmup 3 \
  > $OUT/b_n2_gloo_one_gpu.json 2> $OUT/b_n2.err
echo "n2 exit $?" >> $OUT/b_n2.err
