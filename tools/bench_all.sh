# Every bench configuration once (one box), lines into gpurun_out/b_<cfg>.json
for c in ${CFGS:-c2 c2lcg c3 c3lcg c4 c1 c5}; do
  extra=""; [ $c = c5 ] && extra="--steps 5"
  python bench.py --config $c $extra > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err
done
