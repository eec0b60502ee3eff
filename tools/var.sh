for v in default c16 p16 p4; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  for c in c2 c3; do
    echo "== $v $c"; env $L python bench.py --config $c --no-comparators --no-cpu-baseline --e2e-steps 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])"
  done
done
