for v in default early; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "== $v"; env $L python tools/exp_c3.py 2>&1 | grep -E "536870913|268435457"
done
BSG_LIB=build/var_early/libbsg.so python -m pytest tests/test_shuffle_gpu.py -q -m gpu -x -k "fixtures or exhaustive or boundaries or range or sharded" 2>&1 | tail -1
