for v in default g48 g64 g96; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "== $v"; env $L python tools/exp_part.py 2>&1 | head -2
done
BSG_LIB=build/var_g64/libbsg.so python -m pytest tests/test_shuffle_gpu.py -q -m gpu -x -k "partition or scatter or sharded" 2>&1 | tail -1
