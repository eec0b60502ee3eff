python -m pytest tests/test_shuffle_gpu.py -q -m gpu -x -k "fixtures or exhaustive or boundaries or partition or range" > gpurun_out/pytest_v.txt 2>&1
for v in default c16 s1b; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "== $v"; env $L python tools/exp_c3.py 2>&1 | grep -E "536870913|536870912 values  "
  env $L python tools/exp_part.py 2>&1 | head -1
done
BSG_LIB=build/var_c16/libbsg.so python -m pytest tests/test_shuffle_gpu.py -q -m gpu -x -k "fixtures or exhaustive or boundaries or range or sharded" > gpurun_out/pytest_c16.txt 2>&1
