python -m pytest tests/test_shuffle_gpu.py -x -q -m gpu -k "partitioned or fixtures or bijection" > gpurun_out/pytest_part.txt 2>&1
for v in default t512 t1024; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "== $v"; env $L python tools/exp_part.py 2>&1 | head -3
  env $L ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_once.py 29 2 2>/dev/null | grep -E "k_part|k_place" | awk -F'","' '{print $5 " " $NF}' | cut -c1-40,200- | tail -3
done
