for v in default p2p; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "== $v"; env $L ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_once.py 29 2 2>/dev/null | grep -E "k_part2" | awk -F'","' '{print substr($5,1,40), $NF}' | tail -1
  env $L python tools/exp_part.py 2>&1 | head -2
done
BSG_LIB=build/var_p2p/libbsg.so python -m pytest tests/test_shuffle_gpu.py -q -m gpu -x -k "partition or scatter or sharded" 2>&1 | tail -1
