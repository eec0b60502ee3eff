# usage: VARS="a b c" bash tools/run_var.sh -- per-kernel ncu times and the C2 shuffle time of each
# build/var_<v>/libbsg.so next to the default build (one box, interleaved)
mkdir -p gpurun_out
for v in default $VARS; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "== $v $(env $L timeout 300 python tools/exp_partition.py ${P23_CASES:-1} 2>&1 | grep -o '[0-9.]* ms' | head -1)" | tee -a gpurun_out/var.txt
  env $L ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_once.py 29 2 1 2>/dev/null | grep -E "k_part|k_place" | awk -F'","' '{print substr($5,1,50), $NF}' | tail -3 | tee -a gpurun_out/var.txt
done
