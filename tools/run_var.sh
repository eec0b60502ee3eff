# usage: VARS="a b c" bash tools/run_var.sh  -- times each build/var_<v>/libbsg.so (and the default) on the C2 shuffle
mkdir -p gpurun_out
for v in default $VARS; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "== $v" | tee -a gpurun_out/var.txt
  env $L timeout 300 python tools/exp_partition.py ${P23_CASES:-2} 2>&1 | tee -a gpurun_out/var.txt
  env $L ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/run_once.py 29 2 1 2>/dev/null | grep -E "k_part|k_place" | awk -F'","' '{print substr($5,1,50), $(NF-2), $NF}' | tail -3 | tee -a gpurun_out/var.txt
done
