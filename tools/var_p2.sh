for v in default p2t512 p2t1024; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "== $v"
  env $L ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv python tools/run_once.py 29 2 2>/dev/null | grep -E "k_part2" | awk -F'","' '{print substr($5,1,40), $(NF-2), $NF}' | tail -3
done
