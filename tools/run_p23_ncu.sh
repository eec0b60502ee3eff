mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active
for env in "BSG_P23=0" "BSG_P23=1 BSG_P23_LAG=2" "BSG_P23=1 BSG_P23_LAG=3 BSG_P23_S2=6"; do
  echo "== $env" >> gpurun_out/p23_ncu.txt
  env $env ncu --metrics $M --clock-control none --csv python tools/run_once.py 29 2 1 2>/dev/null | grep -E "k_part|k_place" | awk -F'","' '{print substr($5,1,60), $(NF-2), $NF}' | tail -12 >> gpurun_out/p23_ncu.txt
done
cat gpurun_out/p23_ncu.txt
