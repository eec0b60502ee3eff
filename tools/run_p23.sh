mkdir -p gpurun_out
for env in ${P23_ENVS:-"BSG_P23=0"}; do
  env ${env//,/ } timeout 300 python tools/exp_p23.py ${P23_CASES:-8} 2>&1 | tee -a gpurun_out/p23.txt
done
