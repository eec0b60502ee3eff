# usage: ENVS="A=1 A=2,B=3" bash tools/run_env.sh -- C2 shuffle time and equality under each env setting
for e in "" $ENVS; do echo "[$e] $(env ${e//,/ } timeout 300 python tools/exp_partition.py ${CASES:-2} 2>&1 | grep -o '[0-9.]* ms.*equal=[A-Za-z]*' | tr '\n' ' ')"; done
