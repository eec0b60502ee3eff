# VARS="a b" CFGS="c2 c3" bash tools/run_vars.sh -- per-kernel times of variant builds next to the default build
for v in default $VARS; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  for c in ${CFGS:-c2}; do env $L python tools/ktime.py $c ${REPS:-5} 2>/dev/null | grep -v -E "Memset|window"; done
done
