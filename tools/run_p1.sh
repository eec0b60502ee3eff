for v in ${VARS:-f0m3 f1m2 f1m3 f1t512m2}; do
  for c in ${CFGS:-c2 c3}; do
    BSG_LIB=build/var_$v/libbsg.so python tools/ktime.py $c 5 2>/dev/null | grep -v Memset
  done
done
