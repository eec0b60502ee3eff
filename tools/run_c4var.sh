# A/B of batched-kernel variants (build/var_<v>) on the C4 bench, interleaved twice
for i in 1 2; do for v in default $VARS; do
  if [ $v = default ]; then L=""; else L="BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "$v $(env $L timeout 300 python bench.py --config c4 --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["value"], d["graph_replay"]["ms_per_step"])')"
done; done
