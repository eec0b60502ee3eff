for v in default lb1 lb2; do
  if [ $v = default ]; then L=""; else L="LD_LIBRARY_PATH=build/var_$v BSG_LIB=build/var_$v/libbsg.so"; fi
  echo "== $v"; env $L python tools/exp_c3.py 2>&1 | grep -E "536870913|268435457"
  env $L python -c "
import sys,torch; sys.path.insert(0,'.'); import paper_2106_06161_b200 as b
v=torch.arange((1<<20)+1,dtype=torch.int64,device='cuda'); o=torch.empty_like(v); c=b.ShuffleConfig()
for _ in range(10): b.shuffle_values_into(v,c,o)
torch.cuda.synchronize(); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True); e0.record()
for _ in range(200): b.shuffle_values_into(v,c,o)
e1.record(); torch.cuda.synchronize(); print('2^20+1 us/call', e0.elapsed_time(e1)/200*1e3)"
done
python -m pytest tests/test_shuffle_gpu.py -q -m gpu -x -k "fixtures or exhaustive or boundaries or compact or range or concurrent or determinism" 2>&1 | tail -1
