python bench.py --config c4 --no-cpu-baseline --steps 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'])"
python -m pytest tests/test_shuffle_gpu.py -q -m gpu -x -k "batched" 2>&1 | tail -1
