# A/B: weight gradients on a side stream vs in-line
for v in 1 0; do
DELTA_SIDE_STREAM=$v timeout 600 python bench.py --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('side=$v', d['value'], d['no_eviction']['images_per_s'], d['e2e']['value'])"
done
timeout 600 python -m pytest tests/test_runtime_gpu.py -q -x 2>&1 | tail -2
