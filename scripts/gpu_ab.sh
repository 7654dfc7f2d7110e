# A/B: 3x3 stride-1 input gradients on our kernel (fused BN backward) vs cuDNN
for v in 0 1; do
DELTA_OWN_DGRAD_3X3=$v timeout 600 python bench.py --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('own3x3=$v', d['value'], d['no_eviction']['images_per_s'], d['roofline']['op_ms'])"
done
DELTA_OWN_DGRAD_3X3=1 timeout 600 python -m pytest tests/test_runtime_gpu.py -q -x 2>&1 | tail -2
