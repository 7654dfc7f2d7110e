# A/B on one box: bench variants selected by environment assignments.
# usage: bash scripts/gpu_ab.sh "ENV=a" "ENV=b" ...   (each run twice, interleaved)
for rep in 1 2; do
  for v in "$@"; do
    env $v timeout 600 python bench.py --steps 20 --warmup 5 --bert-batch 32 --no-verify-max-batch 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d.get('bert') or {}; print('$v', 'resnet', d['value'], 'noev', d['no_eviction_images_per_s'], 'bert', b.get('seq_per_s'), 'clk', d['clocks']['sm_mhz'])"
  done
done
