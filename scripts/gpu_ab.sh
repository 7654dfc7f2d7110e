# A/B: stats fused into every conv epilogue vs only long-K convs
timeout 600 python bench.py --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['value'], d['no_eviction']['images_per_s'], d['roofline']['op_ms'])"
DELTA_FUSE_STATS_MIN_KDIM=0 timeout 600 python bench.py --steps 10 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fuse-all', d['value'], d['no_eviction']['images_per_s'], d['roofline']['op_ms'])"
