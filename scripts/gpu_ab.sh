# A/B: DELTA anchor sets at the 50% budget
for a in out+narrow out; do
timeout 600 python bench.py --steps 10 --anchors $a 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('anchors=$a', d.get('value'), d.get('no_eviction',{}).get('images_per_s'), d.get('plan',{}).get('counts'), d.get('recompute',{}).get('ms_per_step'))" 2>&1 | tail -1
done
