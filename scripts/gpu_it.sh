mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
DELTA_CONV_GATHER=1 timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -m gpu -k "conv" 2>&1 | tail -1
for m in tma gather ""; do DELTA_STEM_MODE=$m timeout 120 python scripts/kbench_stem.py; done
python -c "import torch; a=torch.load('/tmp/stem_tma.pt'); b=torch.load('/tmp/stem_rows.pt'); c=torch.load('/tmp/stem_gather.pt'); print('bit-identical', torch.equal(a,b), torch.equal(a,c))"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['no_eviction'], d['e2e']['value'])"
