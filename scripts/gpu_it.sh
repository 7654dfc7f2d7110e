mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
DELTA_STEM_MODE=tma timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -m gpu -k "stem or wgrad" 2>&1 | tail -1
timeout 300 python scripts/kbench.py 256 2>&1 | grep shape | cut -c1-100
timeout 300 python scripts/kbench_wgrad.py 2>&1 | cut -c1-110
timeout 300 python scripts/kbench_dgrad.py 2>&1 | grep shape | cut -c1-150
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['no_eviction'], d['e2e']['value'])"
