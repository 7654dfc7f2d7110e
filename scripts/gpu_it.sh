timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -1
DELTA_REG_STATS_ALL=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -1
for m in 1 0 1 0; do DELTA_REG_STATS_ALL=$m timeout 900 python bench.py --cpu-sample-s 1 > gpurun_out/bench.log 2>&1; echo -n "REGALL=$m "; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['no_eviction']['images_per_s'], d['e2e']['value'])"; done
