timeout 600 python -m pytest tests/test_runtime_gpu.py -x -q 2>&1 | tail -1
timeout 600 python scripts/node_times.py 2>&1 | grep -E "fc|sum "
for i in 1 2; do timeout 900 python bench.py --cpu-sample-s 1 > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['no_eviction']['images_per_s'], d['e2e']['value'])"; done
