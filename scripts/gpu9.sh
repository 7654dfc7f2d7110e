timeout 900 python -m pytest tests/test_runtime_gpu.py -q -x 2>&1 | tail -3
timeout 900 python bench.py 2>&1 | tail -1
