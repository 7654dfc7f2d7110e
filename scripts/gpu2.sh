timeout 1200 python -m pytest tests/test_runtime_gpu.py -q -x --durations=0 2>&1 | tail -30
