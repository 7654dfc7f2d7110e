timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_runtime_gpu.py -q -x 2>&1 | tail -2
timeout 300 python scripts/kbench.py 256 2>&1 | grep kernel | grep bn_backward
timeout 900 python bench.py 2>&1 | tail -1
