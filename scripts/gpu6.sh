timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -5
timeout 300 python scripts/kbench.py 256 2>&1 | grep -v Exception | tail -18
