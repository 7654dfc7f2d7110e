set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "dgrad" 2>&1 | tail -30
