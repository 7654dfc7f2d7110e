nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -30
timeout 300 python scripts/kbench.py 256 2>&1 | tail -30
