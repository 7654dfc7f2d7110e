timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "bn or maxpool or avgpool" 2>&1 | tail -2
timeout 300 python scripts/kbench.py 256 2>&1 | grep kernel
