timeout 300 python scripts/kbench.py 256 2>&1 | grep kernel
