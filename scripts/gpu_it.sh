timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k wgrad 2>&1 | tail -1
timeout 300 python scripts/kbench_wgrad.py 2>&1 | cut -c1-75 > /tmp/new.txt; DELTA_LIB=$PWD/build/ab/libdelta.so timeout 300 python scripts/kbench_wgrad.py 2>&1 | cut -c1-75 > /tmp/old.txt; paste -d'|' /tmp/new.txt /tmp/old.txt
