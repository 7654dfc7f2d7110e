timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k maxpool 2>&1 | tail -1
python scripts/kbench_pool.py; DELTA_LIB=$PWD/build/ab/libdelta.so python scripts/kbench_pool.py
