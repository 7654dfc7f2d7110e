timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -1
for L in new old; do if [ $L = old ]; then export DELTA_LIB=$PWD/build/ab/libdelta.so; else unset DELTA_LIB; fi; echo $L; timeout 300 python scripts/kbench_dgrad.py 2>&1 | grep shape | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if 'bn_bwd_us' in d: print(d['shape'], d['bn_bwd_us'], d['plain_us'])"; done
