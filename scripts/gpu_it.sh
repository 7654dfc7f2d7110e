mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -m gpu 2>&1 | tail -1
timeout 300 python scripts/kbench_dgrad.py 2>&1 | grep shape | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print({k:v for k,v in d.items() if k in ('shape','add_mask_us','bn_bwd_us','add_stride2_us','add_full_us')})"
