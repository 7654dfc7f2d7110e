timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -m gpu 2>&1 | tail -2
timeout 600 python -m pytest tests/test_runtime_gpu.py -q -x -m gpu 2>&1 | tail -2
for G in 0 1; do echo "GRID=$G"; DELTA_BN_BWD_GRID=$G timeout 300 python scripts/kbench.py 256 2>&1 | grep bn_backward; done
for G in 0 1 0 1; do
 DELTA_BN_BWD_GRID=$G timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/ab.log 2>&1; echo "GRID=$G"; tail -1 gpurun_out/ab.log | cut -c90-200
done
