timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_runtime_gpu.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --export-trace gpurun_out/resnet50_bs256_trace.json 2>&1 | tail -1
