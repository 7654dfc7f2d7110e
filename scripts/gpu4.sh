timeout 900 python bench.py --export-trace gpurun_out/resnet50_bs256_trace.json 2>&1 | tail -5
