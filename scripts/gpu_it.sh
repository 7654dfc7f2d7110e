timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
DELTA_CONV_HALO=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "conv_fwd" 2>&1 | tail -1
timeout 600 python scripts/node_times.py 2>&1 | grep -E "layer1.[012].conv2$"
for m in new old new old; do if [ $m = old ]; then export DELTA_LIB=$PWD/build/ab/libdelta.so; else unset DELTA_LIB; fi; timeout 900 python bench.py --cpu-sample-s 1 > gpurun_out/bench.log 2>&1; echo -n "$m "; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['no_eviction']['images_per_s'], d['e2e']['value'])"; done
