timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for m in 1 0; do echo "RB=$m"; DELTA_RESIDENT_B=$m timeout 300 python scripts/kbench.py 256 2>&1 | grep shape | cut -c1-60 | head -9; done
for m in 1 0 1 0; do DELTA_RESIDENT_B=$m timeout 900 python bench.py --cpu-sample-s 1 > gpurun_out/bench.log 2>&1; echo -n "RB=$m "; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['no_eviction']['images_per_s'], d['e2e']['value'])"; done
