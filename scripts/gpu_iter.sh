# quick GPU iteration: parity tests, bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_iter.json; cut -c1-300 gpurun_out/bench_iter.json
