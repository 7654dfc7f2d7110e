# quick GPU iteration: kernel + runtime parity tests, kernel micro-bench, bench
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python scripts/kbench.py 256 2>&1 | head -4
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_iter.json; cat gpurun_out/bench_iter.json | cut -c1-600
