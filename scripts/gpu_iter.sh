# quick GPU iteration: parity tests, bench (+ optional max-batch verification)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_iter.log 2>&1; tail -3 gpurun_out/pytest_iter.log
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_iter.json; cut -c1-200 gpurun_out/bench_iter.json
if [ "$MB" = "1" ]; then timeout 1500 python scripts/max_batch_verify.py > gpurun_out/max_batch.log 2>&1; tail -3 gpurun_out/max_batch.log | cut -c1-400; fi
