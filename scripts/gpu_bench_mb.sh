set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log > gpurun_out/bench_full.json; tail -3 gpurun_out/bench_full.log | cut -c1-300
timeout 1500 python scripts/max_batch_verify.py > gpurun_out/max_batch.log 2>&1; tail -4 gpurun_out/max_batch.log | cut -c1-1500
