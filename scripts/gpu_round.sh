# One gpurun call: GPU parity tests, smoke, bench (+reference arm), ncu launch list and
# full captures of the top kernels, max-batch verification.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/prof1.log 2>&1; tail -1 gpurun_out/prof1.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_conv_fwd -s 40 -c 6 -o gpurun_out/conv_fwd python scripts/profile_step.py > gpurun_out/prof2.log 2>&1; tail -1 gpurun_out/prof2.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_bn_bwd -s 30 -c 6 -o gpurun_out/bn_bwd python scripts/profile_step.py > gpurun_out/prof3.log 2>&1; tail -1 gpurun_out/prof3.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_bn_apply -s 2 -c 2 -o gpurun_out/bn_apply python scripts/profile_step.py > gpurun_out/prof4.log 2>&1; tail -1 gpurun_out/prof4.log
timeout 1500 python scripts/max_batch_verify.py > gpurun_out/max_batch.log 2>&1; tail -2 gpurun_out/max_batch.log | cut -c1-600
ls -la gpurun_out
