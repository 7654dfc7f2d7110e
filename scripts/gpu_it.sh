timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -m gpu 2>&1 | tail -2
for L in build/ab/libdelta.so paper_2203_15980_b200/libdelta.so build/ab/libdelta.so paper_2203_15980_b200/libdelta.so; do
 DELTA_LIB=$L timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/ab.log 2>&1; echo "$L"; tail -1 gpurun_out/ab.log | cut -c90-200
done
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v8.csv python scripts/profile_step.py > gpurun_out/prof1.log 2>&1; tail -1 gpurun_out/prof1.log
