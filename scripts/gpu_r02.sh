# round-2 GPU pass: tests, smoke, bench, launch list, one full ncu capture.
# usage: bash scripts/gpu_r02.sh TAG [skip-tests]
TAG=${1:-x}
mkdir -p gpurun_out
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
  echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_$TAG.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
  echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py --steps 20 --warmup 5 --detail gpurun_out/bench_detail_$TAG.json > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?"; tail -c 2500 gpurun_out/bench_$TAG.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python scripts/profile_step.py > gpurun_out/prof_$TAG.log 2>&1
echo "ncu list rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_$TAG.csv "$TAG" > gpurun_out/launches_${TAG}_summary.txt 2>&1
head -12 gpurun_out/launches_${TAG}_summary.txt
