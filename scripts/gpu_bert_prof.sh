# BERT profiling pass: parity/timing script, ncu launch list of one eager
# DELTA step, full ncu captures of the attention kernels.
# usage: bash scripts/gpu_bert_prof.sh TAG [BATCH]
TAG=${1:-x}
BS=${2:-32}
mkdir -p gpurun_out
timeout 600 python scripts/bert_step.py --batch $BS > gpurun_out/bert_$TAG.log 2>&1; tail -c 1500 gpurun_out/bert_$TAG.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/bert_launches_$TAG.csv python scripts/bert_step.py --batch $BS --profile > gpurun_out/bert_prof_$TAG.log 2>&1
echo "ncu list rc=$?"
python scripts/summarize_launches.py gpurun_out/bert_launches_$TAG.csv "bert $TAG" > gpurun_out/bert_launches_${TAG}_summary.txt 2>&1
head -30 gpurun_out/bert_launches_${TAG}_summary.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_attn -s 3 -c 3 \
  -o gpurun_out/bert_attn_$TAG python scripts/bert_step.py --batch $BS --profile > gpurun_out/bert_prof2_$TAG.log 2>&1
echo "ncu attn rc=$?"; tail -2 gpurun_out/bert_prof2_$TAG.log
