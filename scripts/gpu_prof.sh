set -x
mkdir -p gpurun_out
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv python scripts/profile_step.py > gpurun_out/prof1.log 2>&1
tail -3 gpurun_out/prof1.log
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_conv_fwd -s 20 -c 3 -o gpurun_out/r01_conv_fwd python scripts/profile_step.py > gpurun_out/prof2.log 2>&1
tail -3 gpurun_out/prof2.log
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:k_bn_bwd_apply -s 4 -c 1 -o gpurun_out/r01_bn_bwd_apply python scripts/profile_step.py > gpurun_out/prof3.log 2>&1
tail -3 gpurun_out/prof3.log
ls -la gpurun_out
