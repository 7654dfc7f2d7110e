# DRAM traffic of every conv_fwd launch of one eager DELTA@50% step (ncu, cheap metrics)
mkdir -p gpurun_out
ncu --profile-from-start off -k regex:k_conv_fwd --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/conv_traffic.csv python scripts/profile_step.py > /dev/null 2>&1
ncu --profile-from-start off -k regex:k_wgrad --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wgrad_traffic.csv python scripts/profile_step.py > /dev/null 2>&1
ls -la gpurun_out/*traffic*
