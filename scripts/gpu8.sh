ncu --set full --clock-control none --import-source on -k regex:k_conv_fwd -s 2 -c 1 -o gpurun_out/r01_conv3x3_v2 python scripts/conv_one.py 56 64 64 3 1 1 > gpurun_out/p.log 2>&1
tail -2 gpurun_out/p.log
