ncu --set full --clock-control none -k regex:k_bn_bwd -s 3 -c 3 -o gpurun_out/r01_bnbwd python scripts/bnbwd_one.py > gpurun_out/p.log 2>&1; tail -1 gpurun_out/p.log
