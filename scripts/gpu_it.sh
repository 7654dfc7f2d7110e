for G in 1 0 1 0 1 0; do
 DELTA_FUSE_BN3_SUMS=$G timeout 600 python bench.py --steps 50 --warmup 10 > gpurun_out/ab.log 2>&1; echo "SUMS=$G $(tail -1 gpurun_out/ab.log | cut -c90-125)"
done
