timeout 1500 python scripts/max_batch_verify.py 2>&1 | tail -8
