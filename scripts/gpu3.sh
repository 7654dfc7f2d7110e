timeout 600 python scripts/debug_fwd.py 16 2>&1 | grep -v "^Exception\|Traceback\|File\|Attribute" | tail -70
