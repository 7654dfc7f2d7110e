"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals: python scripts/summarize_launches.py launches.csv [title]"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    name = re.sub(r"\(CUtensorMap.*|\(.*", "", r[ki])[:100]
    tot[name] += float(r[vi]) / 1e6
    cnt[name] += 1
all_ms = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
print(f"launches {sum(cnt.values())}  total {all_ms:.2f} ms")
OURS = re.compile(r"(delta_k::|unnamed>::|anonymous namespace\)::)k_")
ours = sum(v for k, v in tot.items() if OURS.search(k))
print(f"our kernels (delta_k::k_*): {ours:.2f} ms = {100 * ours / all_ms:.1f}%  "
      f"(other: {', '.join(k for k in tot if not OURS.search(k)) or 'none'})")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"  {v:7.3f} ms {100 * v / all_ms:5.1f}%  n={cnt[k]:4d}  {k}")
