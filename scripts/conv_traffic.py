"""Summarise the ncu DRAM traffic of the forward conv launches of one eager
DELTA@50% step (gpurun_out/conv_traffic.csv from scripts/gpu_traffic.sh) against
their algorithmic bytes (input + output of each conv node) -> the committed
profiles/r01_conv_traffic.json that bench.py reports as roofline.traffic."""
import csv
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_15980_b200 import graph as G  # noqa: E402

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/conv_traffic.csv"
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
launch = {}
for r in rows[1:]:
    d = launch.setdefault(int(r[ii]), {"name": r[ki]})
    d[r[mi]] = float(r[vi].replace(",", ""))
seq = [launch[k] for k in sorted(launch)]
g = G.build_resnet(50, 256)
convs = [n for n in g.nodes if n.op == "conv"]
# the 3x3 stride-1 64->64 convs run on the halo kernel (conv_halo_default)
halo = [n for n in convs
        if g.convs[n.attrs["conv"]].k == 3 and g.convs[n.attrs["conv"]].stride == 1
        and g.convs[n.attrs["conv"]].cin == 64 and g.convs[n.attrs["conv"]].cout == 64]
fwd_nodes = [n for n in convs if n not in halo]
# the forward phase issues exactly these convs, in order, before any recompute
fwd = seq[:len(fwd_nodes)]
assert all(re.search(r"k_conv_fwd<\d+, \d+, \d+, 0>", d["name"]) for d in fwd)
dram = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in fwd)
alg = sum(n.hbm_bytes for n in fwd_nodes)
out = {"launches": len(fwd), "dram_bytes_per_launch": round(dram / len(fwd)),
       "algorithmic_bytes_per_launch": round(alg / len(fwd)),
       "traffic_over_algorithmic": round(dram / alg, 3),
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (scripts/gpu_traffic.sh) "
                 "over the forward k_conv_fwd launches of one eager DELTA@50% ResNet-50 bs256 step"}
print(json.dumps(out))
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                 "profiles", "r01_conv_traffic.json"), "w"), indent=1)
