"""Per-node device time of one eager DELTA@50% ResNet-50 bs256 step (events per
action through the C++ executor) against each node's serial roofline
max(FLOPs/TC peak, algorithmic bytes/HBM peak); sorted by the gap."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_15980_b200.runtime import DeltaRuntime

rt = DeltaRuntime(depth=50, batch=256)
rt.measure_costs()
rt.plan(0.5)
rt.step_device()
torch.cuda.synchronize()
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
tc, hbm = peaks["bf16_tflops"], peaks["hbm_gbs"]
for _ in range(2):
    timing = {}
    with torch.cuda.stream(rt.stream):
        rt.run_program(timing=timing)
    torch.cuda.synchronize()
rows = []
for nid, lst in timing.items():
    if nid == "swap":
        continue
    n = rt.nodes[nid]
    for ms, rec in lst:
        roof = max(n.flops / (tc * 1e9), (n.hbm_bytes or 2 * n.nbytes) / (hbm * 1e6))
        rows.append((ms - roof, ms, roof, n.name + (" (rec)" if rec else ""), n.op))
rows.sort(reverse=True)
tot = sum(r[1] for r in rows)
print(f"sum {tot:.3f} ms, roofline {sum(r[2] for r in rows):.3f} ms")
for gap, ms, roof, name, op in rows[:40]:
    print(f"{gap * 1e3:8.1f} us gap  {ms * 1e3:8.1f} us  roof {roof * 1e3:7.1f}  {op:18s} {name}")
