"""Executed comparison grid on the GPU: ResNet-50 at the
bench batch, budgets x policies x heuristics, every cell planned, executed,
timed and checked bit-identical to the no-eviction step.
    python scripts/exec_grid.py [batch] [out_prefix]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_15980_b200 import grid as GR  # noqa: E402
from paper_2203_15980_b200 import planner as P  # noqa: E402
from paper_2203_15980_b200.runtime import DeltaRuntime  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/exec_grid"
rt = DeltaRuntime(50, B, seed=0)
g = torch.Generator().manual_seed(0)
x = torch.zeros(rt.x_dev.shape, dtype=torch.bfloat16)
x[..., :3] = torch.randn(B, 224, 224, 3, generator=g).to(torch.bfloat16)
y = torch.randint(0, 1000, (B,), generator=g)
for s in range(2):
    rt.x_slots[s].copy_(x)
    rt.y_slots[s].copy_(y)
rt.measure_costs(iters=3)
text, detail = GR.executed_comparison(
    rt, [0.4, 0.5, 0.6, 0.7, 0.8],
    [P.PolicyMode.Delta, P.PolicyMode.RecomputeOnly, P.PolicyMode.OffloadOnly],
    [P.Heuristic.Base, P.Heuristic.Lru, P.Heuristic.Greedy], steps=5, warmup=2)
open(out + ".csv", "w").write(text)
json.dump({"batch": B, "link_gbs": rt.link_gbs, "cells": detail}, open(out + ".json", "w"), indent=1)
print(text)
print("bit-identical:", sum(1 for c in detail if c.get("bit_identical")), "of",
      sum(1 for c in detail if not c["infeasible"]), "feasible cells")
