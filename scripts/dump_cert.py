"""Dump an executed timeline (device action log) + plan for offline analysis."""
import sys, json
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2203_15980_b200 import planner as P
from paper_2203_15980_b200.runtime import DeltaRuntime

frac = float(sys.argv[1]); policy = P.PolicyMode(int(sys.argv[2])); out = sys.argv[3]
torch.backends.cudnn.deterministic = True
base = DeltaRuntime(50, 16, seed=0, lr=0.0)
base.measure_costs(iters=2)
rt = DeltaRuntime(50, 16, seed=0, lr=0.0)
for n, m in zip(rt.nodes, base.nodes):
    n.cost_us = m.cost_us
rt.link_gbs = base.link_gbs
prog = rt.plan(frac, policy=policy)
findings = []
ev = rt.executed_timeline(findings)
plan = P.run_iteration(rt.trace(), rt.config).events
np.savez(out, ev=ev, plan=plan, actions=prog.actions)
open(out + ".trace.json", "w").write(rt.trace().to_json())
json.dump({"budget": rt.config.budget, "bw": list(rt.config.cost_model.bandwidth_bytes_per_us),
           "policy": int(policy), "findings": findings}, open(out + ".cfg.json", "w"))
print("ok", len(ev), findings[:3])
