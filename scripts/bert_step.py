"""BERT-large under DELTA on one B200: parity gate (DELTA step == no-eviction
step, bit for bit), graph-replayed step times at no eviction and at the
budget, and the per-op device-time breakdown of one eager step.

    python scripts/bert_step.py [--batch 32] [--budget 0.4] [--layers 24] [--profile]

--profile: one eager DELTA step between cudaProfilerStart/Stop only (for ncu).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_15980_b200 import bert as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--layers", type=int, default=24)
ap.add_argument("--budget", type=float, default=0.4)
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--profile", action="store_true")
args = ap.parse_args()

cfg = B.BertConfig(batch=args.batch, layers=args.layers)
rt = B.BertRuntime(cfg, seed=0)
batch = rt.synthetic_batch(0)
for slot in range(2):
    for d, s in zip(rt.in_slots[slot], batch):
        d.copy_(s)
if args.profile:
    rt.plan(args.budget)
    for _ in range(2):
        rt.step_device()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    rt.step_device()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profiled one step", rt.program.plan_counts)
    sys.exit(0)

rt.measure_costs(iters=3)
lr = rt.lr
rt.lr = 0.0
rt.plan(None)
rng0 = rt.rng.clone()
rt.step_device()
l0, g0 = rt.loss.clone(), rt.params.grad.clone()
prog = rt.plan(args.budget)
rt.rng.copy_(rng0)
rt.step_device()
torch.cuda.synchronize()
parity = {"loss_equal": bool(torch.equal(l0, rt.loss)), "grads_equal": bool(torch.equal(g0, rt.params.grad)),
          "loss": float(l0.item())}
del g0
rt.lr = lr


def timed(frac):
    p = rt.plan(frac)
    rt.step_device()
    rt.capture()
    for _ in range(3):
        rt.step_device()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(rt.stream)
    for _ in range(args.steps):
        rt.step_device()
    e1.record(rt.stream)
    torch.cuda.synchronize()
    return p, e0.elapsed_time(e1) / args.steps


bp, base_ms = timed(None)
dp_, delta_ms = timed(args.budget)
rt.graph = None
timing = {}
with torch.cuda.stream(rt.stream):
    rt.run_program(timing=timing)
torch.cuda.synchronize()
by_op = {}
flops = 0.0
for nid, lst in timing.items():
    if nid == "swap":
        continue
    n = rt.nodes[nid]
    for ms, rec in lst:
        k = n.op + (".re" if rec else "")
        a = by_op.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += ms
        a[2] += n.flops
        flops += n.flops
out = {"batch": args.batch, "layers": args.layers, "budget": args.budget, "parity": parity,
       "no_eviction_ms": round(base_ms, 3), "delta_ms": round(delta_ms, 3),
       "ratio": round(base_ms / delta_ms, 4),
       "seq_per_s": round(args.batch / (delta_ms * 1e-3), 1),
       "tokens_per_s": round(args.batch * cfg.seq / (delta_ms * 1e-3), 0),
       "peak_act_gb": round(dp_.arena_bytes / 1e9, 3), "no_eviction_gb": round(bp.arena_bytes / 1e9, 3),
       "plan": dp_.plan_counts, "step_tflop": round(flops / 1e12, 3),
       "by_op": {k: {"n": v[0], "ms": round(v[1], 3),
                     "tflops": round(v[2] / (v[1] * 1e-3) / 1e12, 1) if v[2] else None}
                 for k, v in sorted(by_op.items(), key=lambda kv: -kv[1][1])}}
print(json.dumps(out))
