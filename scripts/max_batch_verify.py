"""Config 3: largest batch that trains on one B200, no-eviction vs DELTA.
Planner search (paper_2203_15980_b200.maxbatch) with capacity = free HBM
after the persistent state, then two real training steps at each found size.
Costs: per-sample costs of the measured bs256 ResNet-50 trace (tests/golden),
scaled linearly; ResNet-101's extra layer3 blocks reuse layer3.1's costs."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_15980_b200 import graph as G  # noqa: E402
from paper_2203_15980_b200 import kernels as K  # noqa: E402
from paper_2203_15980_b200 import maxbatch as MB  # noqa: E402
from paper_2203_15980_b200.runtime import DeltaRuntime  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tr = json.load(open(os.path.join(ROOT, "tests/golden/resnet50_bs256_trace.json")))
per = {n["name"]: n["compute_cost_us"] / 256 for n in tr["nodes"]}


def per_sample(depth):
    return MB.per_sample_costs(depth, per)


def run(depth, batch, anchors, delta, steps=2):
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    rt = DeltaRuntime(depth, batch, seed=0, anchors=anchors)
    ps = per_sample(depth)
    for n in rt.nodes:
        n.cost_us = max(1, int(round(ps.get(n.name, 1 / 256) * batch)))
    rt.link_gbs = LINK
    free = torch.cuda.mem_get_info()[0]  # runtime buffers already allocated
    room = free - MB.transient_workspace_bytes(rt.g, batch) - MARGIN
    if delta:
        prog = rt.plan(budget=room)
    else:
        prog = rt.plan(None)
    x = torch.zeros(rt.x_dev.shape, dtype=torch.bfloat16)
    y = torch.randint(0, 1000, (batch,))
    t0 = time.time()
    losses = [rt.step(x, y) for _ in range(steps)]
    torch.cuda.synchronize()
    dt = (time.time() - t0) / steps
    res = dict(depth=depth, batch=batch, anchors=anchors, delta=delta,
               arena_gb=round(prog.arena_bytes / 1e9, 2), counts=prog.plan_counts,
               peak_alloc_gb=round(torch.cuda.max_memory_allocated() / 1e9, 2),
               img_s=round(batch / dt, 1), loss=losses[-1])
    del rt, prog
    import gc
    gc.collect()  # the executor's host callbacks close a reference cycle
    torch.cuda.empty_cache()
    return res


LINK = min(K.probe_link()[:2])
MARGIN = 6 * 2**30  # cuDNN workspace + allocator slack
total = torch.cuda.get_device_properties(0).total_memory
out = {"gpu_total_gb": round(total / 1e9, 1), "link_gbs": round(LINK, 2), "results": []}
for depth in (50, 101):
    free = torch.cuda.mem_get_info()[0] - MARGIN - 2 * 2**30  # params/optimizer (~0.4 GB) + slack
    b = MB.search(depth, free, per_sample(depth), int(LINK * 1e3), delta=False)
    d = MB.search(depth, free, per_sample(depth), int(LINK * 1e3), delta=True, anchors="out")
    if b is None or d is None:
        print(json.dumps(dict(depth=depth, error="no feasible batch", free_gb=free / 1e9)))
        continue
    entry = dict(depth=depth, planned_no_eviction=b.batch, planned_delta=d.batch,
                 ratio=round(d.batch / b.batch, 3))
    try:
        entry["run_no_eviction"] = run(depth, b.batch, "out", False)
    except Exception as e:
        entry["run_no_eviction"] = dict(error=str(e)[:300])
    try:
        entry["run_delta"] = run(depth, d.batch, "out", True)
    except Exception as e:
        entry["run_delta"] = dict(error=str(e)[:300])
    out["results"].append(entry)
    print(json.dumps(entry), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "max_batch.json"), "w"), indent=1)
