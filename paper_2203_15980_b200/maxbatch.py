"""Max-batch search (config 3: largest batch that trains under DELTA vs the
no-eviction baseline in the same HBM).

The planner decides feasibility exactly: a batch fits when the lowered plan's
arena (activation) footprint plus the batch-proportional workspace outside
the budget fits the HBM left after the persistent state.  Node costs come
from the GPU cost model measured at a reference batch and scale linearly in
the batch (every op is batch-parallel).  `verify` then runs real steps at the
found sizes.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import graph as G
from . import planner as P


@dataclass
class Fit:
    batch: int
    arena_bytes: int
    workspace_bytes: int
    anchors: str
    counts: dict | None = None


def resident_workspace_bytes(g: G.Graph, batch: int) -> int:
    """Batch-proportional buffers DeltaRuntime allocates up front, outside the
    activation budget (runtime.workspace_plan)."""
    from .runtime import workspace_plan
    ws = workspace_plan(g)
    return sum(v for k, v in ws.items() if k != "transient")


def transient_workspace_bytes(g: G.Graph, batch: int) -> int:
    """the stride-2 3x3 input-gradient scratch alive inside one backward node
    (runtime.workspace_plan's 'transient')."""
    from .runtime import workspace_plan
    return workspace_plan(g)["transient"]


def workspace_bytes(g: G.Graph, batch: int) -> int:
    return resident_workspace_bytes(g, batch) + transient_workspace_bytes(g, batch)


def _graph(depth, batch, anchors, costs_per_sample):
    from .runtime import apply_anchors
    g = G.build_resnet(depth, batch)
    apply_anchors(g, anchors)
    for n in g.nodes:
        n.cost_us = max(1, int(round(costs_per_sample.get(n.name, 1.0) * batch)))
    return g


def fits(depth, batch, capacity, anchors, costs_per_sample, link_bpus, delta: bool):
    g = _graph(depth, batch, anchors, costs_per_sample)
    ws = workspace_bytes(g, batch)
    room = capacity - ws
    if room <= 0:
        return None
    t = G.to_trace(g)
    cm = P.CostModel((link_bpus, 1), (1, 1))
    if delta:
        prog = P.Program(t, P.EngineConfig(budget=room, cost_model=cm), align=G.ALIGN)
    else:
        total = sum(n.nbytes for n in g.nodes)
        prog = P.Program(t, P.EngineConfig(budget=total, policy_mode=P.PolicyMode.Baseline,
                                           cost_model=cm), align=G.ALIGN)
    if prog.infeasible or prog.arena_bytes > room:
        return None
    return Fit(batch, prog.arena_bytes, ws, anchors, prog.plan_counts)


def per_sample_costs(depth: int, per50: dict) -> dict:
    """Per-sample node costs for ResNet-`depth` from ResNet-50's (same node
    names); blocks ResNet-50 lacks (layer3.6+) take layer3.1's costs."""
    if depth == 50:
        return dict(per50)
    g = G.build_resnet(depth, 1)
    out = {}
    for n in g.nodes:
        key = n.name
        if key not in per50 and key.startswith("layer3."):
            key = "layer3.1." + key.split(".", 2)[2]
        out[n.name] = per50.get(key, min(per50.values()))
    return out


def search(depth, capacity, costs_per_sample, link_bpus, delta: bool, anchors="out+narrow",
           lo=1, hi=65536, multiple=8) -> Fit | None:
    """Largest batch (multiple of `multiple`) that fits; binary search."""
    best = None
    lo_b, hi_b = max(1, lo // multiple), hi // multiple
    while lo_b <= hi_b:
        mid = (lo_b + hi_b) // 2
        f = fits(depth, mid * multiple, capacity, anchors, costs_per_sample, link_bpus, delta)
        if f is not None:
            best = f
            lo_b = mid + 1
        else:
            hi_b = mid - 1
    return best
