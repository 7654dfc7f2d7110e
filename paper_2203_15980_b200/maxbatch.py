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
    activation budget: input staging, BN-statistics partials (2 scratch
    buffers), maxpool argmax scratch, head gradients."""
    x = g.nodes[0].nbytes
    convs = [n for n in g.nodes if n.op == "conv"]
    parts = 2 * max((((n.shape[0] * n.shape[1] * n.shape[2] + 127) // 128) * 33 // 32 + 1)
                    * n.shape[3] * 8 for n in convs)
    mp = next(n for n in g.nodes if n.op == "maxpool")
    return x + parts + mp.nbytes // 2 + batch * 1000 * 8


def transient_workspace_bytes(g: G.Graph, batch: int) -> int:
    """cuDNN dgrad outputs alive at once during a backward node (conv1 +
    downsample input gradients of a block)."""
    convs = [n for n in g.nodes if n.op == "conv"]
    return 2 * max(g.nodes[n.parents[0]].nbytes for n in convs)


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
