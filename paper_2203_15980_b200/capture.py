"""DELTA trace capture from an arbitrary PyTorch training step.

The ResNet trace the B200 runtime executes is registered by hand
(graph.py).  This module derives the same kind of trace from any model by
watching one training step at the ATen level:

* forward: every op that allocates a new tensor becomes a Produce node
  (ref OpNode, include/deltasim/trace.hpp:14-23): `output_bytes` = the bytes
  of its new storages, `parents` = the earlier nodes whose tensors it reads,
  `compute_cost_us` = the op's device time (CUDA events; CPU wall time when
  the step runs on the CPU) — exactly what a recompute of it costs;
* backward: every op of `loss.backward()` that allocates a gradient becomes a
  backward-phase Produce node whose parents are the saved activations and
  upstream gradients it reads (the trace format's backward Produce, SPEC.md:44;
  SURVEY F5), so saved-tensor reads are accesses the planner must honour;
* the step's inputs (the batch, the labels) are uncomputable, evict-pinned
  nodes; parameters, buffers, optimizer state and the parameter gradients are
  outside the activation budget (as in the paper) and are not nodes.

Views and in-place ops share their input's storage and therefore its node
(an in-place op's time is added to that node's cost).  The result is a
deltasim Trace the planner (and the reference simulator) accepts.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import torch
from torch.utils._python_dispatch import TorchDispatchMode
from torch.utils._pytree import tree_flatten

from . import planner as P


@dataclass
class CapturedNode:
    id: int
    name: str
    phase: str                      # "F" or "B"
    parents: list
    storages: dict = field(default_factory=dict)  # storage ptr -> bytes
    cost_us: float = 0.0
    shapes: list = field(default_factory=list)


def _storage_key(t: torch.Tensor):
    try:
        return t.untyped_storage().data_ptr()
    except Exception:  # noqa: BLE001 - tensors without storage (meta, sparse)
        return None


class _Recorder(TorchDispatchMode):
    def __init__(self, cap: "_Capture"):
        super().__init__()
        self.cap = cap

    def __torch_dispatch__(self, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        cap = self.cap
        flat_in, _ = tree_flatten((args, kwargs))
        ins = [t for t in flat_in if isinstance(t, torch.Tensor)]
        in_keys = {_storage_key(t) for t in ins}
        t0 = cap.clock_start()
        out = func(*args, **kwargs)
        dt = cap.clock_stop(t0)
        flat_out, _ = tree_flatten(out)
        outs = [t for t in flat_out if isinstance(t, torch.Tensor)]
        parents = []
        for t in ins:
            n = cap.node_of.get(_storage_key(t))
            if n is not None and n not in parents:
                parents.append(n)
        fresh = {}
        for t in outs:
            k = _storage_key(t)
            if k is None or k in in_keys or k in cap.excluded:
                continue  # a view / in-place result, or a parameter / buffer
            fresh[k] = t.untyped_storage().nbytes()
        if not fresh:
            # view or in-place: its time belongs to the node it aliases
            for t in outs:
                n = cap.node_of.get(_storage_key(t))
                if n is not None:
                    cap.pending_cost.append((n, dt))
                    break
            return out
        node = CapturedNode(len(cap.nodes), f"{len(cap.nodes)}:{func.__name__}", cap.phase,
                            parents, fresh, 0.0, [tuple(t.shape) for t in outs])
        cap.pending_cost.append((node.id, dt))
        cap.nodes.append(node)
        for k in fresh:
            cap.node_of[k] = node.id
        return out


class _Capture:
    def __init__(self, device: torch.device, timing: bool):
        self.device = device
        self.cuda = device.type == "cuda" and timing
        self.timing = timing
        self.nodes: list[CapturedNode] = []
        self.node_of: dict = {}
        self.excluded: set = set()
        self.phase = "F"
        self.pending_cost: list = []

    def clock_start(self):
        if not self.timing:
            return None
        if self.cuda:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            return e
        return time.perf_counter()

    def clock_stop(self, t0):
        if t0 is None:
            return None
        if self.cuda:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            return (t0, e)
        return (time.perf_counter() - t0) * 1e6

    def resolve_costs(self):
        if self.cuda:
            torch.cuda.synchronize()
        for nid, dt in self.pending_cost:
            if dt is None:
                continue
            us = dt[0].elapsed_time(dt[1]) * 1e3 if isinstance(dt, tuple) else dt
            self.nodes[nid].cost_us += us


def capture_trace(model: torch.nn.Module, inputs, loss_fn=None, *, name: str = "captured",
                  timing: bool = True, warmup: int = 1) -> tuple:
    """Watch one training step of `model` and return (Trace, [CapturedNode]).

    `inputs`: a tensor or tuple of tensors (the batch; uncomputable nodes).
    `loss_fn(output, *inputs) -> scalar` (default: output.float().mean()).
    Costs are measured on the device the inputs live on (`warmup` untimed
    steps first); with timing=False every node costs 1 µs."""
    if isinstance(inputs, torch.Tensor):
        inputs = (inputs,)
    if loss_fn is None:
        loss_fn = lambda out, *ins: out.float().mean()  # noqa: E731
    device = inputs[0].device
    for _ in range(warmup if timing else 0):
        model.zero_grad(set_to_none=True)
        loss_fn(model(*inputs[:1]), *inputs).backward()
    model.zero_grad(set_to_none=True)
    cap = _Capture(device, timing)
    for p in list(model.parameters()) + list(model.buffers()):
        cap.excluded.add(_storage_key(p))
    for i, t in enumerate(inputs):
        n = CapturedNode(len(cap.nodes), f"input{i}", "F", [], {_storage_key(t):
                                                               t.untyped_storage().nbytes()},
                         0.0, [tuple(t.shape)])
        cap.nodes.append(n)
        cap.node_of[_storage_key(t)] = n.id
    with _Recorder(cap):
        out = model(*inputs[:1])
        loss = loss_fn(out, *inputs)
        cap.phase = "B"
        loss.backward()
    cap.resolve_costs()
    # parameter gradients live outside the activation budget
    grads = {_storage_key(p.grad) for p in model.parameters() if p.grad is not None}
    for n in cap.nodes:
        for k in list(n.storages):
            if k in grads:
                del n.storages[k]
    return _to_trace(cap.nodes, len(inputs), name), cap.nodes


def _to_trace(nodes: list, n_inputs: int, name: str) -> P.Trace:
    """Drop nodes left without bytes (parameter-gradient-only ops) and no
    children, splice any with children out (their readers inherit their
    parents), renumber densely, emit forward then backward Produce events."""
    children = {n.id: 0 for n in nodes}
    for n in nodes:
        for p in n.parents:
            children[p] += 1
    keep, remap, alias = [], {}, {}
    for n in nodes:
        parents = []
        for p in n.parents:
            for q in alias.get(p, [p]):
                if q not in parents:
                    parents.append(q)
        n.parents = parents
        if sum(n.storages.values()) == 0:
            alias[n.id] = parents  # empty node: its readers depend on its parents
            continue
        keep.append(n)
    t = P.Trace(name)
    for n in keep:
        remap[n.id] = len(remap)
    for n in keep:
        is_input = n.id < n_inputs
        t.nodes.append(P.OpNode(remap[n.id], n.name, max(1, int(math.ceil(n.cost_us))),
                                int(sum(n.storages.values())),
                                [remap[p] for p in n.parents if p in remap],
                                uncomputable=is_input, evict_pinned=is_input))
    for ph, phase in (("F", P.Phase.Forward), ("B", P.Phase.Backward)):
        for n in keep:
            if n.phase == ph:
                t.schedule.append(P.AccessEvent(remap[n.id], phase, P.AccessKind.Produce))
    return t
