"""Host-side mirror of the reference `deltasim` interface for the DELTA path.

Same names, field meanings and error behaviour as the reference C++ API
(/root/reference/proj/include/deltasim/{trace,policy,engine,metrics}.hpp),
backed by libdelta through the C ABI.  `run_iteration` is the reference's
training-step executor entry (src/engine.cpp:627); `lower` is the B200
extension that turns the plan into an arena/stream action program.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from ._lib import (DeltaAction, DeltaConfig, DeltaError, DeltaEvent,
                   DeltaProgramInfo, DeltaSummary, check, lib, take_string)


class Phase(enum.IntEnum):
    Forward = 0
    Backward = 1


class AccessKind(enum.IntEnum):
    Produce = 0
    Use = 1


class Heuristic(enum.IntEnum):
    Base = 0
    Lru = 1
    Greedy = 2


class PolicyMode(enum.IntEnum):
    Delta = 0
    RecomputeOnly = 1
    OffloadOnly = 2
    Baseline = 3


class ReleaseAction(enum.IntEnum):
    Evict = 0
    Offload = 1


class SwapCostMode(enum.IntEnum):
    OneWay = 0
    RoundTrip = 1


class PrefetchGuard(enum.IntEnum):
    And = 0
    PaperOr = 1


class EventKind(enum.IntEnum):
    Compute = 0
    Offload = 1
    Reload = 2
    Recompute = 3
    Stall = 4
    Evict = 5
    Use = 6
    Free = 7


class StreamKind(enum.IntEnum):
    Compute = 0
    Copy = 1


@dataclass
class OpNode:                      # ref include/deltasim/trace.hpp:14-23
    id: int
    name: str
    compute_cost_us: int
    output_bytes: int
    parents: list = field(default_factory=list)
    uncomputable: bool = False
    evict_pinned: bool = False
    offload_pinned: bool = False


@dataclass
class AccessEvent:                 # ref include/deltasim/trace.hpp:25-31
    node: int
    phase: Phase = Phase.Forward
    kind: AccessKind = AccessKind.Produce


@dataclass
class Trace:                       # ref include/deltasim/trace.hpp:33-41
    name: str = ""
    nodes: list = field(default_factory=list)
    schedule: list = field(default_factory=list)

    def find(self, node_id: int) -> Optional[OpNode]:
        for n in self.nodes:
            if n.id == node_id:
                return n
        return None

    def to_json(self) -> str:
        """Canonical JSON (serialize_trace, ref src/trace.cpp:288)."""
        h = _CTrace(self)
        try:
            p, n = C.c_void_p(), C.c_uint64()
            check(lib.delta_trace_serialize(h.ptr, C.byref(p), C.byref(n)))
            return take_string(p, n.value)
        finally:
            h.close()

    @staticmethod
    def from_json(text: str) -> "Trace":
        """parse_trace (ref src/trace.cpp:211): strict schema + validation."""
        b = text.encode()
        h = C.c_void_p()
        check(lib.delta_trace_parse(b, len(b), C.byref(h)))
        lib.delta_trace_free(h)
        d = json.loads(text)
        t = Trace(d["name"])
        for n in d["nodes"]:
            t.nodes.append(OpNode(n["id"], n["name"], n["compute_cost_us"], n["output_bytes"],
                                  list(n["parents"]), n["uncomputable"], n["evict_pinned"],
                                  n["offload_pinned"]))
        for e in d["schedule"]:
            t.schedule.append(AccessEvent(e["node"], Phase(0 if e["phase"] == "F" else 1),
                                          AccessKind(0 if e["kind"] == "P" else 1)))
        return t

    def validate(self):
        """(n_errors, n_warnings, first_error) — validate_trace (src/trace.cpp:58)."""
        h = _CTrace(self)
        try:
            ne, nw, p = C.c_uint32(), C.c_uint32(), C.c_void_p()
            check(lib.delta_trace_validate(h.ptr, C.byref(ne), C.byref(nw), C.byref(p)))
            msg = None
            if p.value:
                msg = C.string_at(p).decode()
                lib.delta_free(p)
            return ne.value, nw.value, msg
        finally:
            h.close()


class _CTrace:
    """Owned delta_trace handle built from a Python Trace (no validation)."""

    def __init__(self, t: Trace):
        self.ptr = C.c_void_p()
        check(lib.delta_trace_new(t.name.encode(), C.byref(self.ptr)))
        try:
            for n in t.nodes:
                par = (C.c_uint64 * max(1, len(n.parents)))(*n.parents)
                flags = (1 if n.uncomputable else 0) | (2 if n.evict_pinned else 0) | \
                        (4 if n.offload_pinned else 0)
                check(lib.delta_trace_add_node(self.ptr, n.id, n.name.encode(),
                                               int(n.compute_cost_us), int(n.output_bytes),
                                               par, len(n.parents), flags))
            for e in t.schedule:
                check(lib.delta_trace_add_event(self.ptr, e.node, int(e.phase), int(e.kind)))
        except BaseException:
            self.close()
            raise

    def close(self):
        if self.ptr:
            lib.delta_trace_free(self.ptr)
            self.ptr = C.c_void_p()


@dataclass
class CostModel:                   # ref include/deltasim/policy.hpp:18-26
    bandwidth_bytes_per_us: tuple = (64000, 1)
    effective_fraction: tuple = (7, 20)
    swap_cost_mode: SwapCostMode = SwapCostMode.OneWay


@dataclass
class EngineConfig:                # ref include/deltasim/engine.hpp:26-42
    budget: int = 0
    heuristic: Heuristic = Heuristic.Base
    policy_mode: PolicyMode = PolicyMode.Delta
    cost_model: CostModel = field(default_factory=CostModel)
    watermark_fraction: tuple = (3, 4)
    prefetch_limit: int = 2
    prefetch_enabled: bool = True
    overlap_enabled: bool = True
    prefetch_guard: PrefetchGuard = PrefetchGuard.And
    scripted_decisions: list = field(default_factory=list)

    def watermark_bytes(self) -> int:
        return self.budget * self.watermark_fraction[0] // self.watermark_fraction[1]

    def to_c(self):
        c = DeltaConfig()
        c.budget = self.budget
        c.heuristic = int(self.heuristic)
        c.policy_mode = int(self.policy_mode)
        c.bw_num, c.bw_den = self.cost_model.bandwidth_bytes_per_us
        c.eff_num, c.eff_den = self.cost_model.effective_fraction
        c.swap_cost_mode = int(self.cost_model.swap_cost_mode)
        c.prefetch_guard = int(self.prefetch_guard)
        c.watermark_num, c.watermark_den = self.watermark_fraction
        c.prefetch_limit = self.prefetch_limit
        c.prefetch_enabled = 1 if self.prefetch_enabled else 0
        c.overlap_enabled = 1 if self.overlap_enabled else 0
        keep = []
        if self.scripted_decisions:
            nodes = (C.c_uint64 * len(self.scripted_decisions))(*[n for n, _ in self.scripted_decisions])
            acts = (C.c_uint32 * len(self.scripted_decisions))(*[int(a) for _, a in self.scripted_decisions])
            c.scripted_nodes = C.cast(nodes, C.POINTER(C.c_uint64))
            c.scripted_actions = C.cast(acts, C.POINTER(C.c_uint32))
            c.n_scripted = len(self.scripted_decisions)
            keep = [nodes, acts]
        return c, keep


EVENT_DTYPE = np.dtype([("ts", "<u8"), ("node", "<u8"), ("duration", "<u8"), ("bytes", "<u8"),
                        ("burst", "<u4"), ("stream", "u1"), ("kind", "u1"), ("phase", "u1"),
                        ("prefetch", "u1")])
ACTION_DTYPE = np.dtype([("op", "<u4"), ("stream", "<u4"), ("node", "<u8"), ("offset", "<u8"),
                         ("bytes", "<u8"), ("host_offset", "<u8"), ("event", "<u4"),
                         ("n_inputs", "<u4"), ("inputs_at", "<u8"), ("plan_event", "<u8")])
assert EVENT_DTYPE.itemsize == C.sizeof(DeltaEvent)
assert ACTION_DTYPE.itemsize == C.sizeof(DeltaAction)


class RunResult:
    """Owned delta_result: the plan (ref RunResult, engine.hpp:97-113)."""

    def __init__(self, ptr: C.c_void_p):
        self._ptr = ptr
        s = DeltaSummary()
        check(lib.delta_result_summary(ptr, C.byref(s)))
        self.peak_bytes = s.peak_bytes
        self.wall_time_us = s.wall_time_us
        self.total_stall_us = s.total_stall_us
        self.copy_busy_us = s.copy_busy_us
        self.copy_stall_us = s.copy_stall_us
        self.counts = dict(evict=s.evict, offload=s.offload, reload=s.reload,
                           recompute=s.recompute, prefetch_reload=s.prefetch_reload,
                           recompute_of_swapout=s.recompute_of_swapout)
        self.infeasible = (s.infeasible_node, s.infeasible_deficit) if s.infeasible else None
        n = C.c_uint64()
        ev = lib.delta_result_events(ptr, C.byref(n))
        self.events = (np.ctypeslib.as_array(C.cast(ev, C.POINTER(C.c_uint8)),
                                             shape=(n.value * EVENT_DTYPE.itemsize,))
                       .view(EVENT_DTYPE).copy() if n.value else np.zeros(0, EVENT_DTYPE))
        dp = lib.delta_result_decisions(ptr, C.byref(n))
        self.decisions = [(dp[i].node, ReleaseAction(dp[i].action)) for i in range(n.value)]

    def completed(self) -> bool:
        return self.infeasible is None

    def chrome_trace(self) -> str:
        """timeline_to_chrome_trace (ref src/metrics.cpp:255)."""
        p, n = C.c_void_p(), C.c_uint64()
        check(lib.delta_chrome_trace(self._ptr, C.byref(p), C.byref(n)))
        return take_string(p, n.value)

    def __del__(self):
        if getattr(self, "_ptr", None) and lib is not None:
            lib.delta_result_free(self._ptr)
            self._ptr = None


def chrome_trace_events(events: np.ndarray) -> str:
    """timeline_to_chrome_trace of an EVENT_DTYPE array (ref src/metrics.cpp:255)."""
    ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    p, n = C.c_void_p(), C.c_uint64()
    check(lib.delta_chrome_trace_events(ev.ctypes.data_as(C.c_void_p), len(ev), C.byref(p),
                                        C.byref(n)))
    return take_string(p, n.value)


def _plan(fn, trace: Trace, cfg: EngineConfig) -> RunResult:
    h = _CTrace(trace)
    try:
        c, keep = cfg.to_c()
        out = C.c_void_p()
        check(fn(h.ptr, C.byref(c), C.byref(out)))
        return RunResult(out)
    finally:
        h.close()


def run_iteration(trace: Trace, cfg: EngineConfig) -> RunResult:
    """ref src/engine.cpp:627 — validates, then plans one training step."""
    return _plan(lib.delta_plan, trace, cfg)


def run_unconstrained_baseline(trace: Trace, cfg: EngineConfig) -> RunResult:
    """ref src/engine.cpp:635 — Baseline policy, budget = sum of output bytes."""
    return _plan(lib.delta_plan_baseline, trace, cfg)


def report_json(run: RunResult, baseline: RunResult) -> str:
    """report_to_json(summarize(run, baseline)) (ref src/metrics.cpp:132,159)."""
    p, n = C.c_void_p(), C.c_uint64()
    check(lib.delta_report_json(run._ptr, baseline._ptr, C.byref(p), C.byref(n)))
    return take_string(p, n.value)


def comparison(trace: Trace, budgets, policies, heuristics, base: EngineConfig | None = None,
               fmt: str = "csv") -> str:
    """run_comparison + comparison_to_csv / _json (ref src/engine.cpp:646-671,
    src/metrics.cpp:314-348): the planned budget x policy x heuristic grid."""
    base = base or EngineConfig()
    h = _CTrace(trace)
    try:
        c, keep = base.to_c()
        b = (C.c_uint64 * max(1, len(budgets)))(*budgets)
        pm = (C.c_uint32 * max(1, len(policies)))(*[int(x) for x in policies])
        hm = (C.c_uint32 * max(1, len(heuristics)))(*[int(x) for x in heuristics])
        p, n = C.c_void_p(), C.c_uint64()
        check(lib.delta_comparison(h.ptr, C.byref(c), b, len(budgets), pm, len(policies), hm,
                                   len(heuristics), int(fmt == "json"), C.byref(p), C.byref(n)))
        return take_string(p, n.value)
    finally:
        h.close()


def plan_time_ns(trace: Trace, cfg: EngineConfig, iters: int = 1000) -> float:
    h = _CTrace(trace)
    try:
        c, keep = cfg.to_c()
        out = C.c_double()
        check(lib.delta_plan_time_ns(h.ptr, C.byref(c), iters, C.byref(out)))
        return out.value
    finally:
        h.close()


def transfer_time_us(nbytes: int, cfg: EngineConfig) -> int:
    c, keep = cfg.to_c()
    out = C.c_uint64()
    check(lib.delta_transfer_time_us(nbytes, C.byref(c), C.byref(out)))
    return out.value


# ---- B200 extension: plan -> arena action program -------------------------

ACT_COMPUTE, ACT_RECOMPUTE, ACT_OFFLOAD, ACT_RELOAD, ACT_RECORD, ACT_WAIT = range(6)
STREAM_COMPUTE, STREAM_D2H, STREAM_H2D = range(3)
LOWER_DUPLEX_COPIES = 1


class Program:
    """Lowered plan: arena offsets + action list on the compute stream and the
    copy stream(s) (csrc/rt/lower.cpp).  duplex=False (default): every copy on
    one copy stream in plan order, the reference's single copy stream;
    duplex=True: reloads on a second copy engine, concurrent with offloads."""

    def __init__(self, trace: Trace, cfg: EngineConfig, align: int = 256, duplex: bool = False):
        h = _CTrace(trace)
        try:
            c, keep = cfg.to_c()
            self._ptr = C.c_void_p()
            check(lib.delta_lower_ex(h.ptr, C.byref(c), align, LOWER_DUPLEX_COPIES if duplex else 0,
                                     C.byref(self._ptr)))
        finally:
            h.close()
        info = DeltaProgramInfo()
        check(lib.delta_program_info_get(self._ptr, C.byref(info)))
        self.arena_bytes = info.arena_bytes
        self.pool_peak_bytes = info.pool_peak_bytes
        self.host_bytes = info.host_bytes
        self.n_events = info.n_events
        n = C.c_uint64()
        ap = lib.delta_program_actions(self._ptr, C.byref(n))
        raw = np.ctypeslib.as_array(C.cast(ap, C.POINTER(C.c_uint8)),
                                    shape=(n.value * ACTION_DTYPE.itemsize,))
        self.actions = raw.view(ACTION_DTYPE).copy()
        ip = lib.delta_program_inputs(self._ptr, C.byref(n))
        self.inputs = (np.ctypeslib.as_array(ip, shape=(n.value,)).copy()
                       if n.value else np.zeros(0, np.uint64))
        pp = lib.delta_program_plan(self._ptr)
        # borrow: summarise the plan without taking ownership
        s = DeltaSummary()
        check(lib.delta_result_summary(pp, C.byref(s)))
        self.infeasible = (s.infeasible_node, s.infeasible_deficit) if s.infeasible else None
        self.plan_counts = dict(evict=s.evict, offload=s.offload, reload=s.reload,
                                recompute=s.recompute, prefetch_reload=s.prefetch_reload)
        self.plan_peak_bytes = s.peak_bytes
        self.plan_wall_us = s.wall_time_us
        ne = C.c_uint64()
        dp = lib.delta_result_decisions(pp, C.byref(ne))
        self.decisions = [(dp[i].node, ReleaseAction(dp[i].action)) for i in range(ne.value)]

    def __del__(self):
        if getattr(self, "_ptr", None) and lib is not None:
            lib.delta_program_free(self._ptr)
            self._ptr = None


__all__ = [
    "Phase", "AccessKind", "Heuristic", "PolicyMode", "ReleaseAction", "SwapCostMode",
    "PrefetchGuard", "EventKind", "StreamKind", "OpNode", "AccessEvent", "Trace",
    "CostModel", "EngineConfig", "RunResult", "run_iteration", "run_unconstrained_baseline",
    "report_json", "comparison", "plan_time_ns", "transfer_time_us", "Program", "DeltaError",
    "chrome_trace_events",
]
