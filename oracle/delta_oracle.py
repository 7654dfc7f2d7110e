"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of the reference DELTA
simulator's hot path (the training-step executor and its Filter/Director).

Restates /root/reference/proj/src/{engine,policy,state,device,metrics}.cpp;
every function cites the file:line it follows.  It is the checker for the
libdelta planner on machines where oracle/_ref (the reference itself, built
from source) is not available, and it is pinned against the reference's golden
vectors (tests/golden/*, tests/test_oracle_cpu.py).  Python integers make the
U128 products of the reference exact without emulation.

Never imported by the product package.
"""
from __future__ import annotations

import heapq
import json
from dataclasses import dataclass, field

# enums (ref include/deltasim/engine.hpp, policy.hpp, state.hpp)
FORWARD, BACKWARD = 0, 1
PRODUCE, USE = 0, 1
BASE, LRU, GREEDY = 0, 1, 2
DELTA, RECOMPUTE_ONLY, OFFLOAD_ONLY, BASELINE = 0, 1, 2, 3
EVICT, OFFLOAD = 0, 1
COMPUTE_S, COPY_S = 0, 1
K_COMPUTE, K_OFFLOAD, K_RELOAD, K_RECOMPUTE, K_STALL, K_EVICT, K_USE, K_FREE = range(8)
KIND_NAMES = ["Compute", "Offload", "Reload", "Recompute", "Stall", "Evict", "Use", "Free"]


class Infeasible(Exception):
    def __init__(self, node, deficit):
        super().__init__(f"infeasible at {node} deficit {deficit}")
        self.node, self.deficit = node, deficit


class IllegalTransition(Exception):
    pass


class Unrecoverable(Exception):
    pass


@dataclass
class Node:
    id: int
    name: str
    cost: int
    bytes: int
    parents: list
    uncomputable: bool = False
    evict_pinned: bool = False
    offload_pinned: bool = False


@dataclass
class OTrace:
    name: str
    nodes: list
    schedule: list  # (node, phase, kind)


@dataclass
class OConfig:
    budget: int = 0
    heuristic: int = BASE
    policy: int = DELTA
    bw: tuple = (64000, 1)
    eff: tuple = (7, 20)
    round_trip: bool = False
    watermark: tuple = (3, 4)
    prefetch_limit: int = 2
    prefetch_enabled: bool = True
    overlap_enabled: bool = True
    paper_or: bool = False
    scripted: list = field(default_factory=list)

    def eff_num(self):  # ref src/policy.cpp:26-29
        return self.bw[0] * self.eff[0]

    def eff_den(self):  # ref src/policy.cpp:31-34
        return self.bw[1] * self.eff[1]

    def watermark_bytes(self):  # ref src/engine.cpp:35-38
        return self.budget * self.watermark[0] // self.watermark[1]


def trace_from_json(text: str) -> OTrace:
    d = json.loads(text)
    nodes = [Node(n["id"], n["name"], n["compute_cost_us"], n["output_bytes"], list(n["parents"]),
                  n["uncomputable"], n["evict_pinned"], n["offload_pinned"]) for n in d["nodes"]]
    sched = [(e["node"], FORWARD if e["phase"] == "F" else BACKWARD,
              PRODUCE if e["kind"] == "P" else USE) for e in d["schedule"]]
    return OTrace(d["name"], nodes, sched)


def config_from(cfg) -> OConfig:
    """From a paper_2203_15980_b200.planner.EngineConfig-like object."""
    return OConfig(cfg.budget, int(cfg.heuristic), int(cfg.policy_mode),
                   tuple(cfg.cost_model.bandwidth_bytes_per_us),
                   tuple(cfg.cost_model.effective_fraction),
                   int(cfg.cost_model.swap_cost_mode) == 1, tuple(cfg.watermark_fraction),
                   cfg.prefetch_limit, bool(cfg.prefetch_enabled), bool(cfg.overlap_enabled),
                   int(cfg.prefetch_guard) == 1,
                   [(n, int(a)) for n, a in cfg.scripted_decisions])


def transfer_time_us(m: int, cfg: OConfig) -> int:
    """ceil(m * eff_den / eff_num) — ref src/policy.cpp:58-64."""
    num, den = cfg.eff_num(), cfg.eff_den()
    return (m * den + num - 1) // num


class Rec:
    """TensorRecord (ref include/deltasim/state.hpp:30-51)."""
    __slots__ = ("id", "bytes", "cost", "on_gpu", "evicted", "swapout", "uncomputable",
                 "evict_pinned", "offload_pinned", "in_use", "copy_in_flight",
                 "cpu_copy_valid", "produced_backward", "dead", "died_swapout", "last_access")

    def __init__(self, n: Node, now: int, backward: bool):
        self.id, self.bytes, self.cost = n.id, n.bytes, n.cost
        self.on_gpu = True
        self.evicted = self.swapout = self.in_use = self.copy_in_flight = False
        self.cpu_copy_valid = self.dead = self.died_swapout = False
        self.uncomputable, self.evict_pinned = n.uncomputable, n.evict_pinned
        self.offload_pinned = n.offload_pinned
        self.produced_backward = backward
        self.last_access = now


def transition(r: Rec, ev: str, now: int) -> None:
    """Legal state machine, in place — ref src/state.cpp:58-141."""
    ok = True
    if ev == "Use":
        ok = r.on_gpu and not r.dead
        r.last_access = now
    elif ev == "EvictStart":
        ok = (r.on_gpu and not r.evict_pinned and not r.in_use and not r.uncomputable
              and not r.copy_in_flight and not r.dead)
        r.on_gpu, r.evicted, r.cpu_copy_valid = False, True, False
    elif ev == "OffloadStart":
        ok = r.on_gpu and not r.offload_pinned and not r.in_use and not r.copy_in_flight and not r.dead
        r.copy_in_flight = True
    elif ev == "OffloadDone":
        ok = r.on_gpu and r.copy_in_flight
        r.copy_in_flight, r.cpu_copy_valid = False, True
    elif ev == "FreeAfterOffload":
        ok = r.on_gpu and r.cpu_copy_valid and not r.copy_in_flight and not r.in_use
        r.on_gpu, r.swapout = False, True
    elif ev == "ReloadStart":
        ok = (r.swapout or r.dead) and r.cpu_copy_valid and not r.copy_in_flight
        r.copy_in_flight = True
    elif ev == "ReloadDone":
        ok = (r.swapout or r.dead) and r.copy_in_flight
        r.on_gpu, r.swapout, r.copy_in_flight, r.dead = True, False, False, False
        r.last_access = now
    elif ev == "RecomputeDone":
        ok = (not (r.on_gpu or r.in_use or r.copy_in_flight or r.uncomputable)
              and (r.evicted or r.swapout or r.dead))
        r.on_gpu, r.evicted, r.swapout, r.cpu_copy_valid, r.dead = True, False, False, False, False
        r.last_access = now
    elif ev == "FreeDead":
        ok = not (r.in_use or r.copy_in_flight or r.dead)
        r.died_swapout = r.swapout
        r.on_gpu = r.evicted = r.swapout = False
        r.dead = True
    if not ok:
        raise IllegalTransition(f"{ev} on node {r.id}")


def releasable(r: Rec) -> bool:
    """ref src/policy.cpp:111-114."""
    return (r.on_gpu and not r.in_use and not r.copy_in_flight and not r.dead
            and not r.produced_backward and not (r.evict_pinned and r.offload_pinned))


@dataclass
class Result:
    events: list
    decisions: list
    infeasible: tuple | None
    peak_bytes: int
    wall_time_us: int
    total_stall_us: int
    copy_busy_us: int
    copy_stall_us: int
    counts: dict


class Engine:
    """ref src/engine.cpp:73-623."""

    def __init__(self, t: OTrace, cfg: OConfig):
        self.t, self.cfg = t, cfg
        self.node = {n.id: n for n in t.nodes}
        self.pos = {n.id: i for i, n in enumerate(t.nodes)}
        self._index()                                   # ref 126-173
        self.now = 0                                    # Clock
        self.used = self.high = 0                       # MemoryPool
        self.compute_busy = self.copy_busy_until = 0    # Streams
        self.compute_submits = 0
        self.set: dict[int, Rec] = {}
        self.queue: list[int] = []
        self.events: list = []
        self.pending: list = []
        self.inflight_done: dict[int, int] = {}
        self.pin_count = {n.id: 0 for n in t.nodes}
        self.dead_pending = {n.id: False for n in t.nodes}
        self.restored: list[int] = []
        self.decisions: list = []
        self.phase = FORWARD
        self.inflight_release = 0
        self.seq = 0
        self.burst = 0
        self.scripted_pos = 0
        self.counts = dict(evict=0, offload=0, reload=0, recompute=0, prefetch_reload=0,
                           recompute_of_swapout=0)
        self.total_stall = self.copy_busy = self.copy_stall = 0

    def _index(self):
        n = len(self.t.nodes)
        last = {x.id: -1 for x in self.t.nodes}
        for k, (nid, ph, kind) in enumerate(self.t.schedule):
            last[nid] = max(last[nid], k)
            if kind == PRODUCE:
                for p in self.node[nid].parents:
                    last[p] = max(last[p], k)
        ext = dict(last)
        for i in range(n - 1, -1, -1):  # ref 150-157
            c = self.t.nodes[i]
            for p in c.parents:
                if ext[c.id] > ext[p]:
                    ext[p] = ext[c.id]
        self.last, self.ext = last, ext
        self.death = [[] for _ in self.t.schedule]
        for x in self.t.nodes:  # ref 160-170
            if last[x.id] >= 0:
                self.death[last[x.id]].append(x.id)
            if x.uncomputable and ext[x.id] > last[x.id]:
                self.death[ext[x.id]].append(x.id)

    # ---- pool / streams / log ----
    def try_alloc(self, b):
        if b > self.cfg.budget - self.used:
            return False
        self.used += b
        self.high = max(self.high, self.used)
        return True

    def free(self, b):
        assert b <= self.used
        self.used -= b

    def submit_compute(self, d):
        start = max(self.now, self.compute_busy)
        self.compute_busy = start + d
        self.compute_submits += 1
        return start

    def submit_copy(self, d):
        start = max(self.now, self.copy_busy_until)
        self.copy_busy_until = start + d
        return start

    def log(self, kind, ts, dur, node, b, stream, pf=False, burst=0):
        self.events.append((ts, stream, kind, node, dur, b, self.phase, 1 if pf else 0, burst))

    def drain(self, up_to):  # ref 204-234
        while self.pending and self.pending[0][0] <= up_to:
            ts, _seq, offload, node, b = heapq.heappop(self.pending)
            r = self.set[node]
            if offload:
                transition(r, "OffloadDone", ts)
                transition(r, "FreeAfterOffload", ts)
                self.free(b)
                self.inflight_release -= b
                if self.dead_pending[node]:
                    self.dead_pending[node] = False
                    transition(r, "FreeDead", ts)
                else:
                    self.queue.append(node)
            else:
                transition(r, "ReloadDone", ts)
                if self.dead_pending[node]:
                    self.dead_pending[node] = False
                    self.free(b)
                    transition(r, "FreeDead", ts)
                    self.log(K_FREE, ts, 0, node, b, COMPUTE_S)
                else:
                    self.restored.append(node)

    def stall_until(self, t, cause):  # ref 237-246
        before = self.now
        if t > self.now:
            waited = t - self.now
            self.now = t
            self.log(K_STALL, before, waited, cause, 0, COMPUTE_S)
            self.total_stall += waited
            self.copy_stall += waited
        self.drain(self.now)

    # ---- release machinery (ref 250-362) ----
    def releases_allowed(self):
        return self.phase == FORWARD and self.cfg.policy != BASELINE

    def committed_used(self):
        return self.used - self.inflight_release

    def select_victim(self, extra=None):  # ref src/policy.cpp:121-136
        best, best_inv = None, 0
        for nid in sorted(self.set):
            r = self.set[nid]
            if not releasable(r) or (extra and not extra(r)):
                continue
            s = self.now - r.last_access if self.now > r.last_access else 1  # ref state.cpp:35-42
            inv = r.bytes * s if self.cfg.heuristic == BASE else (
                s if self.cfg.heuristic == LRU else r.bytes)
            if best is None or inv > best_inv:
                best, best_inv = nid, inv
        return best

    def recompute_cost(self, nid):  # ref src/policy.cpp:75-109
        total = self.node[nid].cost
        seen = set()
        stack = list(self.node[nid].parents)
        while stack:
            p = stack.pop()
            if p in seen:
                continue
            r = self.set[p]
            if r.on_gpu or r.swapout:
                continue
            if self.node[p].uncomputable:
                if r.cpu_copy_valid:
                    continue
                raise Unrecoverable(f"closure of {nid} reaches lost {p}")
            seen.add(p)
            total += self.node[p].cost
            stack.extend(self.node[p].parents)
        return total

    def decide(self, nid):  # ref src/policy.cpp:138-158
        r = self.set[nid]
        if r.evict_pinned:
            return OFFLOAD
        if r.offload_pinned:
            return EVICT
        num = self.recompute_cost(nid) * self.cfg.eff_num()
        den = r.bytes * self.cfg.eff_den() * (2 if self.cfg.round_trip else 1)
        return EVICT if num <= den else OFFLOAD

    def release_one(self):  # ref 259-333
        now = self.now
        if self.scripted_pos < len(self.cfg.scripted):
            victim, action = self.cfg.scripted[self.scripted_pos]
            self.scripted_pos += 1
        else:
            pol = self.cfg.policy
            if pol == BASELINE:
                return False
            extra = (lambda r: not r.evict_pinned and not r.uncomputable) if pol == RECOMPUTE_ONLY \
                else (lambda r: not r.offload_pinned) if pol == OFFLOAD_ONLY else None
            victim = self.select_victim(extra)
            if victim is None:
                return False
            action = self.decide(victim) if pol == DELTA else (
                EVICT if pol == RECOMPUTE_ONLY else OFFLOAD)
        self.decisions.append((victim, action))
        r = self.set[victim]
        b = r.bytes
        if action == EVICT:
            transition(r, "EvictStart", now)
            self.free(b)
            self.counts["evict"] += 1
            self.log(K_EVICT, now, 0, victim, b, COMPUTE_S)
            return True
        d = transfer_time_us(b, self.cfg)
        transition(r, "OffloadStart", now)
        self.counts["offload"] += 1
        self.copy_busy += d
        if self.cfg.overlap_enabled:
            start = self.submit_copy(d)
            self.log(K_OFFLOAD, start, d, victim, b, COPY_S)
            heapq.heappush(self.pending, (start + d, self.seq, True, victim, b))
            self.seq += 1
            self.inflight_done[victim] = start + d
            self.inflight_release += b
        else:
            start = self.submit_compute(d)
            self.log(K_OFFLOAD, start, d, victim, b, COMPUTE_S)
            self.now = max(self.now, start + d)
            self.copy_stall += d
            transition(r, "OffloadDone", start + d)
            transition(r, "FreeAfterOffload", start + d)
            self.free(b)
            self.queue.append(victim)
        return True

    def watermark_loop(self):  # ref 335-340
        mark = self.cfg.watermark_bytes()
        while self.committed_used() > mark:
            if not self.release_one():
                break

    def alloc_bytes(self, n, for_node):  # ref 344-362
        self.drain(self.now)
        while self.cfg.budget - self.used < n:
            covered = self.cfg.budget - self.committed_used() >= n
            if not covered and self.releases_allowed() and self.release_one():
                continue
            if self.pending:
                ts, _s, _o, node, _b = self.pending[0]
                self.stall_until(ts, node)
                continue
            raise Infeasible(for_node, n - (self.cfg.budget - self.used))
        assert self.try_alloc(n)
        if self.releases_allowed():
            self.watermark_loop()

    # ---- residency (ref 372-454) ----
    def ensure_resident(self, nid, closure_dep=False):
        self.drain(self.now)
        r = self.set[nid]
        if r.on_gpu and r.copy_in_flight:
            self.stall_until(self.inflight_done[nid], nid)
        if r.on_gpu:
            return
        if r.swapout and r.copy_in_flight:
            self.stall_until(self.inflight_done[nid], nid)
            return
        host_ok = r.swapout or (r.dead and r.cpu_copy_valid)
        if host_ok and (r.uncomputable or closure_dep):
            self.demand_reload(nid)
            return
        self.rebuild(nid)

    def demand_reload(self, nid):  # ref 396-419
        r = self.set[nid]
        b = r.bytes
        self.alloc_bytes(b, nid)
        d = transfer_time_us(b, self.cfg)
        transition(r, "ReloadStart", self.now)
        if nid in self.queue:
            self.queue.remove(nid)
        self.counts["reload"] += 1
        self.copy_busy += d
        if self.cfg.overlap_enabled:
            start = self.submit_copy(d)
            self.log(K_RELOAD, start, d, nid, b, COPY_S)
            heapq.heappush(self.pending, (start + d, self.seq, False, nid, b))
            self.seq += 1
            self.inflight_done[nid] = start + d
            self.stall_until(start + d, nid)
        else:
            start = self.submit_compute(d)
            self.log(K_RELOAD, start, d, nid, b, COMPUTE_S)
            self.now = max(self.now, start + d)
            self.copy_stall += d
            transition(r, "ReloadDone", start + d)
            self.restored.append(nid)

    def rebuild(self, nid):  # ref 423-454
        node = self.node[nid]
        r = self.set[nid]
        if node.uncomputable:
            if r.cpu_copy_valid:
                self.demand_reload(nid)
                return
            raise Unrecoverable(f"node {nid} lost")
        held = []
        for p in node.parents:
            self.ensure_resident(p, closure_dep=True)
            self.pin(p, held)
        was_swapout = r.swapout
        if was_swapout and nid in self.queue:
            self.queue.remove(nid)
        self.alloc_bytes(node.bytes, nid)
        start = self.submit_compute(node.cost)
        self.now = max(self.now, start + node.cost)
        self.log(K_RECOMPUTE, start, node.cost, nid, node.bytes, COMPUTE_S)
        for p in node.parents:
            transition(self.set[p], "Use", start + node.cost)
        transition(r, "RecomputeDone", start + node.cost)
        self.counts["recompute"] += 1
        if was_swapout:
            self.counts["recompute_of_swapout"] += 1
        self.restored.append(nid)
        self.unpin_all(held)

    def pin(self, nid, held):  # ref 181-185
        if self.pin_count[nid] == 0:
            self.set[nid].in_use = True
        self.pin_count[nid] += 1
        held.append(nid)

    def unpin_all(self, held):  # ref 187-193
        for nid in held:
            self.pin_count[nid] -= 1
            if self.pin_count[nid] == 0:
                self.set[nid].in_use = False
        held.clear()

    # ---- schedule (ref 458-529) ----
    def do_produce(self, nid):
        node = self.node[nid]
        held = []
        for p in node.parents:
            self.ensure_resident(p)
            self.pin(p, held)
        self.alloc_bytes(node.bytes, nid)
        if nid in self.set:
            raise IllegalTransition(f"node {nid} produced twice")
        self.set[nid] = Rec(node, self.now, self.phase == BACKWARD)
        self.pin(nid, held)
        if self.releases_allowed():
            self.watermark_loop()
        start = self.submit_compute(node.cost)
        end = start + node.cost
        self.now = max(self.now, end)
        self.log(K_COMPUTE, start, node.cost, nid, node.bytes, COMPUTE_S)
        for p in node.parents:
            transition(self.set[p], "Use", end)
        transition(self.set[nid], "Use", end)
        self.unpin_all(held)

    def do_use(self, nid):
        self.ensure_resident(nid)
        transition(self.set[nid], "Use", self.now)
        self.log(K_USE, self.now, 0, nid, self.set[nid].bytes, COMPUTE_S)

    def reclaim(self, nid, k):  # ref 491-517
        r = self.set.get(nid)
        if r is None or r.dead:
            return
        if self.node[nid].uncomputable and not r.cpu_copy_valid and self.ext[nid] > k:
            return
        if r.copy_in_flight:
            self.dead_pending[nid] = True
            return
        if r.on_gpu:
            self.free(r.bytes)
            transition(r, "FreeDead", self.now)
            self.log(K_FREE, self.now, 0, nid, r.bytes, COMPUTE_S)
        else:
            if r.swapout and nid in self.queue:
                self.queue.remove(nid)
            transition(r, "FreeDead", self.now)

    def sweep_dead(self, k):  # ref 519-529
        for nid in self.death[k]:
            self.reclaim(nid, k)
        for nid in self.restored:
            if 0 <= self.last[nid] <= k:
                self.reclaim(nid, k)
        self.restored = []

    def prefetch_burst(self):  # ref 533-585
        if not self.cfg.prefetch_enabled:
            return
        self.drain(self.now)
        count, opened = 0, False
        while self.queue:
            head = self.queue[0]
            r = self.set[head]
            fits = self.used + r.bytes <= self.cfg.watermark_bytes()
            if not fits or (not self.cfg.paper_or and count >= self.cfg.prefetch_limit):
                break
            if not opened:
                opened = True
                self.burst += 1
            assert self.try_alloc(r.bytes)
            d = transfer_time_us(r.bytes, self.cfg)
            transition(r, "ReloadStart", self.now)
            self.queue.pop(0)
            self.counts["reload"] += 1
            self.counts["prefetch_reload"] += 1
            self.copy_busy += d
            if self.cfg.overlap_enabled:
                start = self.submit_copy(d)
                self.log(K_RELOAD, start, d, head, r.bytes, COPY_S, True, self.burst)
                heapq.heappush(self.pending, (start + d, self.seq, False, head, r.bytes))
                self.seq += 1
                self.inflight_done[head] = start + d
            else:
                start = self.submit_compute(d)
                self.log(K_RELOAD, start, d, head, r.bytes, COMPUTE_S, True, self.burst)
                self.now = max(self.now, start + d)
                self.copy_stall += d
                transition(r, "ReloadDone", start + d)
                self.restored.append(head)
            count += 1

    def run(self) -> Result:  # ref 84-121
        infeasible = None
        try:
            for k, (nid, ph, kind) in enumerate(self.t.schedule):
                if self.phase == FORWARD and ph == BACKWARD:
                    self.phase = BACKWARD
                    self.prefetch_burst()
                before = self.compute_submits
                if kind == PRODUCE:
                    self.do_produce(nid)
                else:
                    self.do_use(nid)
                self.sweep_dead(k)
                if self.phase == BACKWARD and self.compute_submits > before:
                    self.prefetch_burst()
        except Infeasible as e:
            infeasible = (e.node, e.deficit)
        self.drain(float("inf"))
        return Result(self.events, self.decisions, infeasible, self.high,
                      max(self.compute_busy, self.copy_busy_until), self.total_stall,
                      self.copy_busy, self.copy_stall, self.counts)


def run_iteration(t: OTrace, cfg: OConfig) -> Result:
    return Engine(t, cfg).run()


def run_unconstrained_baseline(t: OTrace, cfg: OConfig) -> Result:
    """ref src/engine.cpp:635-644."""
    total = sum(n.bytes for n in t.nodes)
    import dataclasses
    c = dataclasses.replace(cfg, policy=BASELINE, budget=total or 1, scripted=[])
    return run_iteration(t, c)


def chrome_trace(events) -> str:
    """timeline_to_chrome_trace — ref src/metrics.cpp:218-280."""
    order = sorted(range(len(events)), key=lambda i: (events[i][0], events[i][1]))
    parts = []
    for i in order:
        ts, stream, kind, node, dur, b, phase, pf, burst = events[i]
        name = KIND_NAMES[kind] + "/" + ("F" if phase == FORWARD else "B")
        if pf:
            name += f"#pf{burst}"
        parts.append(f'{{"name":"{name}","ph":"X","ts":{ts},"dur":{dur},"pid":0,'
                     f'"tid":{0 if stream == COMPUTE_S else 1},"args":{{"node":{node},"bytes":{b}}}}}')
    return "[" + ",".join(parts) + "]"


def report(run: Result, base: Result) -> dict:
    """summarize — ref src/metrics.cpp:27-136 (Report-peak from timeline deltas)."""
    def scan(events):
        deltas, wall, stall, busy, cstall = [], 0, 0, 0, 0
        counts = dict(evict=0, offload=0, reload=0, recompute=0, prefetch_reload=0)
        for ts, stream, kind, node, dur, b, phase, pf, burst in events:
            wall = max(wall, ts + dur)
            if kind == K_COMPUTE:
                deltas.append((ts, b))
            elif kind == K_RECOMPUTE:
                counts["recompute"] += 1
                deltas.append((ts, b))
            elif kind == K_RELOAD:
                counts["reload"] += 1
                counts["prefetch_reload"] += pf
                busy += dur
                cstall += dur if stream == COMPUTE_S else 0
                deltas.append((ts, b))
            elif kind == K_OFFLOAD:
                counts["offload"] += 1
                busy += dur
                cstall += dur if stream == COMPUTE_S else 0
                deltas.append((ts + dur, -b))
            elif kind in (K_EVICT, K_FREE):
                counts["evict"] += kind == K_EVICT
                deltas.append((ts, -b))
            elif kind == K_STALL:
                stall += dur
                cstall += dur
        deltas.sort()
        used = peak = 0
        for _, d in deltas:
            used += d
            peak = max(peak, used)
        return peak, wall, stall, busy, cstall, counts
    p, w, st, busy, cst, c = scan(run.events)
    bp, bw, *_ = scan(base.events)
    ratio = 1.0 if busy == 0 else 1.0 - cst / busy
    return dict(peak_bytes=p, baseline_peak_bytes=bp,
                saving_fraction=0.0 if bp == 0 else 1.0 - p / bp, wall_time_us=w,
                baseline_wall_time_us=bw, overhead_fraction=0.0 if bw == 0 else w / bw - 1.0,
                counts=c, total_stall_us=st, overlap_ratio=min(1.0, max(0.0, ratio)),
                infeasible=run.infeasible is not None)
