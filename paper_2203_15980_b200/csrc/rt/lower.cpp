// Plan -> B200 action program.
//
// The planner (csrc/plan/engine.cpp) decides WHAT happens on the logical
// clock; this pass decides WHERE and WITH WHICH ORDERING it happens on the
// device:
//   1. replay the planner's exact MemoryPool alloc/free sequence
//      (run_iteration_pool_log) to get every allocation's lifetime in
//      pool-op order; the live set at any point is exactly the planner's;
//   2. assign arena offsets offline (greedy by size over known lifetimes:
//      the footprint lands at or just above the pool high-watermark, and the
//      difference is reported as fragmentation, never hidden);
//   3. lower timeline events to actions on the compute stream and the copy
//      stream(s) and insert the minimal cross-stream event edges:
//      read-after-write on a tensor, write-after-read/write on a reused arena
//      range, host-slab RAW between offload and reload, a copy never starting
//      before the compute-stream point the plan issued it at, and a restore
//      of a tensor never starting before its offload landed (the planner
//      waits for that landing, src/engine.cpp:375-380).  With those edges the
//      executed timeline keeps the plan's causal order, so the reference's
//      replay_check can certify it with measured timestamps.
//      Copies: ONE copy stream in plan order (the reference's single copy
//      stream) unless DELTA_LOWER_DUPLEX_COPIES puts reloads on a second one.
// Everything here runs once per plan; the step itself replays the program
// (captured as a CUDA graph by the host runtime).
#include "lower.hpp"

#include <algorithm>
#include <limits>
#include <unordered_map>

namespace delta_rt {

using namespace deltasim;

namespace {

constexpr std::uint64_t kNever = std::numeric_limits<std::uint64_t>::max();

struct Alloc {
  NodeId node;
  std::uint64_t bytes;     // rounded to the arena alignment
  std::uint64_t born;      // pool-op index of the alloc
  std::uint64_t died = kNever;
  std::uint64_t offset = 0;
  // accesses, as (stream, position-in-stream) of the actions touching it
  std::vector<std::pair<std::uint32_t, std::uint64_t>> touches;
};

struct Pending {  // action before event insertion
  delta_action a;
  std::vector<std::pair<std::uint32_t, std::uint64_t>> deps;  // (stream, pos)
};

}  // namespace

Program lower_plan(const Trace& trace, const EngineConfig& cfg,
                   std::uint64_t align, std::uint32_t flags) {
  const std::uint32_t reload_stream =
      (flags & DELTA_LOWER_DUPLEX_COPIES) ? DELTA_STREAM_H2D : DELTA_STREAM_D2H;
  if (align == 0 || (align & (align - 1))) throw ArgumentError("lower: align must be a power of two");
  Program prog;
  std::vector<PoolOp> ops;
  prog.plan = run_iteration_pool_log(trace, cfg, &ops);

  std::unordered_map<NodeId, std::size_t> pos;
  for (std::size_t i = 0; i < trace.nodes.size(); ++i) pos[trace.nodes[i].id] = i;

  // ---- 1. lifetimes in pool-op order ----
  std::vector<Alloc> allocs;
  std::unordered_map<NodeId, std::size_t> live;  // node -> alloc index
  std::vector<std::size_t> alloc_of_op(ops.size(), SIZE_MAX);
  for (std::size_t k = 0; k < ops.size(); ++k) {
    const PoolOp& op = ops[k];
    if (op.alloc) {
      if (live.count(op.node)) throw InternalError("lower: double alloc of node " + std::to_string(op.node));
      std::uint64_t b = (op.bytes + align - 1) & ~(align - 1);
      live[op.node] = allocs.size();
      alloc_of_op[k] = allocs.size();
      allocs.push_back(Alloc{op.node, b, k, kNever, 0, {}});
    } else {
      auto it = live.find(op.node);
      if (it == live.end()) throw InternalError("lower: free of non-live node " + std::to_string(op.node));
      allocs[it->second].died = k;
      alloc_of_op[k] = it->second;
      live.erase(it);
    }
  }

  // ---- 2. offsets: offline packing of known lifetimes ----
  // Several greedy orders (largest first; longest-lived first; size x
  // lifetime; allocation order), each placing an allocation at the lowest
  // offset clear of every already-placed overlapping lifetime; the smallest
  // footprint wins (ties: the earlier order).  The footprint can only exceed
  // the pool peak through fragmentation, which is reported, never hidden.
  {
    const std::size_t n = allocs.size();
    auto life = [&](const Alloc& a) {
      return (a.died == kNever ? std::uint64_t(ops.size()) : a.died) - a.born;
    };
    // best_fit: the smallest gap that holds the allocation (else the top)
    auto pack = [&](const std::vector<std::size_t>& order, std::vector<std::uint64_t>& off,
                    bool best_fit) {
      off.assign(n, 0);
      std::vector<std::size_t> placed;
      placed.reserve(n);
      std::vector<std::pair<std::uint64_t, std::uint64_t>> busy;
      std::uint64_t footprint = 0;
      for (std::size_t idx : order) {
        const Alloc& a = allocs[idx];
        busy.clear();
        for (std::size_t j : placed) {
          const Alloc& b = allocs[j];
          if (a.born < b.died && b.born < a.died) busy.push_back({off[j], off[j] + b.bytes});
        }
        std::sort(busy.begin(), busy.end());
        std::uint64_t o = 0, pick = kNever, pick_gap = kNever;
        for (auto& r : busy) {
          if (r.first >= o + a.bytes) {  // a gap [o, r.first) that fits
            if (!best_fit) break;
            if (r.first - o < pick_gap) {
              pick_gap = r.first - o;
              pick = o;
            }
          }
          o = std::max(o, r.second);
        }
        if (!best_fit || pick == kNever) pick = o;
        off[idx] = pick;
        footprint = std::max(footprint, pick + a.bytes);
        placed.push_back(idx);
      }
      return footprint;
    };
    std::vector<std::size_t> base(n);
    for (std::size_t i = 0; i < n; ++i) base[i] = i;
    std::vector<std::vector<std::size_t>> orders;
    auto by = [&](auto key) {
      std::vector<std::size_t> o = base;
      std::stable_sort(o.begin(), o.end(), [&](std::size_t x, std::size_t y) {
        const auto kx = key(allocs[x]), ky = key(allocs[y]);
        if (kx != ky) return kx > ky;
        return allocs[x].born < allocs[y].born;
      });
      orders.push_back(std::move(o));
    };
    by([](const Alloc& a) { return a.bytes; });
    by([&](const Alloc& a) { return life(a); });
    by([&](const Alloc& a) { return static_cast<unsigned __int128>(a.bytes) * life(a); });
    orders.push_back(base);  // allocation order
    // a few deterministic perturbations of the size order (fixed seed: the
    // packing is a pure function of the plan)
    std::uint64_t rng = 0x9E3779B97F4A7C15ull;
    for (int rep = 0; rep < 24; ++rep) {
      std::vector<std::size_t> o = orders[0];
      for (std::size_t i = 0; i + 1 < o.size(); ++i) {
        rng ^= rng << 13;
        rng ^= rng >> 7;
        rng ^= rng << 17;
        if ((rng & 3) == 0) std::swap(o[i], o[i + 1]);
      }
      orders.push_back(std::move(o));
    }
    std::uint64_t best = kNever;
    std::vector<std::uint64_t> off, best_off;
    for (const auto& o : orders) {
      for (int bf = 0; bf < 2; ++bf) {
        const std::uint64_t f = pack(o, off, bf == 1);
        if (f < best) {
          best = f;
          best_off = off;
        }
      }
      if (best <= prog.plan.peak_bytes) break;  // cannot do better than the pool peak
    }
    for (std::size_t i = 0; i < n; ++i) allocs[i].offset = n ? best_off[i] : 0;
    prog.arena_bytes = n ? best : 0;
  }

  // ---- 3. actions with dependencies ----
  std::vector<Pending> pend;
  std::uint64_t stream_len[3] = {0, 0, 0};
  std::unordered_map<NodeId, std::size_t> cur;         // node -> alloc holding its data
  std::unordered_map<NodeId, std::pair<std::uint32_t, std::uint64_t>> writer;  // alloc data writer
  std::unordered_map<NodeId, std::uint64_t> host_slot;
  std::unordered_map<NodeId, std::pair<std::uint32_t, std::uint64_t>> host_writer;
  std::uint64_t host_bytes = 0;
  // the latest compute-stream action: the plan's issue point of a copy
  bool have_compute = false;
  std::pair<std::uint32_t, std::uint64_t> last_compute{0, 0};

  // region hazards for a new allocation: every earlier, already-dead
  // allocation overlapping it contributes its touches.
  auto reuse_deps = [&](std::size_t ai, std::vector<std::pair<std::uint32_t, std::uint64_t>>& deps) {
    const Alloc& a = allocs[ai];
    for (std::size_t j = 0; j < allocs.size(); ++j) {
      const Alloc& b = allocs[j];
      if (b.died == kNever || b.died > a.born) continue;
      if (b.offset < a.offset + a.bytes && a.offset < b.offset + b.bytes)
        deps.insert(deps.end(), b.touches.begin(), b.touches.end());
    }
  };
  auto emit = [&](delta_action act, std::vector<std::pair<std::uint32_t, std::uint64_t>> deps) {
    act.event = 0;
    std::uint32_t s = act.stream;
    std::uint64_t p = stream_len[s]++;
    pend.push_back({act, std::move(deps)});
    return std::make_pair(s, p);
  };

  std::size_t next_op = 0;
  const auto& events = prog.plan.timeline.events;
  auto apply_ops_until = [&](std::uint64_t before_event) {
    while (next_op < ops.size() && ops[next_op].before_event <= before_event) {
      const PoolOp& op = ops[next_op];
      if (op.alloc) cur[op.node] = alloc_of_op[next_op];
      ++next_op;
    }
  };

  for (std::uint64_t e = 0; e < events.size(); ++e) {
    apply_ops_until(e);
    const TimelineEvent& ev = events[e];
    delta_action act{};
    act.node = ev.node;
    act.plan_event = e;
    switch (ev.kind) {
      case EventKind::Compute:
      case EventKind::Recompute: {
        std::size_t ai = cur.at(ev.node);
        Alloc& a = allocs[ai];
        act.op = ev.kind == EventKind::Compute ? DELTA_ACT_COMPUTE : DELTA_ACT_RECOMPUTE;
        act.stream = DELTA_STREAM_COMPUTE;
        act.offset = a.offset;
        act.bytes = a.bytes;
        std::vector<std::pair<std::uint32_t, std::uint64_t>> deps;
        reuse_deps(ai, deps);
        const OpNode& n = trace.nodes[pos.at(ev.node)];
        act.n_inputs = static_cast<std::uint32_t>(n.parents.size());
        act.inputs_at = prog.inputs.size();
        std::vector<std::size_t> in_allocs;
        for (NodeId p : n.parents) {
          std::size_t pi = cur.at(p);
          prog.inputs.push_back(allocs[pi].offset);
          in_allocs.push_back(pi);
          deps.push_back(writer.at(p));
        }
        // a restore after an offload starts once that offload has landed
        auto ho = host_writer.find(ev.node);
        if (ho != host_writer.end()) deps.push_back(ho->second);
        auto me = emit(act, std::move(deps));
        have_compute = true;
        last_compute = me;
        a.touches.push_back(me);
        for (std::size_t pi : in_allocs) allocs[pi].touches.push_back(me);
        writer[ev.node] = me;
        break;
      }
      case EventKind::Offload: {
        std::size_t ai = cur.at(ev.node);
        Alloc& a = allocs[ai];
        act.op = DELTA_ACT_OFFLOAD;
        act.stream = DELTA_STREAM_D2H;
        act.offset = a.offset;
        act.bytes = ev.bytes;
        auto hs = host_slot.find(ev.node);
        if (hs == host_slot.end()) {
          hs = host_slot.emplace(ev.node, host_bytes).first;
          host_bytes += (ev.bytes + align - 1) & ~(align - 1);
        }
        act.host_offset = hs->second;
        std::vector<std::pair<std::uint32_t, std::uint64_t>> deps{writer.at(ev.node)};
        auto hw = host_writer.find(ev.node);  // an earlier offload of this node
        if (hw != host_writer.end()) deps.push_back(hw->second);
        if (have_compute) deps.push_back(last_compute);  // issue point
        auto me = emit(act, std::move(deps));
        a.touches.push_back(me);
        host_writer[ev.node] = me;
        break;
      }
      case EventKind::Reload: {
        std::size_t ai = cur.at(ev.node);
        Alloc& a = allocs[ai];
        act.op = DELTA_ACT_RELOAD;
        act.stream = reload_stream;
        act.offset = a.offset;
        act.bytes = ev.bytes;
        act.host_offset = host_slot.at(ev.node);
        std::vector<std::pair<std::uint32_t, std::uint64_t>> deps{host_writer.at(ev.node)};
        reuse_deps(ai, deps);
        if (have_compute) deps.push_back(last_compute);  // issue point
        auto me = emit(act, std::move(deps));
        a.touches.push_back(me);
        writer[ev.node] = me;
        break;
      }
      default:
        break;  // Evict / Free / Use / Stall: bookkeeping only
    }
  }

  // ---- 4. minimal event edges ----
  // pos_in_stream -> global pending index, per stream
  std::vector<std::vector<std::size_t>> by_stream(3);
  for (std::size_t i = 0; i < pend.size(); ++i) by_stream[pend[i].a.stream].push_back(i);
  std::vector<std::int64_t> need_event(pend.size(), -1);
  std::vector<std::vector<std::pair<std::uint32_t, std::uint64_t>>> waits(pend.size());
  {
    std::int64_t waited[3][3];
    for (auto& r : waited) for (auto& v : r) v = -1;
    std::uint64_t seen[3] = {0, 0, 0};
    for (std::size_t i = 0; i < pend.size(); ++i) {
      std::uint32_t s = pend[i].a.stream;
      std::int64_t want[3] = {-1, -1, -1};
      for (auto& d : pend[i].deps)
        if (d.first != s) want[d.first] = std::max<std::int64_t>(want[d.first], std::int64_t(d.second));
      for (std::uint32_t t = 0; t < 3; ++t) {
        if (want[t] < 0 || want[t] <= waited[s][t]) continue;
        if (std::uint64_t(want[t]) >= seen[t]) throw InternalError("lower: dependency on a later action");
        waits[i].push_back({t, std::uint64_t(want[t])});
        waited[s][t] = want[t];
      }
      ++seen[s];
    }
  }
  std::uint32_t n_events = 0;
  for (auto& w : waits)
    for (auto& d : w) {
      std::size_t g = by_stream[d.first][d.second];
      if (need_event[g] < 0) need_event[g] = n_events++;
    }
  for (std::size_t i = 0; i < pend.size(); ++i) {
    for (auto& d : waits[i]) {
      delta_action w{};
      w.op = DELTA_ACT_WAIT;
      w.stream = pend[i].a.stream;
      w.node = pend[i].a.node;
      w.event = static_cast<std::uint32_t>(need_event[by_stream[d.first][d.second]]);
      w.plan_event = pend[i].a.plan_event;
      prog.actions.push_back(w);
    }
    prog.actions.push_back(pend[i].a);
    if (need_event[i] >= 0) {
      delta_action r{};
      r.op = DELTA_ACT_RECORD;
      r.stream = pend[i].a.stream;
      r.node = pend[i].a.node;
      r.event = static_cast<std::uint32_t>(need_event[i]);
      r.plan_event = pend[i].a.plan_event;
      prog.actions.push_back(r);
    }
  }
  prog.n_events = n_events;
  prog.host_bytes = host_bytes;
  prog.pool_peak = prog.plan.peak_bytes;
  return prog;
}

}  // namespace delta_rt
