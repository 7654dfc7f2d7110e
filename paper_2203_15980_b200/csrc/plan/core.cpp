// libdelta planner core: trace validation, the per-tensor state machine, the
// byte-counted pool / logical streams, and the Filter/Director free
// functions.  Semantics follow the reference line by line where they decide
// anything (cited per function); data structures are our own.
#include <algorithm>
#include <limits>
#include <sstream>
#include <unordered_map>
#include <unordered_set>

#include "deltasim/deltasim.hpp"

namespace deltasim {

std::string u128_to_string(U128 v) {
  char buf[48];
  int pos = 47;
  buf[pos] = '\0';
  do {
    buf[--pos] = static_cast<char>('0' + static_cast<unsigned>(v % 10));
    v /= 10;
  } while (v != 0);
  return std::string(buf + pos);
}

// ---------------------------------------------------------------------------
// Trace lookups and validation (ref src/trace.cpp:26-155)

std::optional<std::size_t> Trace::index_of(NodeId id) const {
  for (std::size_t i = 0; i < nodes.size(); ++i)
    if (nodes[i].id == id) return i;
  return std::nullopt;
}

const OpNode* Trace::find(NodeId id) const {
  auto i = index_of(id);
  return i ? &nodes[*i] : nullptr;
}

const char* to_string(TraceViolationCode c) {
  static const char* const names[] = {
      "DuplicateNodeId",   "CycleOrForwardRef",    "UncomputableHasParents",
      "UncomputableNotEvictPinned", "BothPinned",  "DanglingNodeRef",
      "UseBeforeProduce",  "DuplicateProduce",     "ParentNotProduced",
      "ForwardAfterBackward", "ZeroOutputBytes"};
  auto k = static_cast<std::size_t>(c);
  return k < sizeof(names) / sizeof(names[0]) ? names[k] : "?";
}

// One pass over nodes, one over the schedule; O(N + E) with a hash index
// (the reference's Trace::find inside the schedule loop is O(E*N)).  Error
// order, codes and messages match ref src/trace.cpp:58-148.
std::vector<TraceViolation> validate_trace(const Trace& t) {
  std::vector<TraceViolation> out;
  auto at_node = [&](TraceViolationCode code, NodeId id, std::string msg,
                     Severity sev = Severity::Error) {
    out.push_back({code, sev, id, std::nullopt, std::move(msg)});
  };
  auto at_event = [&](TraceViolationCode code, std::size_t k, std::string msg) {
    out.push_back({code, Severity::Error, std::nullopt, k, std::move(msg)});
  };
  const std::string N = "node ";

  std::unordered_map<NodeId, std::size_t> first;  // id -> first position
  first.reserve(t.nodes.size() * 2);
  for (std::size_t i = 0; i < t.nodes.size(); ++i) {
    const OpNode& n = t.nodes[i];
    if (!first.emplace(n.id, i).second) {
      at_node(TraceViolationCode::DuplicateNodeId, n.id,
              N + std::to_string(n.id) + " declared more than once");
      continue;
    }
    for (NodeId p : n.parents) {
      if (p == n.id || !first.count(p)) {
        at_node(TraceViolationCode::CycleOrForwardRef, n.id,
                N + std::to_string(n.id) + " parent " + std::to_string(p) +
                    " is not a previously declared node");
      }
    }
    if (n.uncomputable && !n.parents.empty())
      at_node(TraceViolationCode::UncomputableHasParents, n.id,
              "uncomputable node " + std::to_string(n.id) + " has parents");
    if (n.uncomputable && !n.evict_pinned)
      at_node(TraceViolationCode::UncomputableNotEvictPinned, n.id,
              "uncomputable node " + std::to_string(n.id) +
                  " must be evict_pinned");
    if (n.evict_pinned && n.offload_pinned)
      at_node(TraceViolationCode::BothPinned, n.id,
              N + std::to_string(n.id) +
                  " is both evict_pinned and offload_pinned; it can never be "
                  "released",
              Severity::Warning);
    if (n.output_bytes == 0)
      at_node(TraceViolationCode::ZeroOutputBytes, n.id,
              N + std::to_string(n.id) + " has zero output_bytes");
  }

  std::unordered_set<NodeId> produced;
  produced.reserve(t.nodes.size() * 2);
  bool backward_seen = false;
  const std::string E = "event ";
  for (std::size_t k = 0; k < t.schedule.size(); ++k) {
    const AccessEvent& ev = t.schedule[k];
    auto it = first.find(ev.node);
    if (it == first.end()) {
      at_event(TraceViolationCode::DanglingNodeRef, k,
               E + std::to_string(k) + " references undeclared node " +
                   std::to_string(ev.node));
      continue;
    }
    if (ev.phase == Phase::Backward) {
      backward_seen = true;
    } else if (backward_seen) {
      at_event(TraceViolationCode::ForwardAfterBackward, k,
               E + std::to_string(k) + " is Forward but follows a Backward event");
    }
    if (ev.kind == AccessKind::Produce) {
      if (!produced.insert(ev.node).second)
        at_event(TraceViolationCode::DuplicateProduce, k,
                 E + std::to_string(k) + " produces node " +
                     std::to_string(ev.node) + " a second time");
      for (NodeId p : t.nodes[it->second].parents) {
        if (!produced.count(p))
          at_event(TraceViolationCode::ParentNotProduced, k,
                   E + std::to_string(k) + " produces node " +
                       std::to_string(ev.node) + " before its parent " +
                       std::to_string(p));
      }
    } else if (!produced.count(ev.node)) {
      at_event(TraceViolationCode::UseBeforeProduce, k,
               E + std::to_string(k) + " uses node " + std::to_string(ev.node) +
                   " before it is produced");
    }
  }
  return out;
}

bool trace_is_valid(const Trace& t) {
  for (const TraceViolation& v : validate_trace(t))
    if (v.severity == Severity::Error) return false;
  return true;
}

// ---------------------------------------------------------------------------
// Tensor state machine (ref src/state.cpp:23-141)

const char* to_string(TensorEvent e) {
  static const char* const names[] = {
      "Produce",     "Use",         "EvictStart",    "OffloadStart",
      "OffloadDone", "ReloadStart", "ReloadDone",    "RecomputeDone",
      "FreeAfterOffload", "FreeDead"};
  auto k = static_cast<std::size_t>(e);
  return k < 10 ? names[k] : "?";
}

bool TensorRecord::location_invariant_holds() const {
  if (dead) return !on_gpu && !in_use && !copy_in_flight;
  if (int(on_gpu) + int(evicted) + int(swapout) != 1) return false;
  if (swapout && !cpu_copy_valid) return false;
  if (evicted && (cpu_copy_valid || uncomputable)) return false;
  if (in_use && !on_gpu) return false;
  return true;
}

MicroDur staleness(const TensorRecord& r, MicroTime now) {
  if (!r.on_gpu)
    throw StateError("staleness: node " + std::to_string(r.node_id) +
                     " is not resident");
  return now > r.last_access ? now - r.last_access : 1;
}

namespace {
[[noreturn]] void reject(const TensorRecord& r, TensorEvent ev) {
  std::ostringstream os;
  os << "illegal transition " << to_string(ev) << " on node " << r.node_id
     << " [on_gpu=" << r.on_gpu << " evicted=" << r.evicted
     << " swapout=" << r.swapout << " uncomputable=" << r.uncomputable
     << " in_use=" << r.in_use << " copy_in_flight=" << r.copy_in_flight
     << " cpu_copy_valid=" << r.cpu_copy_valid << " dead=" << r.dead << "]";
  throw IllegalTransition(os.str());
}
}  // namespace

TensorRecord transition(const TensorRecord& r, TensorEvent ev, MicroTime now) {
  TensorRecord s = r;
  bool ok = true;
  switch (ev) {
    case TensorEvent::Produce:
      ok = !(r.on_gpu || r.evicted || r.swapout || r.dead);
      s.on_gpu = true;
      s.last_access = now;
      break;
    case TensorEvent::Use:
      ok = r.on_gpu && !r.dead;
      s.last_access = now;
      break;
    case TensorEvent::EvictStart:
      ok = r.on_gpu && !r.evict_pinned && !r.in_use && !r.uncomputable &&
           !r.copy_in_flight && !r.dead;
      s.on_gpu = false;
      s.evicted = true;
      s.cpu_copy_valid = false;
      break;
    case TensorEvent::OffloadStart:
      ok = r.on_gpu && !r.offload_pinned && !r.in_use && !r.copy_in_flight &&
           !r.dead;
      s.copy_in_flight = true;
      break;
    case TensorEvent::OffloadDone:
      ok = r.on_gpu && r.copy_in_flight;
      s.copy_in_flight = false;
      s.cpu_copy_valid = true;
      break;
    case TensorEvent::FreeAfterOffload:
      ok = r.on_gpu && r.cpu_copy_valid && !r.copy_in_flight && !r.in_use;
      s.on_gpu = false;
      s.swapout = true;
      break;
    case TensorEvent::ReloadStart:  // may revive a dead tensor with a copy
      ok = (r.swapout || r.dead) && r.cpu_copy_valid && !r.copy_in_flight;
      s.copy_in_flight = true;
      break;
    case TensorEvent::ReloadDone:
      ok = (r.swapout || r.dead) && r.copy_in_flight;
      s.on_gpu = true;
      s.swapout = false;
      s.copy_in_flight = false;
      s.dead = false;
      s.last_access = now;
      break;
    case TensorEvent::RecomputeDone:
      ok = !(r.on_gpu || r.in_use || r.copy_in_flight || r.uncomputable) &&
           (r.evicted || r.swapout || r.dead);
      s.on_gpu = true;
      s.evicted = false;
      s.swapout = false;
      s.cpu_copy_valid = false;
      s.dead = false;
      s.last_access = now;
      break;
    case TensorEvent::FreeDead:
      ok = !(r.in_use || r.copy_in_flight || r.dead);
      s.on_gpu = false;
      s.evicted = false;
      s.swapout = false;
      s.dead = true;
      s.died_swapout = r.swapout;
      break;
  }
  if (!ok) reject(r, ev);
  return s;
}

TensorRecord& ResidentSet::produce(const OpNode& node, MicroTime now,
                                   Phase phase) {
  auto [it, fresh] = records_.try_emplace(node.id);
  if (!fresh)
    throw IllegalTransition("node " + std::to_string(node.id) +
                            " produced twice");
  TensorRecord& r = it->second;
  r.node_id = node.id;
  r.bytes = node.output_bytes;
  r.own_cost = node.compute_cost_us;
  r.uncomputable = node.uncomputable;
  r.evict_pinned = node.evict_pinned;
  r.offload_pinned = node.offload_pinned;
  r.produced_backward = phase == Phase::Backward;
  r = transition(r, TensorEvent::Produce, now);
  resident_bytes_ += r.bytes;
  return r;
}

TensorRecord& ResidentSet::apply(NodeId id, TensorEvent ev, MicroTime now) {
  auto it = records_.find(id);
  if (it == records_.end())
    throw IllegalTransition("node " + std::to_string(id) +
                            " has no record for event " + to_string(ev));
  TensorRecord& r = it->second;
  bool before = r.on_gpu;
  r = transition(r, ev, now);
  if (before != r.on_gpu) {
    if (r.on_gpu)
      resident_bytes_ += r.bytes;
    else
      resident_bytes_ -= r.bytes;
  }
  return r;
}

bool ResidentSet::contains(NodeId id) const { return records_.count(id) != 0; }

const TensorRecord& ResidentSet::at(NodeId id) const {
  auto it = records_.find(id);
  if (it == records_.end())
    throw StateError("node " + std::to_string(id) + " was never produced");
  return it->second;
}

TensorRecord& ResidentSet::at(NodeId id) {
  return const_cast<TensorRecord&>(std::as_const(*this).at(id));
}

Bytes ResidentSet::recount_resident_bytes() const {
  Bytes sum = 0;
  for (const auto& kv : records_)
    if (kv.second.on_gpu) sum += kv.second.bytes;
  return sum;
}

void ResidentSet::check_resident_bytes() const {
  Bytes again = recount_resident_bytes();
  if (again != resident_bytes_)
    throw InternalError("resident_bytes drift: cached " +
                        std::to_string(resident_bytes_) + " vs recount " +
                        std::to_string(again));
}

void ResidentSet::append_sorted(const TensorRecord& r) {
  records_.emplace_hint(records_.end(), r.node_id, r);
  if (r.on_gpu) resident_bytes_ += r.bytes;
}

// ---------------------------------------------------------------------------
// Logical device (ref src/device.cpp:5-43)

AllocResult MemoryPool::try_alloc(Bytes n) {
  Bytes room = budget_ - used_;
  if (n > room) return Insufficient{n - room};
  used_ += n;
  high_watermark_ = std::max(high_watermark_, used_);
  return Allocated{};
}

void MemoryPool::free(Bytes n) {
  if (n > used_)
    throw InternalError("pool free of " + std::to_string(n) +
                        " bytes exceeds used " + std::to_string(used_));
  used_ -= n;
}

std::pair<MicroTime, MicroTime> Stream::submit(MicroTime now,
                                               MicroDur duration,
                                               std::string label, NodeId node) {
  MicroTime start = std::max(now, busy_until_);
  busy_until_ = start + duration;
  busy_total_ += duration;
  log_.push_back({start, busy_until_, std::move(label), node});
  return {start, busy_until_};
}

MicroDur Clock::wait_for(MicroTime t) {
  if (t <= now_) return 0;
  MicroDur waited = t - now_;
  now_ = t;
  return waited;
}

void Clock::advance_to(MicroTime t) { now_ = std::max(now_, t); }

// ---------------------------------------------------------------------------
// Filter / Director / cost model (ref src/policy.cpp:9-158)

const char* to_string(Heuristic h) {
  switch (h) {
    case Heuristic::Base: return "base";
    case Heuristic::Lru: return "lru";
    case Heuristic::Greedy: return "greedy";
  }
  return "?";
}

const char* to_string(ReleaseAction a) {
  return a == ReleaseAction::Evict ? "Evict"
         : a == ReleaseAction::Offload ? "Offload" : "?";
}

U128 CostModel::eff_num() const {
  return U128(bandwidth_bytes_per_us.num) * effective_fraction.num;
}
U128 CostModel::eff_den() const {
  return U128(bandwidth_bytes_per_us.den) * effective_fraction.den;
}

HeuristicScore score(Heuristic h, const TensorRecord& r, MicroTime now) {
  if (!r.on_gpu)
    throw StateError("score: node " + std::to_string(r.node_id) +
                     " is not resident");
  U128 m = r.bytes, s = staleness(r, now);
  switch (h) {
    case Heuristic::Base: return {m * s};
    case Heuristic::Lru: return {s};
    case Heuristic::Greedy: return {m};
  }
  return {1};
}

// ceil(m * eff_den / eff_num): one-way copy time (ref policy.cpp:58-64).
MicroDur transfer_time_us(Bytes m, const CostModel& cm) {
  U128 d = cm.eff_num();
  U128 us = (U128(m) * cm.eff_den() + d - 1) / d;
  if (us > std::numeric_limits<MicroDur>::max())
    throw ArgumentError("swap cost overflows 64-bit microseconds");
  return static_cast<MicroDur>(us);
}

MicroDur swap_cost_bytes(Bytes m, const CostModel& cm) {
  MicroDur one = transfer_time_us(m, cm);
  return cm.swap_cost_mode == SwapCostMode::RoundTrip ? 2 * one : one;
}

MicroDur swap_cost(const TensorRecord& r, const CostModel& cm) {
  return swap_cost_bytes(r.bytes, cm);
}

// Own cost plus the evicted/dead computable ancestor closure; same LIFO walk
// as ref policy.cpp:75-109 so the same lost node is reported first.
MicroDur recompute_cost(NodeId id, const ResidentSet& set, const Trace& trace) {
  const OpNode* target = trace.find(id);
  if (!target)
    throw StateError("recompute_cost: node " + std::to_string(id) +
                     " not in trace");
  if (target->uncomputable)
    throw StateError("recompute_cost: node " + std::to_string(id) +
                     " is uncomputable");
  MicroDur total = target->compute_cost_us;
  std::unordered_set<NodeId> seen;
  std::vector<NodeId> todo(target->parents.begin(), target->parents.end());
  while (!todo.empty()) {
    NodeId p = todo.back();
    todo.pop_back();
    if (seen.count(p)) continue;
    const TensorRecord& r = set.at(p);
    if (r.on_gpu || r.swapout) continue;
    const OpNode* node = trace.find(p);
    if (node->uncomputable) {
      if (r.cpu_copy_valid) continue;
      throw UnrecoverableError("recompute closure of node " +
                               std::to_string(id) +
                               " reaches lost uncomputable node " +
                               std::to_string(p));
    }
    seen.insert(p);
    total += node->compute_cost_us;
    todo.insert(todo.end(), node->parents.begin(), node->parents.end());
  }
  return total;
}

bool releasable(const TensorRecord& r) {
  return r.on_gpu && !r.in_use && !r.copy_in_flight && !r.dead &&
         !r.produced_backward && !(r.evict_pinned && r.offload_pinned);
}

std::optional<NodeId> select_victim(const ResidentSet& set, Heuristic h,
                                    MicroTime now) {
  return select_victim(set, h, now, nullptr);
}

std::optional<NodeId> select_victim(const ResidentSet& set, Heuristic h,
                                    MicroTime now,
                                    bool (*extra_filter)(const TensorRecord&)) {
  std::optional<NodeId> best;
  U128 best_inv = 0;
  for (const auto& [id, r] : set) {
    if (!releasable(r) || (extra_filter && !extra_filter(r))) continue;
    U128 inv = score(h, r, now).inv;
    if (!best || inv > best_inv) {  // strictly better; ties keep lowest id
      best = id;
      best_inv = inv;
    }
  }
  return best;
}

Decision decide(NodeId id, const ResidentSet& set, const Trace& trace,
                const CostModel& cm, MicroTime /*now: staleness cancels*/) {
  const TensorRecord& r = set.at(id);
  if (!releasable(r))
    throw StateError("decide: node " + std::to_string(id) +
                     " is not releasable");
  if (r.evict_pinned) return {ReleaseAction::Offload, std::nullopt};
  if (r.offload_pinned) return {ReleaseAction::Evict, std::nullopt};
  DecisionScore f;
  f.num = U128(recompute_cost(id, set, trace)) * cm.eff_num();
  f.den = U128(r.bytes) * cm.eff_den();
  if (cm.swap_cost_mode == SwapCostMode::RoundTrip) f.den *= 2;
  return {f.leq_one() ? ReleaseAction::Evict : ReleaseAction::Offload, f};
}

}  // namespace deltasim
