// libdelta planner: DELTA's training-step executor on the logical integer
// clock.  Decisions, timeline and counters are bit-exact with the reference
// Engine (ref src/engine.cpp:73-623); the data layout is new:
//   * node ids are mapped once to dense indices; every per-tensor field is a
//     flat array (no std::map / unordered_map lookups on the hot loop);
//   * the Filter scans a rank-ordered bitset of resident tensors, so the
//     ascending-id tie-break of the reference's std::map walk is preserved
//     while non-resident tensors cost nothing;
//   * the Director's recompute-closure walk uses an epoch-stamped visited
//     array instead of std::set + Trace::find linear scans.
// The plan it emits is what csrc/rt lowers onto the B200 (HBM arena offsets,
// copy-engine swaps, recompute kernel launches).
#include <algorithm>
#include <limits>
#include <queue>
#include <unordered_map>

#include "deltasim/deltasim.hpp"

namespace deltasim {

const char* to_string(PolicyMode m) {
  switch (m) {
    case PolicyMode::Delta: return "delta";
    case PolicyMode::RecomputeOnly: return "recompute-only";
    case PolicyMode::OffloadOnly: return "offload-only";
    case PolicyMode::Baseline: return "baseline";
  }
  return "?";
}

const char* to_string(EventKind k) {
  static const char* const names[] = {"Compute", "Offload", "Reload",
                                      "Recompute", "Stall", "Evict",
                                      "Use", "Free"};
  auto i = static_cast<std::size_t>(k);
  return i < 8 ? names[i] : "?";
}

Bytes EngineConfig::watermark_bytes() const {
  return static_cast<Bytes>(U128(budget) * watermark_fraction.num /
                            watermark_fraction.den);
}

void OffloadQueue::remove(NodeId id) {
  fifo.erase(std::remove(fifo.begin(), fifo.end(), id), fifo.end());
}

namespace {

using Idx = std::uint32_t;

struct Infeasible {
  InfeasibleInfo info;
};

// Copy landing; (ts, seq) order as ref engine.cpp:53-65.
struct Landing {
  MicroTime ts;
  std::uint64_t seq;
  bool offload;
  Idx node;
  Bytes bytes;
};
struct LandsLater {
  bool operator()(const Landing& a, const Landing& b) const {
    return a.ts != b.ts ? a.ts > b.ts : a.seq > b.seq;
  }
};

class Planner {
 public:
  Planner(const Trace& t, const EngineConfig& c, std::vector<PoolOp>* ops)
      : trace_(t), cfg_(c), pool_(c.budget), mark_(c.watermark_bytes()),
        pool_ops_(ops) {
    build_index();
  }

  RunResult run();

 private:
  // ---- static indexing (ref engine.cpp:126-173) ----
  void build_index();

  // ---- state helpers ----
  TensorRecord& R(Idx i) { return rec_[i]; }
  void set_bit(Idx i, bool on) {
    Idx r = rank_[i];
    if (on)
      resident_bits_[r >> 6] |= (1ULL << (r & 63));
    else
      resident_bits_[r >> 6] &= ~(1ULL << (r & 63));
  }
  void apply(Idx i, TensorEvent ev, MicroTime now) {
    bool before = rec_[i].on_gpu;
    rec_[i] = transition(rec_[i], ev, now);
    if (before != rec_[i].on_gpu) set_bit(i, rec_[i].on_gpu);
  }
  void produce(Idx i, MicroTime now) {
    if (produced_[i])
      throw IllegalTransition("node " + std::to_string(ids_[i]) +
                              " produced twice");
    produced_[i] = 1;
    const OpNode& n = trace_.nodes[i];
    TensorRecord& r = rec_[i];
    r.node_id = n.id;
    r.bytes = n.output_bytes;
    r.own_cost = n.compute_cost_us;
    r.uncomputable = n.uncomputable;
    r.evict_pinned = n.evict_pinned;
    r.offload_pinned = n.offload_pinned;
    r.produced_backward = phase_ == Phase::Backward;
    r = transition(r, TensorEvent::Produce, now);
    set_bit(i, true);
  }
  void pin(Idx i, std::vector<Idx>& held) {
    if (pin_[i]++ == 0) rec_[i].in_use = true;
    held.push_back(i);
  }
  void unpin_all(std::vector<Idx>& held) {
    for (Idx i : held)
      if (--pin_[i] == 0) rec_[i].in_use = false;
    held.clear();
  }

  // ---- logical streams ----
  MicroTime submit_compute(MicroDur d) {
    MicroTime start = std::max(clock_.now(), compute_busy_);
    compute_busy_ = start + d;
    ++compute_submits_;
    return start;
  }
  MicroTime submit_copy(MicroDur d) {
    MicroTime start = std::max(clock_.now(), copy_busy_until_);
    copy_busy_until_ = start + d;
    return start;
  }

  void log(EventKind k, MicroTime ts, MicroDur d, Idx i, Bytes b,
           StreamKind s, bool pf = false, std::uint32_t burst = 0) {
    events_.push_back({ts, s, k, ids_[i], d, b, phase_, pf, burst});
  }

  void drain(MicroTime up_to);
  void stall_until(MicroTime t, Idx cause);

  // ---- release machinery (ref engine.cpp:250-362) ----
  bool releases_allowed() const {
    return phase_ == Phase::Forward && cfg_.policy_mode != PolicyMode::Baseline;
  }
  Bytes committed_used() const { return pool_.used() - inflight_release_; }
  std::optional<Idx> filter(bool (*extra)(const TensorRecord&));
  MicroDur closure_cost(Idx i);
  ReleaseAction director(Idx i);
  bool release_one();
  void watermark_loop() {
    while (committed_used() > mark_)
      if (!release_one()) break;
  }
  void alloc_bytes(Bytes n, Idx for_node);

  // ---- residency (ref engine.cpp:370-454) ----
  enum class Restore { Access, ClosureDep };
  void ensure_resident(Idx i, Restore mode);
  void demand_reload(Idx i);
  void rebuild(Idx i);

  // ---- schedule (ref engine.cpp:458-529) ----
  void do_produce(Idx i);
  void do_use(Idx i);
  void reclaim(Idx i, std::size_t k);
  void sweep_dead(std::size_t k);
  void prefetch_burst();

  void queue_remove(Idx i) {
    auto it = std::find(queue_.begin(), queue_.end(), i);
    if (it != queue_.end()) queue_.erase(it);  // ids are unique in the FIFO
  }

  const Trace& trace_;
  const EngineConfig& cfg_;
  MemoryPool pool_;
  const Bytes mark_;
  std::vector<PoolOp>* pool_ops_;

  void pool_free(Idx i, Bytes b) {
    pool_.free(b);
    if (pool_ops_) pool_ops_->push_back({events_.size(), ids_[i], b, false});
  }
  bool pool_alloc(Idx i, Bytes b) {
    if (std::holds_alternative<Insufficient>(pool_.try_alloc(b))) return false;
    if (pool_ops_) pool_ops_->push_back({events_.size(), ids_[i], b, true});
    return true;
  }

  std::size_t n_ = 0;
  std::vector<NodeId> ids_;
  std::unordered_map<NodeId, Idx> index_;
  std::vector<Idx> parent_off_, parent_idx_;  // CSR parents
  std::vector<Idx> sched_node_;
  std::vector<std::ptrdiff_t> last_access_, extended_last_;
  std::vector<Idx> death_off_, death_idx_;  // CSR death lists per event
  std::vector<Idx> rank_, by_rank_;
  std::vector<std::uint64_t> resident_bits_;

  std::vector<TensorRecord> rec_;
  std::vector<std::uint8_t> produced_, dead_pending_;
  std::vector<std::uint32_t> pin_;
  std::vector<MicroTime> inflight_done_;
  std::vector<std::uint32_t> visit_;  // epoch stamps for closure_cost
  std::uint32_t epoch_ = 0;
  std::vector<Idx> stack_;

  Clock clock_;
  MicroTime compute_busy_ = 0, copy_busy_until_ = 0;
  std::uint64_t compute_submits_ = 0;
  std::deque<Idx> queue_;  // offload FIFO, landing order
  std::priority_queue<Landing, std::vector<Landing>, LandsLater> pending_;
  std::vector<Idx> restored_;
  std::vector<TimelineEvent> events_;
  std::vector<std::pair<NodeId, ReleaseAction>> decisions_;

  Phase phase_ = Phase::Forward;
  Bytes inflight_release_ = 0;
  std::uint64_t seq_ = 0;
  std::uint32_t burst_ = 0;
  std::size_t scripted_pos_ = 0;
  std::optional<InfeasibleInfo> infeasible_;
  ActionCounts counts_;
  MicroDur total_stall_ = 0, copy_busy_ = 0, copy_stall_ = 0;
};

void Planner::build_index() {
  n_ = trace_.nodes.size();
  ids_.resize(n_);
  index_.reserve(n_ * 2);
  for (Idx i = 0; i < n_; ++i) {
    ids_[i] = trace_.nodes[i].id;
    index_[ids_[i]] = i;
  }
  parent_off_.assign(n_ + 1, 0);
  for (Idx i = 0; i < n_; ++i) {
    parent_off_[i + 1] = parent_off_[i] + Idx(trace_.nodes[i].parents.size());
  }
  parent_idx_.resize(parent_off_[n_]);
  for (Idx i = 0; i < n_; ++i) {
    Idx o = parent_off_[i];
    for (NodeId p : trace_.nodes[i].parents) parent_idx_[o++] = index_.at(p);
  }
  const std::size_t E = trace_.schedule.size();
  sched_node_.resize(E);
  last_access_.assign(n_, -1);
  auto touch = [&](Idx i, std::ptrdiff_t k) {
    if (k > last_access_[i]) last_access_[i] = k;
  };
  for (std::size_t k = 0; k < E; ++k) {
    Idx i = index_.at(trace_.schedule[k].node);
    sched_node_[k] = i;
    touch(i, std::ptrdiff_t(k));
    if (trace_.schedule[k].kind == AccessKind::Produce)
      for (Idx o = parent_off_[i]; o < parent_off_[i + 1]; ++o)
        touch(parent_idx_[o], std::ptrdiff_t(k));
  }
  // An uncomputable tensor with no host copy must outlive every descendant
  // access (ref engine.cpp:145-157); parents precede children positionally.
  extended_last_ = last_access_;
  for (std::size_t i = n_; i-- > 0;)
    for (Idx o = parent_off_[i]; o < parent_off_[i + 1]; ++o) {
      Idx p = parent_idx_[o];
      extended_last_[p] = std::max(extended_last_[p], extended_last_[i]);
    }
  // Death lists in CSR form, node-position order within each event.
  std::vector<std::pair<std::size_t, Idx>> deaths;
  deaths.reserve(n_ + 8);
  for (Idx i = 0; i < n_; ++i) {
    if (last_access_[i] >= 0) deaths.push_back({std::size_t(last_access_[i]), i});
    if (trace_.nodes[i].uncomputable && extended_last_[i] > last_access_[i])
      deaths.push_back({std::size_t(extended_last_[i]), i});
  }
  death_off_.assign(E + 1, 0);
  for (auto& d : deaths) ++death_off_[d.first + 1];
  for (std::size_t k = 0; k < E; ++k) death_off_[k + 1] += death_off_[k];
  death_idx_.resize(deaths.size());
  {
    std::vector<Idx> fill(death_off_.begin(), death_off_.end() - 1);
    for (auto& d : deaths) death_idx_[fill[d.first]++] = d.second;  // stable
  }
  by_rank_.resize(n_);
  for (Idx i = 0; i < n_; ++i) by_rank_[i] = i;
  std::stable_sort(by_rank_.begin(), by_rank_.end(),
                   [&](Idx a, Idx b) { return ids_[a] < ids_[b]; });
  rank_.resize(n_);
  for (Idx r = 0; r < n_; ++r) rank_[by_rank_[r]] = r;
  resident_bits_.assign((n_ + 63) / 64, 0);

  rec_.assign(n_, TensorRecord{});
  produced_.assign(n_, 0);
  dead_pending_.assign(n_, 0);
  pin_.assign(n_, 0);
  inflight_done_.assign(n_, 0);
  visit_.assign(n_, 0);
  events_.reserve(E * 2 + 16);
}

void Planner::drain(MicroTime up_to) {
  while (!pending_.empty() && pending_.top().ts <= up_to) {
    Landing c = pending_.top();
    pending_.pop();
    Idx i = c.node;
    if (c.offload) {
      apply(i, TensorEvent::OffloadDone, c.ts);
      apply(i, TensorEvent::FreeAfterOffload, c.ts);
      pool_free(i, c.bytes);
      inflight_release_ -= c.bytes;
      if (dead_pending_[i]) {
        dead_pending_[i] = 0;
        apply(i, TensorEvent::FreeDead, c.ts);
      } else {
        queue_.push_back(i);
      }
    } else {
      apply(i, TensorEvent::ReloadDone, c.ts);
      if (dead_pending_[i]) {
        dead_pending_[i] = 0;
        pool_free(i, c.bytes);
        apply(i, TensorEvent::FreeDead, c.ts);
        log(EventKind::Free, c.ts, 0, i, c.bytes, StreamKind::Compute);
      } else {
        restored_.push_back(i);
      }
    }
  }
}

void Planner::stall_until(MicroTime t, Idx cause) {
  MicroTime before = clock_.now();
  MicroDur waited = clock_.wait_for(t);
  if (waited > 0) {
    log(EventKind::Stall, before, waited, cause, 0, StreamKind::Compute);
    total_stall_ += waited;
    copy_stall_ += waited;
  }
  drain(clock_.now());
}

// Filter (Algorithm 2; ref policy.cpp:121-136 + engine.cpp:67-71): walk the
// resident tensors in ascending id, keep the strictly largest score
// denominator.
std::optional<Idx> Planner::filter(bool (*extra)(const TensorRecord&)) {
  const MicroTime now = clock_.now();
  const Heuristic h = cfg_.heuristic;
  std::optional<Idx> best;
  U128 best_inv = 0;
  for (std::size_t w = 0; w < resident_bits_.size(); ++w) {
    std::uint64_t bits = resident_bits_[w];
    while (bits) {
      Idx r = Idx(w * 64 + __builtin_ctzll(bits));
      bits &= bits - 1;
      Idx i = by_rank_[r];
      const TensorRecord& t = rec_[i];
      if (!releasable(t) || (extra && !extra(t))) continue;
      U128 s = now > t.last_access ? now - t.last_access : 1;
      U128 inv = h == Heuristic::Base   ? U128(t.bytes) * s
                 : h == Heuristic::Lru  ? s
                                        : U128(t.bytes);
      if (!best || inv > best_inv) {
        best = i;
        best_inv = inv;
      }
    }
  }
  return best;
}

// recompute_cost (ref policy.cpp:75-109) on dense indices.  Same LIFO order so
// an unrecoverable closure reports the same lost node.
MicroDur Planner::closure_cost(Idx i) {
  if (trace_.nodes[i].uncomputable)
    throw StateError("recompute_cost: node " + std::to_string(ids_[i]) +
                     " is uncomputable");
  if (++epoch_ == 0) {
    std::fill(visit_.begin(), visit_.end(), 0);
    epoch_ = 1;
  }
  MicroDur total = trace_.nodes[i].compute_cost_us;
  stack_.assign(parent_idx_.begin() + parent_off_[i],
                parent_idx_.begin() + parent_off_[i + 1]);
  while (!stack_.empty()) {
    Idx p = stack_.back();
    stack_.pop_back();
    if (visit_[p] == epoch_) continue;
    if (!produced_[p])
      throw StateError("node " + std::to_string(ids_[p]) + " was never produced");
    const TensorRecord& r = rec_[p];
    if (r.on_gpu || r.swapout) continue;
    if (trace_.nodes[p].uncomputable) {
      if (r.cpu_copy_valid) continue;
      throw UnrecoverableError("recompute closure of node " +
                               std::to_string(ids_[i]) +
                               " reaches lost uncomputable node " +
                               std::to_string(ids_[p]));
    }
    visit_[p] = epoch_;
    total += trace_.nodes[p].compute_cost_us;
    stack_.insert(stack_.end(), parent_idx_.begin() + parent_off_[p],
                  parent_idx_.begin() + parent_off_[p + 1]);
  }
  return total;
}

// Director (Algorithm 3; ref policy.cpp:138-158).
ReleaseAction Planner::director(Idx i) {
  const TensorRecord& r = rec_[i];
  if (!releasable(r))
    throw StateError("decide: node " + std::to_string(ids_[i]) +
                     " is not releasable");
  if (r.evict_pinned) return ReleaseAction::Offload;
  if (r.offload_pinned) return ReleaseAction::Evict;
  const CostModel& cm = cfg_.cost_model;
  U128 num = U128(closure_cost(i)) * cm.eff_num();
  U128 den = U128(r.bytes) * cm.eff_den();
  if (cm.swap_cost_mode == SwapCostMode::RoundTrip) den *= 2;
  return num <= den ? ReleaseAction::Evict : ReleaseAction::Offload;
}

bool only_recomputable(const TensorRecord& r) {
  return !r.evict_pinned && !r.uncomputable;
}
bool only_offloadable(const TensorRecord& r) { return !r.offload_pinned; }

bool Planner::release_one() {
  const MicroTime now = clock_.now();
  Idx v;
  ReleaseAction act;
  if (scripted_pos_ < cfg_.scripted_decisions.size()) {
    auto [id, a] = cfg_.scripted_decisions[scripted_pos_++];
    auto it = index_.find(id);
    if (it == index_.end() || !produced_[it->second] ||
        !releasable(rec_[it->second]))
      throw InternalError("scripted decision targets unreleasable node " +
                          std::to_string(id));
    v = it->second;
    act = a;
  } else {
    std::optional<Idx> pick;
    switch (cfg_.policy_mode) {
      case PolicyMode::Delta: pick = filter(nullptr); break;
      case PolicyMode::RecomputeOnly: pick = filter(only_recomputable); break;
      case PolicyMode::OffloadOnly: pick = filter(only_offloadable); break;
      case PolicyMode::Baseline: return false;
    }
    if (!pick) return false;
    v = *pick;
    act = cfg_.policy_mode == PolicyMode::Delta           ? director(v)
          : cfg_.policy_mode == PolicyMode::RecomputeOnly ? ReleaseAction::Evict
                                                          : ReleaseAction::Offload;
  }
  decisions_.emplace_back(ids_[v], act);
  const Bytes bytes = rec_[v].bytes;
  if (act == ReleaseAction::Evict) {
    apply(v, TensorEvent::EvictStart, now);
    pool_free(v, bytes);
    ++counts_.evict;
    log(EventKind::Evict, now, 0, v, bytes, StreamKind::Compute);
    return true;
  }
  const MicroDur d = transfer_time_us(bytes, cfg_.cost_model);
  apply(v, TensorEvent::OffloadStart, now);
  ++counts_.offload;
  copy_busy_ += d;
  if (cfg_.overlap_enabled) {
    MicroTime start = submit_copy(d);
    log(EventKind::Offload, start, d, v, bytes, StreamKind::Copy);
    pending_.push({start + d, seq_++, true, v, bytes});
    inflight_done_[v] = start + d;
    inflight_release_ += bytes;
  } else {
    MicroTime start = submit_compute(d);
    MicroTime end = start + d;
    log(EventKind::Offload, start, d, v, bytes, StreamKind::Compute);
    clock_.advance_to(end);
    copy_stall_ += d;
    apply(v, TensorEvent::OffloadDone, end);
    apply(v, TensorEvent::FreeAfterOffload, end);
    pool_free(v, bytes);
    queue_.push_back(v);
  }
  return true;
}

void Planner::alloc_bytes(Bytes n, Idx for_node) {
  drain(clock_.now());
  while (pool_.available() < n) {
    bool covered = pool_.budget() - committed_used() >= n;
    if (!covered && releases_allowed() && release_one()) continue;
    if (!pending_.empty()) {
      Landing next = pending_.top();
      stall_until(next.ts, next.node);
      continue;
    }
    throw Infeasible{{ids_[for_node], n - pool_.available()}};
  }
  if (!pool_alloc(for_node, n))
    throw InternalError("allocation failed after space was ensured");
  if (releases_allowed()) watermark_loop();
}

void Planner::ensure_resident(Idx i, Restore mode) {
  drain(clock_.now());
  if (!produced_[i])
    throw StateError("node " + std::to_string(ids_[i]) + " was never produced");
  if (rec_[i].on_gpu && rec_[i].copy_in_flight) stall_until(inflight_done_[i], i);
  const TensorRecord& r = rec_[i];
  if (r.on_gpu) return;
  if (r.swapout && r.copy_in_flight) {  // join the in-flight reload
    stall_until(inflight_done_[i], i);
    return;
  }
  bool host_ok = r.swapout || (r.dead && r.cpu_copy_valid);
  if (host_ok && (r.uncomputable || mode == Restore::ClosureDep)) {
    demand_reload(i);
    return;
  }
  rebuild(i);
}

void Planner::demand_reload(Idx i) {
  const Bytes bytes = rec_[i].bytes;
  alloc_bytes(bytes, i);
  const MicroDur d = transfer_time_us(bytes, cfg_.cost_model);
  apply(i, TensorEvent::ReloadStart, clock_.now());
  queue_remove(i);
  ++counts_.reload;
  copy_busy_ += d;
  if (cfg_.overlap_enabled) {
    MicroTime start = submit_copy(d);
    log(EventKind::Reload, start, d, i, bytes, StreamKind::Copy);
    pending_.push({start + d, seq_++, false, i, bytes});
    inflight_done_[i] = start + d;
    stall_until(start + d, i);
  } else {
    MicroTime start = submit_compute(d);
    log(EventKind::Reload, start, d, i, bytes, StreamKind::Compute);
    clock_.advance_to(start + d);
    copy_stall_ += d;
    apply(i, TensorEvent::ReloadDone, start + d);
    restored_.push_back(i);
  }
}

// Recompute engine on the logical clock (ref engine.cpp:423-454).
void Planner::rebuild(Idx i) {
  const OpNode& node = trace_.nodes[i];
  if (node.uncomputable) {
    if (rec_[i].cpu_copy_valid) {
      demand_reload(i);
      return;
    }
    throw UnrecoverableError("node " + std::to_string(ids_[i]) +
                             " is uncomputable and has no host copy");
  }
  std::vector<Idx> held;
  for (Idx o = parent_off_[i]; o < parent_off_[i + 1]; ++o) {
    ensure_resident(parent_idx_[o], Restore::ClosureDep);
    pin(parent_idx_[o], held);
  }
  const bool was_swapout = rec_[i].swapout;
  if (was_swapout) queue_remove(i);
  alloc_bytes(node.output_bytes, i);
  MicroTime start = submit_compute(node.compute_cost_us);
  MicroTime end = start + node.compute_cost_us;
  clock_.advance_to(end);
  log(EventKind::Recompute, start, node.compute_cost_us, i, node.output_bytes,
      StreamKind::Compute);
  for (Idx o = parent_off_[i]; o < parent_off_[i + 1]; ++o)
    apply(parent_idx_[o], TensorEvent::Use, end);
  apply(i, TensorEvent::RecomputeDone, end);
  ++counts_.recompute;
  if (was_swapout) ++counts_.recompute_of_swapout;
  restored_.push_back(i);
  unpin_all(held);
}

void Planner::do_produce(Idx i) {
  const OpNode& node = trace_.nodes[i];
  std::vector<Idx> held;
  for (Idx o = parent_off_[i]; o < parent_off_[i + 1]; ++o) {
    ensure_resident(parent_idx_[o], Restore::Access);
    pin(parent_idx_[o], held);
  }
  alloc_bytes(node.output_bytes, i);
  produce(i, clock_.now());
  pin(i, held);
  if (releases_allowed()) watermark_loop();
  MicroTime start = submit_compute(node.compute_cost_us);
  MicroTime end = start + node.compute_cost_us;
  clock_.advance_to(end);
  log(EventKind::Compute, start, node.compute_cost_us, i, node.output_bytes,
      StreamKind::Compute);
  for (Idx o = parent_off_[i]; o < parent_off_[i + 1]; ++o)
    apply(parent_idx_[o], TensorEvent::Use, end);
  apply(i, TensorEvent::Use, end);
  unpin_all(held);
}

void Planner::do_use(Idx i) {
  ensure_resident(i, Restore::Access);
  MicroTime now = clock_.now();
  apply(i, TensorEvent::Use, now);
  log(EventKind::Use, now, 0, i, rec_[i].bytes, StreamKind::Compute);
}

void Planner::reclaim(Idx i, std::size_t k) {
  if (!produced_[i]) return;
  TensorRecord& r = rec_[i];
  if (r.dead) return;
  if (trace_.nodes[i].uncomputable && !r.cpu_copy_valid &&
      extended_last_[i] > std::ptrdiff_t(k))
    return;
  if (r.copy_in_flight) {
    dead_pending_[i] = 1;
    return;
  }
  const MicroTime now = clock_.now();
  if (r.on_gpu) {
    const Bytes b = r.bytes;
    pool_free(i, b);
    apply(i, TensorEvent::FreeDead, now);
    log(EventKind::Free, now, 0, i, b, StreamKind::Compute);
  } else {
    if (r.swapout) queue_remove(i);
    apply(i, TensorEvent::FreeDead, now);
  }
}

void Planner::sweep_dead(std::size_t k) {
  for (Idx o = death_off_[k]; o < death_off_[k + 1]; ++o) reclaim(death_idx_[o], k);
  for (std::size_t j = 0; j < restored_.size(); ++j) {
    Idx i = restored_[j];
    if (last_access_[i] >= 0 && std::size_t(last_access_[i]) <= k) reclaim(i, k);
  }
  restored_.clear();
}

// Prefetcher (Algorithm 4; ref engine.cpp:533-585).
void Planner::prefetch_burst() {
  if (!cfg_.prefetch_enabled) return;
  drain(clock_.now());
  std::uint64_t issued = 0;
  bool opened = false;
  while (!queue_.empty()) {
    const Idx head = queue_.front();
    const Bytes bytes = rec_[head].bytes;
    const bool fits = pool_.used() + bytes <= mark_;
    if (!fits) break;
    if (cfg_.prefetch_guard == PrefetchGuard::And && issued >= cfg_.prefetch_limit)
      break;
    if (!opened) {
      opened = true;
      ++burst_;
    }
    if (!pool_alloc(head, bytes))
      throw InternalError("prefetch allocation failed after fit check");
    const MicroDur d = transfer_time_us(bytes, cfg_.cost_model);
    apply(head, TensorEvent::ReloadStart, clock_.now());
    queue_.pop_front();
    ++counts_.reload;
    ++counts_.prefetch_reload;
    copy_busy_ += d;
    if (cfg_.overlap_enabled) {
      MicroTime start = submit_copy(d);
      log(EventKind::Reload, start, d, head, bytes, StreamKind::Copy, true, burst_);
      pending_.push({start + d, seq_++, false, head, bytes});
      inflight_done_[head] = start + d;
    } else {
      MicroTime start = submit_compute(d);
      log(EventKind::Reload, start, d, head, bytes, StreamKind::Compute, true,
          burst_);
      clock_.advance_to(start + d);
      copy_stall_ += d;
      apply(head, TensorEvent::ReloadDone, start + d);
      restored_.push_back(head);
    }
    ++issued;
  }
}

RunResult Planner::run() {
  const std::size_t E = trace_.schedule.size();
  try {
    for (std::size_t k = 0; k < E; ++k) {
      const AccessEvent& ev = trace_.schedule[k];
      if (phase_ == Phase::Forward && ev.phase == Phase::Backward) {
        phase_ = Phase::Backward;
        prefetch_burst();
      }
      const std::uint64_t before = compute_submits_;
      if (ev.kind == AccessKind::Produce)
        do_produce(sched_node_[k]);
      else
        do_use(sched_node_[k]);
      sweep_dead(k);
      if (phase_ == Phase::Backward && compute_submits_ > before) prefetch_burst();
    }
  } catch (const Infeasible& e) {
    infeasible_ = e.info;
  }
  drain(std::numeric_limits<MicroTime>::max());

  RunResult out;
  out.timeline.events = std::move(events_);
  for (Idx r = 0; r < n_; ++r) {
    Idx i = by_rank_[r];
    if (produced_[i]) out.final_set.append_sorted(rec_[i]);
  }
  out.infeasible = infeasible_;
  out.peak_bytes = pool_.high_watermark();
  out.wall_time_us = std::max(compute_busy_, copy_busy_until_);
  out.total_stall_us = total_stall_;
  out.copy_busy_us = copy_busy_;
  out.copy_stall_us = copy_stall_;
  out.counts = counts_;
  out.decisions = std::move(decisions_);
  return out;
}

}  // namespace

RunResult run_iteration_unchecked(const Trace& trace, const EngineConfig& cfg) {
  Planner p(trace, cfg, nullptr);
  return p.run();
}

RunResult run_iteration_pool_log(const Trace& trace, const EngineConfig& cfg,
                                 std::vector<PoolOp>* pool_ops) {
  if (!trace_is_valid(trace))
    throw ValidationErrorEx("run_iteration: trace fails validation");
  Planner p(trace, cfg, pool_ops);
  return p.run();
}

RunResult run_iteration(const Trace& trace, const EngineConfig& cfg) {
  if (!trace_is_valid(trace))
    throw ValidationErrorEx("run_iteration: trace fails validation");
  return run_iteration_unchecked(trace, cfg);
}

RunResult run_unconstrained_baseline(const Trace& trace,
                                     const EngineConfig& base_cfg) {
  Bytes total = 0;
  for (const OpNode& n : trace.nodes) total += n.output_bytes;
  EngineConfig cfg = base_cfg;
  cfg.policy_mode = PolicyMode::Baseline;
  cfg.budget = total == 0 ? 1 : total;
  cfg.scripted_decisions.clear();
  return run_iteration(trace, cfg);
}

ComparisonReport run_comparison(const Trace& trace,
                                const std::vector<Bytes>& budgets,
                                const std::vector<PolicyMode>& policies,
                                const std::vector<Heuristic>& heuristics,
                                const EngineConfig& base_cfg) {
  ComparisonReport rep;
  rep.trace_name = trace.name;
  rep.baseline = run_unconstrained_baseline(trace, base_cfg);
  for (Bytes b : budgets)
    for (PolicyMode p : policies)
      for (Heuristic h : heuristics) {
        EngineConfig cfg = base_cfg;
        cfg.budget = b;
        cfg.policy_mode = p;
        cfg.heuristic = h;
        rep.cells.push_back({b, p, h, run_iteration(trace, cfg)});
      }
  return rep;
}

}  // namespace deltasim
