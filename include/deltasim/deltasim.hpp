// delta-b200: drop-in replacement for the reference `deltasim` C++ API.
//
// Every type and free function below keeps the name, field order and
// signature of the reference interface it replaces, so code written against
// the reference (its CLI, its acceptance suite tests/acceptance_main.cpp)
// compiles unmodified against libdelta.  Citations are to
// /root/reference/proj/include/deltasim/*.hpp.
//
// The implementation is new: a flat-array planner (csrc/plan/) that
// reproduces the reference decisions bit-exactly on its logical integer
// clock, feeding a B200 executor (csrc/rt/, csrc/kernels/).
#pragma once

#include <cstddef>
#include <cstdint>
#include <deque>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

namespace deltasim {

// ---- units and exact arithmetic (ref types.hpp:9-33) ----------------------
using NodeId = std::uint64_t;
using Bytes = std::uint64_t;
using MicroTime = std::uint64_t;  // logical planner clock, microseconds
using MicroDur = std::uint64_t;
using U128 = unsigned __int128;

struct Frac64 {
  std::uint64_t num = 0;
  std::uint64_t den = 1;
  constexpr bool operator==(const Frac64&) const = default;
};

// Reciprocal heuristic score kept as its denominator; a LARGER `inv` is a
// SMALLER score (ref types.hpp:27-33).
struct HeuristicScore {
  U128 inv = 1;
  bool operator==(const HeuristicScore& o) const { return inv == o.inv; }
  bool operator<(const HeuristicScore& o) const { return inv > o.inv; }
  bool operator<=(const HeuristicScore& o) const { return inv >= o.inv; }
};

// ---- error taxonomy (ref types.hpp:35-65) ----------------------------------
#define DELTASIM_ERROR(Name)                 \
  struct Name : std::runtime_error {         \
    using std::runtime_error::runtime_error; \
  }
DELTASIM_ERROR(SchemaError);
DELTASIM_ERROR(ValidationErrorEx);
DELTASIM_ERROR(ArgumentError);
DELTASIM_ERROR(StateError);
DELTASIM_ERROR(IllegalTransition);
DELTASIM_ERROR(UnrecoverableError);
DELTASIM_ERROR(MismatchedTrace);
DELTASIM_ERROR(TooLarge);
DELTASIM_ERROR(IoError);
DELTASIM_ERROR(InternalError);
#undef DELTASIM_ERROR

std::string u128_to_string(U128 v);

// ---- tensor registration: op graph + access schedule (ref trace.hpp) -------
enum class Phase : std::uint8_t { Forward, Backward };
enum class AccessKind : std::uint8_t { Produce, Use };

struct OpNode {
  NodeId id = 0;
  std::string name;
  MicroDur compute_cost_us = 0;
  Bytes output_bytes = 0;
  std::vector<NodeId> parents;
  bool uncomputable = false;
  bool evict_pinned = false;
  bool offload_pinned = false;
};

struct AccessEvent {
  NodeId node = 0;
  Phase phase = Phase::Forward;
  AccessKind kind = AccessKind::Produce;
  bool operator==(const AccessEvent&) const = default;
};

struct Trace {
  std::string name;
  std::vector<OpNode> nodes;
  std::vector<AccessEvent> schedule;
  std::optional<std::size_t> index_of(NodeId id) const;
  const OpNode* find(NodeId id) const;
};

enum class TraceViolationCode {
  DuplicateNodeId,
  CycleOrForwardRef,
  UncomputableHasParents,
  UncomputableNotEvictPinned,
  BothPinned,
  DanglingNodeRef,
  UseBeforeProduce,
  DuplicateProduce,
  ParentNotProduced,
  ForwardAfterBackward,
  ZeroOutputBytes,
};
enum class Severity { Error, Warning };

struct TraceViolation {
  TraceViolationCode code;
  Severity severity = Severity::Error;
  std::optional<NodeId> node;
  std::optional<std::size_t> event_index;
  std::string message;
};

const char* to_string(TraceViolationCode c);
std::vector<TraceViolation> validate_trace(const Trace& t);
bool trace_is_valid(const Trace& t);
Trace parse_trace(const std::string& text);
std::string serialize_trace(const Trace& t);
Trace gen_linear_chain(std::size_t n, Bytes bytes_per, MicroDur cost_per,
                       std::uint64_t seed);
Trace gen_resnet_like(std::size_t blocks, Bytes branch_bytes,
                      std::uint64_t seed);
Trace gen_transformer_like(std::size_t layers, Bytes hidden_bytes,
                           std::uint64_t seed);

// ---- per-tensor state machine (ref state.hpp) -----------------------------
enum class TensorEvent : std::uint8_t {
  Produce,
  Use,
  EvictStart,
  OffloadStart,
  OffloadDone,
  ReloadStart,
  ReloadDone,
  RecomputeDone,
  FreeAfterOffload,
  FreeDead,
};
const char* to_string(TensorEvent e);

struct TensorRecord {
  NodeId node_id = 0;
  Bytes bytes = 0;
  MicroDur own_cost = 0;
  bool on_gpu = false;
  bool evicted = false;
  bool swapout = false;
  bool uncomputable = false;
  bool evict_pinned = false;
  bool offload_pinned = false;
  bool in_use = false;
  bool copy_in_flight = false;
  bool cpu_copy_valid = false;
  bool produced_backward = false;
  bool dead = false;
  bool died_swapout = false;
  MicroTime last_access = 0;
  bool location_invariant_holds() const;
};

MicroDur staleness(const TensorRecord& r, MicroTime now);
TensorRecord transition(const TensorRecord& r, TensorEvent ev, MicroTime now);

// Produced tensors in ascending id order (std::map: references returned by
// produce()/at() stay valid across later inserts, as in the reference).  The
// engine keeps its own dense table and only materialises this set for
// RunResult::final_set and for the free policy functions.
class ResidentSet {
 public:
  TensorRecord& produce(const OpNode& node, MicroTime now, Phase phase);
  TensorRecord& apply(NodeId id, TensorEvent ev, MicroTime now);
  bool contains(NodeId id) const;
  const TensorRecord& at(NodeId id) const;
  TensorRecord& at(NodeId id);
  Bytes resident_bytes() const { return resident_bytes_; }
  Bytes recount_resident_bytes() const;
  void check_resident_bytes() const;
  auto begin() const { return records_.begin(); }
  auto end() const { return records_.end(); }
  std::size_t size() const { return records_.size(); }

  // libdelta extension: append a record whose id exceeds every present id.
  void append_sorted(const TensorRecord& r);

 private:
  std::map<NodeId, TensorRecord> records_;
  Bytes resident_bytes_ = 0;
};

// ---- simulated device (ref device.hpp) — kept for API parity; the planner
// ---- uses the same semantics, the executor replaces it with HBM/CUDA. ----
struct Allocated {};
struct Insufficient {
  Bytes deficit = 0;
};
using AllocResult = std::variant<Allocated, Insufficient>;

class MemoryPool {
 public:
  explicit MemoryPool(Bytes budget) : budget_(budget) {}
  AllocResult try_alloc(Bytes n);
  void free(Bytes n);
  Bytes budget() const { return budget_; }
  Bytes used() const { return used_; }
  Bytes available() const { return budget_ - used_; }
  Bytes high_watermark() const { return high_watermark_; }

 private:
  Bytes budget_;
  Bytes used_ = 0;
  Bytes high_watermark_ = 0;
};

enum class StreamKind : std::uint8_t { Compute, Copy };

struct StreamInterval {
  MicroTime start;
  MicroTime end;
  std::string label;
  NodeId node;
};

class Stream {
 public:
  explicit Stream(StreamKind kind) : kind_(kind) {}
  std::pair<MicroTime, MicroTime> submit(MicroTime now, MicroDur duration,
                                         std::string label, NodeId node);
  StreamKind kind() const { return kind_; }
  MicroTime busy_until() const { return busy_until_; }
  MicroDur busy_total() const { return busy_total_; }
  const std::vector<StreamInterval>& log() const { return log_; }

 private:
  StreamKind kind_;
  MicroTime busy_until_ = 0;
  MicroDur busy_total_ = 0;
  std::vector<StreamInterval> log_;
};

class Clock {
 public:
  MicroTime now() const { return now_; }
  MicroDur wait_for(MicroTime t);
  void advance_to(MicroTime t);

 private:
  MicroTime now_ = 0;
};

// ---- Filter + Director + cost model (ref policy.hpp) ----------------------
enum class Heuristic : std::uint8_t { Base, Lru, Greedy };
enum class ReleaseAction : std::uint8_t { Evict, Offload };
enum class SwapCostMode : std::uint8_t { OneWay, RoundTrip };
const char* to_string(Heuristic h);
const char* to_string(ReleaseAction a);

struct CostModel {
  Frac64 bandwidth_bytes_per_us{64000, 1};
  Frac64 effective_fraction{7, 20};
  SwapCostMode swap_cost_mode = SwapCostMode::OneWay;
  U128 eff_num() const;
  U128 eff_den() const;
};

struct DecisionScore {
  U128 num = 0;
  U128 den = 1;
  bool leq_one() const { return num <= den; }
};

struct Decision {
  ReleaseAction action;
  std::optional<DecisionScore> score;
};

HeuristicScore score(Heuristic h, const TensorRecord& r, MicroTime now);
MicroDur swap_cost(const TensorRecord& r, const CostModel& cm);
MicroDur swap_cost_bytes(Bytes m, const CostModel& cm);
MicroDur transfer_time_us(Bytes m, const CostModel& cm);  // one-way
MicroDur recompute_cost(NodeId id, const ResidentSet& set, const Trace& trace);
bool releasable(const TensorRecord& r);
std::optional<NodeId> select_victim(const ResidentSet& set, Heuristic h,
                                    MicroTime now);
std::optional<NodeId> select_victim(const ResidentSet& set, Heuristic h,
                                    MicroTime now,
                                    bool (*extra_filter)(const TensorRecord&));
Decision decide(NodeId id, const ResidentSet& set, const Trace& trace,
                const CostModel& cm, MicroTime now);

// ---- training-step executor: plan on the logical clock (ref engine.hpp) ---
enum class PolicyMode : std::uint8_t { Delta, RecomputeOnly, OffloadOnly, Baseline };
enum class PrefetchGuard : std::uint8_t { And, PaperOr };
const char* to_string(PolicyMode m);

struct EngineConfig {
  Bytes budget = 0;
  Heuristic heuristic = Heuristic::Base;
  PolicyMode policy_mode = PolicyMode::Delta;
  CostModel cost_model;
  Frac64 watermark_fraction{3, 4};
  std::uint64_t prefetch_limit = 2;
  bool prefetch_enabled = true;
  bool overlap_enabled = true;
  PrefetchGuard prefetch_guard = PrefetchGuard::And;
  std::vector<std::pair<NodeId, ReleaseAction>> scripted_decisions;
  Bytes watermark_bytes() const;
};

enum class EventKind : std::uint8_t {
  Compute,
  Offload,
  Reload,
  Recompute,
  Stall,
  Evict,
  Use,
  Free,
};
const char* to_string(EventKind k);

struct TimelineEvent {
  MicroTime ts = 0;
  StreamKind stream = StreamKind::Compute;
  EventKind kind = EventKind::Compute;
  NodeId node = 0;
  MicroDur duration = 0;
  Bytes bytes = 0;
  Phase phase = Phase::Forward;
  bool prefetch = false;
  std::uint32_t burst = 0;
};

struct Timeline {
  std::vector<TimelineEvent> events;
};

struct OffloadQueue {
  std::deque<NodeId> fifo;
  void push(NodeId id) { fifo.push_back(id); }
  void remove(NodeId id);
  bool empty() const { return fifo.empty(); }
  NodeId front() const { return fifo.front(); }
  void pop() { fifo.pop_front(); }
};

struct InfeasibleInfo {
  NodeId node = 0;
  Bytes deficit = 0;
};

struct ActionCounts {
  std::uint64_t evict = 0;
  std::uint64_t offload = 0;
  std::uint64_t reload = 0;
  std::uint64_t recompute = 0;
  std::uint64_t prefetch_reload = 0;
  std::uint64_t recompute_of_swapout = 0;
};

struct RunResult {
  Timeline timeline;
  ResidentSet final_set;
  std::optional<InfeasibleInfo> infeasible;
  Bytes peak_bytes = 0;
  MicroTime wall_time_us = 0;
  MicroDur total_stall_us = 0;
  MicroDur copy_busy_us = 0;
  MicroDur copy_stall_us = 0;
  ActionCounts counts;
  std::vector<std::pair<NodeId, ReleaseAction>> decisions;
  bool completed() const { return !infeasible.has_value(); }
};

RunResult run_iteration(const Trace& trace, const EngineConfig& cfg);

struct ComparisonCell {
  Bytes budget = 0;
  PolicyMode policy = PolicyMode::Delta;
  Heuristic heuristic = Heuristic::Base;
  RunResult result;
};

struct ComparisonReport {
  std::string trace_name;
  RunResult baseline;
  std::vector<ComparisonCell> cells;
};

ComparisonReport run_comparison(const Trace& trace,
                                const std::vector<Bytes>& budgets,
                                const std::vector<PolicyMode>& policies,
                                const std::vector<Heuristic>& heuristics,
                                const EngineConfig& base_cfg);
RunResult run_unconstrained_baseline(const Trace& trace,
                                     const EngineConfig& base_cfg);

// libdelta extension: the planner run on an already-validated trace (the
// executor re-plans with the same trace every time the cost table changes).
RunResult run_iteration_unchecked(const Trace& trace, const EngineConfig& cfg);

// libdelta extension: every MemoryPool alloc/free the planner performed, in
// order, each tagged with the number of timeline events logged before it.
// The B200 arena lowering replays this sequence so that its live set equals
// the planner's pool at every step (csrc/rt/lower.cpp).
struct PoolOp {
  std::uint64_t before_event;  // timeline index the op precedes
  NodeId node;
  Bytes bytes;
  bool alloc;                  // false = free
};
RunResult run_iteration_pool_log(const Trace& trace, const EngineConfig& cfg,
                                 std::vector<PoolOp>* pool_ops);

// ---- report / chrome-trace parity surface (ref metrics.hpp) ---------------
struct Report {
  Bytes peak_bytes = 0;
  Bytes baseline_peak_bytes = 0;
  double saving_fraction = 0.0;
  MicroTime wall_time_us = 0;
  MicroTime baseline_wall_time_us = 0;
  double overhead_fraction = 0.0;
  std::uint64_t evict_count = 0;
  std::uint64_t offload_count = 0;
  std::uint64_t reload_count = 0;
  std::uint64_t recompute_count = 0;
  std::uint64_t prefetch_reload_count = 0;
  MicroDur total_stall_us = 0;
  double overlap_ratio = 1.0;
  bool infeasible = false;
};

Report summarize(const Timeline& timeline, const Timeline& baseline);
Report summarize(const RunResult& run, const RunResult& baseline);
enum class ReportFormat : std::uint8_t { Json, Csv };
std::string report_to_json(const Report& r);
std::string report_to_csv(const Report& r);
Report report_from_json(const std::string& text);
std::size_t write_report(const Report& r, ReportFormat format,
                         const std::string& path);
std::string timeline_to_chrome_trace(const Timeline& t);
Timeline timeline_from_chrome_trace(const std::string& text);
std::size_t write_chrome_trace(const Timeline& t, const std::string& path);
std::string comparison_to_csv(const ComparisonReport& rep);
std::string comparison_to_json(const ComparisonReport& rep);

}  // namespace deltasim
