// extern "C" boundary over the libdelta planner and plan lowering
// (include/delta/delta.h).  Exceptions never cross: each C++ exception class
// of the reference taxonomy maps to its own status code and the message is
// kept in a thread-local buffer for delta_last_error().
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../rt/lower.hpp"
#include "delta/delta.h"
#include "deltasim/deltasim.hpp"

using namespace deltasim;

struct delta_trace {
  Trace t;
};
struct delta_result {
  RunResult r;
  std::vector<delta_event> events;
  std::vector<delta_decision> decisions;
};
struct delta_program {
  delta_rt::Program p;
  delta_result plan;
};

namespace {

thread_local std::string g_err;

template <class F>
delta_status guard(F&& f) {
  try {
    f();
    g_err.clear();
    return DELTA_OK;
  } catch (const SchemaError& e) { g_err = e.what(); return DELTA_E_SCHEMA; }
  catch (const ValidationErrorEx& e) { g_err = e.what(); return DELTA_E_VALIDATION; }
  catch (const ArgumentError& e) { g_err = e.what(); return DELTA_E_ARGUMENT; }
  catch (const StateError& e) { g_err = e.what(); return DELTA_E_STATE; }
  catch (const IllegalTransition& e) { g_err = e.what(); return DELTA_E_ILLEGAL; }
  catch (const UnrecoverableError& e) { g_err = e.what(); return DELTA_E_UNRECOVERABLE; }
  catch (const MismatchedTrace& e) { g_err = e.what(); return DELTA_E_MISMATCHED; }
  catch (const TooLarge& e) { g_err = e.what(); return DELTA_E_TOO_LARGE; }
  catch (const IoError& e) { g_err = e.what(); return DELTA_E_IO; }
  catch (const InternalError& e) { g_err = e.what(); return DELTA_E_INTERNAL; }
  catch (const std::exception& e) { g_err = e.what(); return DELTA_E_UNKNOWN; }
  catch (...) { g_err = "unknown exception"; return DELTA_E_UNKNOWN; }
}

char* dup_str(const std::string& s, uint64_t* len) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (!p) throw std::bad_alloc();
  std::memcpy(p, s.data(), s.size() + 1);
  if (len) *len = s.size();
  return p;
}

EngineConfig to_cfg(const delta_config* c) {
  if (!c) throw ArgumentError("null config");
  EngineConfig cfg;
  cfg.budget = c->budget;
  if (c->heuristic > 2) throw ArgumentError("bad heuristic");
  if (c->policy_mode > 3) throw ArgumentError("bad policy mode");
  cfg.heuristic = static_cast<Heuristic>(c->heuristic);
  cfg.policy_mode = static_cast<PolicyMode>(c->policy_mode);
  if (c->bw_den == 0 || c->eff_den == 0 || c->watermark_den == 0)
    throw ArgumentError("zero denominator in config");
  if (c->bw_num == 0 || c->eff_num == 0) throw ArgumentError("bandwidth must be positive");
  cfg.cost_model.bandwidth_bytes_per_us = {c->bw_num, c->bw_den};
  cfg.cost_model.effective_fraction = {c->eff_num, c->eff_den};
  cfg.cost_model.swap_cost_mode =
      c->swap_cost_mode ? SwapCostMode::RoundTrip : SwapCostMode::OneWay;
  cfg.watermark_fraction = {c->watermark_num, c->watermark_den};
  cfg.prefetch_limit = c->prefetch_limit;
  cfg.prefetch_enabled = c->prefetch_enabled != 0;
  cfg.overlap_enabled = c->overlap_enabled != 0;
  cfg.prefetch_guard = c->prefetch_guard ? PrefetchGuard::PaperOr : PrefetchGuard::And;
  for (uint64_t i = 0; i < c->n_scripted; ++i)
    cfg.scripted_decisions.emplace_back(
        c->scripted_nodes[i],
        c->scripted_actions[i] ? ReleaseAction::Offload : ReleaseAction::Evict);
  return cfg;
}

void fill(delta_result* out) {
  out->events.clear();
  out->events.reserve(out->r.timeline.events.size());
  for (const TimelineEvent& e : out->r.timeline.events) {
    delta_event d{};
    d.ts = e.ts;
    d.node = e.node;
    d.duration = e.duration;
    d.bytes = e.bytes;
    d.burst = e.burst;
    d.stream = static_cast<uint8_t>(e.stream);
    d.kind = static_cast<uint8_t>(e.kind);
    d.phase = static_cast<uint8_t>(e.phase);
    d.prefetch = e.prefetch ? 1 : 0;
    out->events.push_back(d);
  }
  out->decisions.clear();
  for (auto& [n, a] : out->r.decisions) out->decisions.push_back({n, uint32_t(a), 0});
}

}  // namespace

namespace delta_rt {
void set_error(const std::string& msg) { g_err = msg; }
}  // namespace delta_rt

// for translation units that also see the C type `delta_rt` (rt/executor.cu)
void delta_set_error(const std::string& msg) { delta_rt::set_error(msg); }

namespace delta_rt {
}  // namespace delta_rt

extern "C" {

const char* delta_last_error(void) { return g_err.c_str(); }
void delta_free(void* p) { std::free(p); }
const char* delta_version(void) { return "delta-b200 0.1 (sm_100a)"; }

delta_status delta_trace_new(const char* name, delta_trace** out) {
  return guard([&] {
    auto* t = new delta_trace;
    t->t.name = name ? name : "";
    *out = t;
  });
}

delta_status delta_trace_add_node(delta_trace* t, uint64_t id, const char* name,
                                  uint64_t cost, uint64_t bytes,
                                  const uint64_t* parents, uint64_t n_parents,
                                  uint32_t flags) {
  return guard([&] {
    OpNode n;
    n.id = id;
    n.name = name ? name : "";
    n.compute_cost_us = cost;
    n.output_bytes = bytes;
    n.parents.assign(parents, parents + n_parents);
    n.uncomputable = flags & DELTA_NODE_UNCOMPUTABLE;
    n.evict_pinned = flags & DELTA_NODE_EVICT_PINNED;
    n.offload_pinned = flags & DELTA_NODE_OFFLOAD_PINNED;
    t->t.nodes.push_back(std::move(n));
  });
}

delta_status delta_trace_add_event(delta_trace* t, uint64_t node, uint32_t phase,
                                   uint32_t kind) {
  return guard([&] {
    if (phase > 1 || kind > 1) throw ArgumentError("bad phase/kind");
    t->t.schedule.push_back({node, static_cast<Phase>(phase), static_cast<AccessKind>(kind)});
  });
}

delta_status delta_trace_set_cost(delta_trace* t, uint64_t id, uint64_t cost) {
  return guard([&] {
    for (OpNode& n : t->t.nodes)
      if (n.id == id) {
        n.compute_cost_us = cost;
        return;
      }
    throw ArgumentError("set_cost: unknown node " + std::to_string(id));
  });
}

delta_status delta_trace_parse(const char* json, uint64_t len, delta_trace** out) {
  return guard([&] {
    auto* t = new delta_trace;
    try {
      t->t = parse_trace(std::string(json, len));
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

delta_status delta_trace_serialize(const delta_trace* t, char** out, uint64_t* len) {
  return guard([&] { *out = dup_str(serialize_trace(t->t), len); });
}

delta_status delta_trace_validate(const delta_trace* t, uint32_t* n_err,
                                  uint32_t* n_warn, char** first_error) {
  return guard([&] {
    uint32_t e = 0, w = 0;
    std::string first;
    for (const TraceViolation& v : validate_trace(t->t)) {
      if (v.severity == Severity::Error) {
        if (e++ == 0) first = std::string(to_string(v.code)) + ": " + v.message;
      } else {
        ++w;
      }
    }
    if (n_err) *n_err = e;
    if (n_warn) *n_warn = w;
    if (first_error) *first_error = e ? dup_str(first, nullptr) : nullptr;
  });
}

uint64_t delta_trace_num_nodes(const delta_trace* t) { return t->t.nodes.size(); }
uint64_t delta_trace_num_events(const delta_trace* t) { return t->t.schedule.size(); }
void delta_trace_free(delta_trace* t) { delete t; }

void delta_config_default(delta_config* c) {
  EngineConfig d;
  std::memset(c, 0, sizeof(*c));
  c->budget = 0;
  c->heuristic = DELTA_HEUR_BASE;
  c->policy_mode = DELTA_POLICY_DELTA;
  c->bw_num = d.cost_model.bandwidth_bytes_per_us.num;
  c->bw_den = d.cost_model.bandwidth_bytes_per_us.den;
  c->eff_num = d.cost_model.effective_fraction.num;
  c->eff_den = d.cost_model.effective_fraction.den;
  c->swap_cost_mode = 0;
  c->prefetch_guard = 0;
  c->watermark_num = d.watermark_fraction.num;
  c->watermark_den = d.watermark_fraction.den;
  c->prefetch_limit = d.prefetch_limit;
  c->prefetch_enabled = 1;
  c->overlap_enabled = 1;
}

delta_status delta_plan(const delta_trace* t, const delta_config* c, delta_result** out) {
  return guard([&] {
    auto* r = new delta_result;
    try {
      r->r = run_iteration(t->t, to_cfg(c));
      fill(r);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

delta_status delta_plan_baseline(const delta_trace* t, const delta_config* c,
                                 delta_result** out) {
  return guard([&] {
    auto* r = new delta_result;
    try {
      r->r = run_unconstrained_baseline(t->t, to_cfg(c));
      fill(r);
    } catch (...) {
      delete r;
      throw;
    }
    *out = r;
  });
}

delta_status delta_result_summary(const delta_result* res, delta_summary* s) {
  return guard([&] {
    const RunResult& r = res->r;
    std::memset(s, 0, sizeof(*s));
    s->peak_bytes = r.peak_bytes;
    s->wall_time_us = r.wall_time_us;
    s->total_stall_us = r.total_stall_us;
    s->copy_busy_us = r.copy_busy_us;
    s->copy_stall_us = r.copy_stall_us;
    s->evict = r.counts.evict;
    s->offload = r.counts.offload;
    s->reload = r.counts.reload;
    s->recompute = r.counts.recompute;
    s->prefetch_reload = r.counts.prefetch_reload;
    s->recompute_of_swapout = r.counts.recompute_of_swapout;
    s->infeasible = r.infeasible ? 1 : 0;
    if (r.infeasible) {
      s->infeasible_node = r.infeasible->node;
      s->infeasible_deficit = r.infeasible->deficit;
    }
    s->n_events = res->events.size();
    s->n_decisions = res->decisions.size();
  });
}

const delta_event* delta_result_events(const delta_result* r, uint64_t* n) {
  if (n) *n = r->events.size();
  return r->events.data();
}

const delta_decision* delta_result_decisions(const delta_result* r, uint64_t* n) {
  if (n) *n = r->decisions.size();
  return r->decisions.data();
}

delta_status delta_report_json(const delta_result* run, const delta_result* base,
                               char** out, uint64_t* len) {
  return guard([&] { *out = dup_str(report_to_json(summarize(run->r, base->r)), len); });
}

delta_status delta_comparison(const delta_trace* t, const delta_config* base,
                              const uint64_t* budgets, uint64_t n_budgets,
                              const uint32_t* policies, uint64_t n_policies,
                              const uint32_t* heuristics, uint64_t n_heuristics, int32_t json,
                              char** out, uint64_t* len) {
  return guard([&] {
    std::vector<Bytes> b(budgets, budgets + n_budgets);
    std::vector<PolicyMode> p;
    for (uint64_t i = 0; i < n_policies; ++i) {
      if (policies[i] > uint32_t(PolicyMode::Baseline)) throw ArgumentError("comparison: bad policy");
      p.push_back(static_cast<PolicyMode>(policies[i]));
    }
    std::vector<Heuristic> h;
    for (uint64_t i = 0; i < n_heuristics; ++i) {
      if (heuristics[i] > uint32_t(Heuristic::Greedy)) throw ArgumentError("comparison: bad heuristic");
      h.push_back(static_cast<Heuristic>(heuristics[i]));
    }
    const ComparisonReport rep = run_comparison(t->t, b, p, h, to_cfg(base));
    *out = dup_str(json ? comparison_to_json(rep) : comparison_to_csv(rep), len);
  });
}

delta_status delta_chrome_trace(const delta_result* r, char** out, uint64_t* len) {
  return guard([&] { *out = dup_str(timeline_to_chrome_trace(r->r.timeline), len); });
}

delta_status delta_chrome_trace_events(const delta_event* ev, uint64_t n, char** out,
                                       uint64_t* len) {
  return guard([&] {
    Timeline t;
    t.events.reserve(n);
    for (uint64_t i = 0; i < n; ++i) {
      TimelineEvent e;
      e.ts = ev[i].ts;
      e.node = ev[i].node;
      e.duration = ev[i].duration;
      e.bytes = ev[i].bytes;
      e.burst = ev[i].burst;
      if (ev[i].stream > 1 || ev[i].kind > static_cast<uint8_t>(EventKind::Free) || ev[i].phase > 1)
        throw ArgumentError("chrome_trace_events: bad event " + std::to_string(i));
      e.stream = static_cast<StreamKind>(ev[i].stream);
      e.kind = static_cast<EventKind>(ev[i].kind);
      e.phase = static_cast<Phase>(ev[i].phase);
      e.prefetch = ev[i].prefetch != 0;
      t.events.push_back(e);
    }
    *out = dup_str(timeline_to_chrome_trace(t), len);
  });
}

void delta_result_free(delta_result* r) { delete r; }

delta_status delta_plan_time_ns(const delta_trace* t, const delta_config* c,
                                uint32_t iters, double* ns) {
  return guard([&] {
    EngineConfig cfg = to_cfg(c);
    if (iters == 0) iters = 1;
    volatile uint64_t sink = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (uint32_t i = 0; i < iters; ++i) sink += run_iteration(t->t, cfg).wall_time_us;
    auto t1 = std::chrono::steady_clock::now();
    (void)sink;
    *ns = std::chrono::duration<double, std::nano>(t1 - t0).count() / iters;
  });
}

delta_status delta_transfer_time_us(uint64_t bytes, const delta_config* c, uint64_t* us) {
  return guard([&] { *us = transfer_time_us(bytes, to_cfg(c).cost_model); });
}

delta_status delta_lower(const delta_trace* t, const delta_config* c, uint64_t align,
                         delta_program** out) {
  return delta_lower_ex(t, c, align, 0, out);
}

delta_status delta_lower_ex(const delta_trace* t, const delta_config* c, uint64_t align,
                            uint32_t flags, delta_program** out) {
  return guard([&] {
    auto* p = new delta_program;
    try {
      p->p = delta_rt::lower_plan(t->t, to_cfg(c), align, flags);
      p->plan.r = p->p.plan;
      fill(&p->plan);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

delta_status delta_program_info_get(const delta_program* p, delta_program_info* info) {
  return guard([&] {
    info->arena_bytes = p->p.arena_bytes;
    info->pool_peak_bytes = p->p.pool_peak;
    info->host_bytes = p->p.host_bytes;
    info->n_actions = p->p.actions.size();
    info->n_inputs = p->p.inputs.size();
    info->n_events = p->p.n_events;
  });
}

const delta_action* delta_program_actions(const delta_program* p, uint64_t* n) {
  if (n) *n = p->p.actions.size();
  return p->p.actions.data();
}

const uint64_t* delta_program_inputs(const delta_program* p, uint64_t* n) {
  if (n) *n = p->p.inputs.size();
  return p->p.inputs.data();
}

const delta_result* delta_program_plan(const delta_program* p) { return &p->plan; }
void delta_program_free(delta_program* p) { delete p; }

}  // extern "C"
