// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim around the UNMODIFIED reference simulator
// (/root/reference/proj/src/*.cpp, compiled with -Ddeltasim=deltasim_ref by
// oracle/Makefile into oracle/_ref/libdeltaref.so).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// load it, as the checker and as the timed CPU baseline.
//
// Every entry takes the trace as canonical JSON (parse_trace,
// src/trace.cpp:211) and a flat config mirroring EngineConfig
// (include/deltasim/engine.hpp:26-42) and returns a malloc'd JSON string.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include <nlohmann/json.hpp>

#include "deltasim/engine.hpp"
#include "deltasim/metrics.hpp"
#include "deltasim/oracle.hpp"
#include "deltasim/trace.hpp"

using namespace deltasim;
using json = nlohmann::ordered_json;

extern "C" {

typedef struct {
  uint64_t budget;
  uint32_t heuristic;  // 0 base 1 lru 2 greedy
  uint32_t policy;     // 0 delta 1 recompute-only 2 offload-only 3 baseline
  uint64_t bw_num, bw_den, eff_num, eff_den;
  uint32_t swap_mode;  // 0 one-way 1 round-trip
  uint32_t guard;      // 0 and 1 paper-or
  uint64_t wm_num, wm_den, prefetch_limit;
  uint32_t prefetch_enabled, overlap_enabled;
  const uint64_t* scripted_nodes;
  const uint32_t* scripted_actions;
  uint64_t n_scripted;
} dref_config;

}  // extern "C"

namespace {

EngineConfig to_cfg(const dref_config* c) {
  EngineConfig cfg;
  cfg.budget = c->budget;
  cfg.heuristic = static_cast<Heuristic>(c->heuristic);
  cfg.policy_mode = static_cast<PolicyMode>(c->policy);
  cfg.cost_model.bandwidth_bytes_per_us = {c->bw_num, c->bw_den};
  cfg.cost_model.effective_fraction = {c->eff_num, c->eff_den};
  cfg.cost_model.swap_cost_mode = static_cast<SwapCostMode>(c->swap_mode);
  cfg.watermark_fraction = {c->wm_num, c->wm_den};
  cfg.prefetch_limit = c->prefetch_limit;
  cfg.prefetch_enabled = c->prefetch_enabled != 0;
  cfg.overlap_enabled = c->overlap_enabled != 0;
  cfg.prefetch_guard = static_cast<PrefetchGuard>(c->guard);
  for (uint64_t i = 0; i < c->n_scripted; ++i) {
    cfg.scripted_decisions.emplace_back(
        c->scripted_nodes[i], static_cast<ReleaseAction>(c->scripted_actions[i]));
  }
  return cfg;
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.data(), s.size() + 1);
  return p;
}

json result_json(const RunResult& r) {
  json j;
  j["ok"] = true;
  j["completed"] = r.completed();
  if (r.infeasible) {
    j["infeasible"] = {r.infeasible->node, r.infeasible->deficit};
  } else {
    j["infeasible"] = nullptr;
  }
  j["peak_bytes"] = r.peak_bytes;
  j["wall_time_us"] = r.wall_time_us;
  j["total_stall_us"] = r.total_stall_us;
  j["copy_busy_us"] = r.copy_busy_us;
  j["copy_stall_us"] = r.copy_stall_us;
  j["counts"] = {r.counts.evict,         r.counts.offload,
                 r.counts.reload,        r.counts.recompute,
                 r.counts.prefetch_reload, r.counts.recompute_of_swapout};
  json dec = json::array();
  for (auto& [n, a] : r.decisions) dec.push_back({n, static_cast<int>(a)});
  j["decisions"] = std::move(dec);
  json ev = json::array();
  for (const TimelineEvent& e : r.timeline.events) {
    ev.push_back({e.ts, static_cast<int>(e.stream), static_cast<int>(e.kind),
                  e.node, e.duration, e.bytes, static_cast<int>(e.phase),
                  e.prefetch ? 1 : 0, e.burst});
  }
  j["events"] = std::move(ev);
  j["chrome"] = timeline_to_chrome_trace(r.timeline);
  return j;
}

template <class F>
char* guarded(F&& f) {
  try {
    return dup(f());
  } catch (const std::exception& e) {
    json j;
    j["ok"] = false;
    j["what"] = e.what();
    return dup(j.dump());
  }
}

}  // namespace

extern "C" {

char* dref_run(const char* trace_json, const dref_config* c, int baseline) {
  return guarded([&] {
    Trace t = parse_trace(trace_json);
    EngineConfig cfg = to_cfg(c);
    RunResult r = baseline ? run_unconstrained_baseline(t, cfg)
                           : run_iteration(t, cfg);
    return result_json(r).dump();
  });
}

char* dref_report(const char* trace_json, const dref_config* c) {
  return guarded([&] {
    Trace t = parse_trace(trace_json);
    EngineConfig cfg = to_cfg(c);
    RunResult base = run_unconstrained_baseline(t, cfg);
    RunResult r = run_iteration(t, cfg);
    return report_to_json(summarize(r, base));
  });
}

// run_comparison + comparison_to_csv / _json of the reference (json: 0 / 1)
char* dref_comparison(const char* trace_json, const dref_config* c, const uint64_t* budgets,
                      uint64_t nb, const uint32_t* policies, uint64_t np,
                      const uint32_t* heuristics, uint64_t nh, int json_out) {
  return guarded([&] {
    Trace t = parse_trace(trace_json);
    std::vector<Bytes> b(budgets, budgets + nb);
    std::vector<PolicyMode> p;
    for (uint64_t i = 0; i < np; ++i) p.push_back(static_cast<PolicyMode>(policies[i]));
    std::vector<Heuristic> h;
    for (uint64_t i = 0; i < nh; ++i) h.push_back(static_cast<Heuristic>(heuristics[i]));
    ComparisonReport rep = run_comparison(t, b, p, h, to_cfg(c));
    return json_out ? comparison_to_json(rep) : comparison_to_csv(rep);
  });
}

// Median-free mean ns per run_iteration over `iters` calls (trace parsed once).
double dref_time_run(const char* trace_json, const dref_config* c, int iters) {
  try {
    Trace t = parse_trace(trace_json);
    EngineConfig cfg = to_cfg(c);
    volatile uint64_t sink = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) sink += run_iteration(t, cfg).wall_time_us;
    auto t1 = std::chrono::steady_clock::now();
    (void)sink;
    return std::chrono::duration<double, std::nano>(t1 - t0).count() / iters;
  } catch (...) {
    return -1.0;
  }
}

char* dref_replay_check(const char* trace_json, const dref_config* c,
                        const char* chrome_json) {
  return guarded([&] {
    Trace t = parse_trace(trace_json);
    EngineConfig cfg = to_cfg(c);
    Timeline tl = timeline_from_chrome_trace(chrome_json);
    json out = json::array();
    for (const auto& v : oracle::replay_check(tl, t, cfg)) {
      out.push_back({oracle::to_string(v.code), v.ts, v.node, v.detail});
    }
    return out.dump();
  });
}

uint64_t dref_brute_force(const char* trace_json, uint64_t max_nodes) {
  try {
    return oracle::brute_force_min_peak(parse_trace(trace_json), max_nodes);
  } catch (...) {
    return ~uint64_t{0};
  }
}

// kind: 0 linear(n,100,5) 1 resnet(n,1<<20) 2 transformer(n,256<<10)
char* dref_generate(int kind, uint64_t n, uint64_t seed) {
  return guarded([&] {
    Trace t = kind == 0   ? gen_linear_chain(n, 100, 5, seed)
              : kind == 1 ? gen_resnet_like(n, 1 << 20, seed)
                          : gen_transformer_like(n, 256 << 10, seed);
    return serialize_trace(t);
  });
}

void dref_free(char* p) { std::free(p); }

}  // extern "C"
