/* delta-b200 C ABI.
 *
 * A thin extern "C" layer over libdelta: plain pointers and sizes, integer
 * status codes, a thread-local last-error string, never an exception across
 * the boundary.  Each entry cites the reference C++ interface it replaces
 * (paths under /root/reference/proj/).  INTEGRATION.md shows the ctypes
 * binding a maintainer of the reference would add.
 *
 * Handles are caller-owned and not thread-safe; independent handles may be
 * used from different threads (the planner has no global mutable state).
 */
#ifndef DELTA_DELTA_H_
#define DELTA_DELTA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception class
 *      (include/deltasim/types.hpp:35-65) plus runtime failures ---- */
typedef int32_t delta_status;
enum {
  DELTA_OK = 0,
  DELTA_E_SCHEMA = 1,        /* SchemaError        */
  DELTA_E_VALIDATION = 2,    /* ValidationErrorEx  */
  DELTA_E_ARGUMENT = 3,      /* ArgumentError      */
  DELTA_E_STATE = 4,         /* StateError         */
  DELTA_E_ILLEGAL = 5,       /* IllegalTransition  */
  DELTA_E_UNRECOVERABLE = 6, /* UnrecoverableError */
  DELTA_E_MISMATCHED = 7,    /* MismatchedTrace    */
  DELTA_E_TOO_LARGE = 8,     /* TooLarge           */
  DELTA_E_IO = 9,            /* IoError            */
  DELTA_E_INTERNAL = 10,     /* InternalError      */
  DELTA_E_CUDA = 20,         /* CUDA runtime / driver failure */
  DELTA_E_UNSUPPORTED = 21,  /* shape or device the kernels do not cover */
  DELTA_E_UNKNOWN = 99
};
/* Infeasibility is a VALUE, not an error (ref src/engine.cpp:104-106):
 * delta_plan returns DELTA_OK and delta_summary.infeasible = 1. */

const char* delta_last_error(void); /* thread-local, valid until next call */
void delta_free(void* p);           /* frees strings returned by this API   */
const char* delta_version(void);

/* ---- tensor registration (ref include/deltasim/trace.hpp:14-41) ---- */
typedef struct delta_trace delta_trace;

enum { DELTA_NODE_UNCOMPUTABLE = 1, DELTA_NODE_EVICT_PINNED = 2,
       DELTA_NODE_OFFLOAD_PINNED = 4 };
enum { DELTA_PHASE_FORWARD = 0, DELTA_PHASE_BACKWARD = 1 };
enum { DELTA_ACCESS_PRODUCE = 0, DELTA_ACCESS_USE = 1 };

delta_status delta_trace_new(const char* name, delta_trace** out);
/* OpNode{id,name,compute_cost_us,output_bytes,parents,flags} */
delta_status delta_trace_add_node(delta_trace* t, uint64_t id, const char* name,
                                  uint64_t compute_cost_us, uint64_t output_bytes,
                                  const uint64_t* parents, uint64_t n_parents,
                                  uint32_t flags);
/* AccessEvent{node,phase,kind} */
delta_status delta_trace_add_event(delta_trace* t, uint64_t node, uint32_t phase,
                                   uint32_t kind);
/* Cost-model update: overwrite OpNode::compute_cost_us of node `id`. */
delta_status delta_trace_set_cost(delta_trace* t, uint64_t id, uint64_t cost_us);
/* parse_trace (src/trace.cpp:211) / serialize_trace (src/trace.cpp:288) */
delta_status delta_trace_parse(const char* json, uint64_t len, delta_trace** out);
delta_status delta_trace_serialize(const delta_trace* t, char** out, uint64_t* len);
/* validate_trace (src/trace.cpp:58): counts of Error / Warning findings and
 * the first error message (delta_free it; NULL when none). */
delta_status delta_trace_validate(const delta_trace* t, uint32_t* n_errors,
                                  uint32_t* n_warnings, char** first_error);
uint64_t delta_trace_num_nodes(const delta_trace* t);
uint64_t delta_trace_num_events(const delta_trace* t);
void delta_trace_free(delta_trace* t);

/* ---- memory-budget config (ref include/deltasim/engine.hpp:26-42,
 *      include/deltasim/policy.hpp:18-26) ---- */
enum { DELTA_HEUR_BASE = 0, DELTA_HEUR_LRU = 1, DELTA_HEUR_GREEDY = 2 };
enum { DELTA_POLICY_DELTA = 0, DELTA_POLICY_RECOMPUTE_ONLY = 1,
       DELTA_POLICY_OFFLOAD_ONLY = 2, DELTA_POLICY_BASELINE = 3 };
enum { DELTA_ACTION_EVICT = 0, DELTA_ACTION_OFFLOAD = 1 };

typedef struct delta_config {
  uint64_t budget;
  uint32_t heuristic;       /* DELTA_HEUR_*   */
  uint32_t policy_mode;     /* DELTA_POLICY_* */
  uint64_t bw_num, bw_den;  /* bandwidth_bytes_per_us as an exact fraction */
  uint64_t eff_num, eff_den;/* effective_fraction */
  uint32_t swap_cost_mode;  /* 0 one-way, 1 round-trip */
  uint32_t prefetch_guard;  /* 0 And, 1 PaperOr */
  uint64_t watermark_num, watermark_den;
  uint64_t prefetch_limit;
  uint32_t prefetch_enabled;
  uint32_t overlap_enabled;
  /* scripted_decisions test hook (engine.hpp:37-39) */
  const uint64_t* scripted_nodes;
  const uint32_t* scripted_actions;
  uint64_t n_scripted;
} delta_config;

/* The reference defaults: 64e9 B/s x 0.35, watermark 3/4, prefetch 2, And. */
void delta_config_default(delta_config* c);

/* ---- planning: run_iteration (src/engine.cpp:627) ---- */
typedef struct delta_result delta_result;

typedef struct delta_event { /* TimelineEvent (engine.hpp:56-66) */
  uint64_t ts, node, duration, bytes;
  uint32_t burst;
  uint8_t stream;   /* 0 compute, 1 copy */
  uint8_t kind;     /* EventKind: Compute Offload Reload Recompute Stall Evict Use Free */
  uint8_t phase;    /* 0 F, 1 B */
  uint8_t prefetch;
} delta_event;

typedef struct delta_decision { uint64_t node; uint32_t action; uint32_t pad; } delta_decision;

typedef struct delta_summary { /* RunResult scalars (engine.hpp:97-113) */
  uint64_t peak_bytes, wall_time_us, total_stall_us, copy_busy_us, copy_stall_us;
  uint64_t evict, offload, reload, recompute, prefetch_reload, recompute_of_swapout;
  uint32_t infeasible, pad;
  uint64_t infeasible_node, infeasible_deficit;
  uint64_t n_events, n_decisions;
} delta_summary;

delta_status delta_plan(const delta_trace* t, const delta_config* c, delta_result** out);
/* run_unconstrained_baseline (src/engine.cpp:635) */
delta_status delta_plan_baseline(const delta_trace* t, const delta_config* c,
                                 delta_result** out);
delta_status delta_result_summary(const delta_result* r, delta_summary* s);
const delta_event* delta_result_events(const delta_result* r, uint64_t* n);
const delta_decision* delta_result_decisions(const delta_result* r, uint64_t* n);
/* report_to_json(summarize(run, baseline)) (src/metrics.cpp:132,159) */
delta_status delta_report_json(const delta_result* run, const delta_result* baseline,
                               char** out, uint64_t* len);
/* timeline_to_chrome_trace (src/metrics.cpp:255) */
delta_status delta_chrome_trace(const delta_result* r, char** out, uint64_t* len);
/* timeline_to_chrome_trace of a caller-built event array (e.g. the executed
 * GPU timeline: the plan's events re-stamped with measured device times) */
delta_status delta_chrome_trace_events(const delta_event* ev, uint64_t n, char** out,
                                       uint64_t* len);
void delta_result_free(delta_result* r);

/* run_comparison (src/engine.cpp:646-671): every budget x policy x heuristic
 * cell planned on `t` with the other fields of `base`, rendered as the
 * reference's comparison CSV (json = 0, src/metrics.cpp:314-328) or JSON
 * (json = 1, :330-348); delta_free the string. */
delta_status delta_comparison(const delta_trace* t, const delta_config* base,
                              const uint64_t* budgets, uint64_t n_budgets,
                              const uint32_t* policies, uint64_t n_policies,
                              const uint32_t* heuristics, uint64_t n_heuristics, int32_t json,
                              char** out, uint64_t* len);

/* CPU planner timing: mean ns per run_iteration over `iters` calls. */
delta_status delta_plan_time_ns(const delta_trace* t, const delta_config* c,
                                uint32_t iters, double* ns_per_plan);

/* Policy free functions (src/policy.cpp:58-73), for known-answer tests. */
delta_status delta_transfer_time_us(uint64_t bytes, const delta_config* c, uint64_t* us);

/* ---- lowering a plan onto the HBM arena (B200 runtime, csrc/rt) ----
 * Replays the planner's exact pool alloc/free sequence, assigns every
 * allocation an arena offset (offline best-fit over known lifetimes) and
 * emits a 3-stream action program with the cross-stream event edges that
 * make slot reuse and copies safe. */
typedef struct delta_program delta_program;

enum { DELTA_STREAM_COMPUTE = 0, DELTA_STREAM_D2H = 1, DELTA_STREAM_H2D = 2 };
enum {
  DELTA_ACT_COMPUTE = 0,   /* run node's op (forward or backward) -> out slot */
  DELTA_ACT_RECOMPUTE = 1, /* re-run node's forward op -> out slot           */
  DELTA_ACT_OFFLOAD = 2,   /* D2H slot -> host slab                          */
  DELTA_ACT_RELOAD = 3,    /* H2D host slab -> slot                          */
  DELTA_ACT_RECORD = 4,    /* record event `event` on `stream`               */
  DELTA_ACT_WAIT = 5       /* make `stream` wait on event `event`            */
};

typedef struct delta_action {
  uint32_t op, stream;
  uint64_t node;
  uint64_t offset;       /* arena offset of the node's buffer              */
  uint64_t bytes;
  uint64_t host_offset;  /* host slab offset (OFFLOAD / RELOAD)             */
  uint32_t event;        /* RECORD / WAIT                                   */
  uint32_t n_inputs;     /* COMPUTE / RECOMPUTE: parents, in trace order   */
  uint64_t inputs_at;    /* index into the program's input-offset array     */
  uint64_t plan_event;   /* timeline index this action lowers               */
} delta_action;

typedef struct delta_program_info {
  uint64_t arena_bytes;       /* footprint of the offset assignment          */
  uint64_t pool_peak_bytes;   /* planner pool high-watermark (byte budget)   */
  uint64_t host_bytes;        /* pinned slab bytes                           */
  uint64_t n_actions, n_inputs, n_events;
} delta_program_info;

delta_status delta_lower(const delta_trace* t, const delta_config* c,
                         uint64_t align, delta_program** out);
/* flags for delta_lower_ex.  Default (0): offloads AND reloads on one copy
 * stream (DELTA_STREAM_D2H) in plan order — the reference's single copy
 * stream (include/deltasim/device.hpp:45-74), so the executed timeline is
 * checkable by its replay_check as is.  DUPLEX: reloads on DELTA_STREAM_H2D,
 * concurrent with offloads (both PCIe directions). */
enum { DELTA_LOWER_DUPLEX_COPIES = 1 };
delta_status delta_lower_ex(const delta_trace* t, const delta_config* c, uint64_t align,
                            uint32_t flags, delta_program** out);
delta_status delta_program_info_get(const delta_program* p, delta_program_info* info);
const delta_action* delta_program_actions(const delta_program* p, uint64_t* n);
const uint64_t* delta_program_inputs(const delta_program* p, uint64_t* n);
/* The plan the program lowers (for parity checks against the oracle). */
const delta_result* delta_program_plan(const delta_program* p);
void delta_program_free(delta_program* p);

#ifdef __cplusplus
}
#endif
#endif /* DELTA_DELTA_H_ */
