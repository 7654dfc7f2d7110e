/* delta-b200 C ABI — the step executor (the reference's training-step
 * executor, src/engine.cpp:84-121 Engine::run, made real).
 *
 * delta_rt replays a lowered plan (delta_program, delta.h) on the GPU: the
 * compute stream runs every node's recipe (a short list of kernel ops), the
 * two copy-engine streams run the swap engine's offloads and reloads, and the
 * program's events order them.  Arena pointers in a recipe are symbolic (the
 * node's output slot, its i-th input slot), so one recipe table serves every
 * plan of the same graph: Compute and Recompute of a node run the SAME ops
 * (a recompute skips the ops flagged first-production-only, e.g. BatchNorm
 * statistics, whose saved values it reuses) and reproduce the retained
 * tensor bit for bit.
 *
 * A DELTA_K_HOST op calls a registered host callback, which enqueues work on
 * the stream it is given and may return a device pointer later ops of the
 * recipe read as a scratch operand: the plug-in point for ops a caller brings
 * itself.  The built-in ResNet recipes use none (every op of the step is one
 * of this library's kernels).
 * Everything is asynchronous on the caller's stream, so a whole step can be
 * captured into one CUDA graph.  Errors are delta_status (delta.h).
 */
#ifndef DELTA_DELTA_RT_H_
#define DELTA_DELTA_RT_H_

#include <stdint.h>

#include "delta/delta.h"
#include "delta/delta_kernels.h"
#include "delta/delta_xformer.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- operand references ---- */
enum {
  DELTA_REF_PTR = 0,     /* absolute device pointer `ptr` (0 = null)          */
  DELTA_REF_OUT = 1,     /* the node's output slot in the arena               */
  DELTA_REF_IN = 2,      /* the node's `index`-th input (parent) slot         */
  DELTA_REF_SCRATCH = 3  /* pointer returned by the recipe's `index`-th HOST op */
};
typedef struct delta_ref {
  uint32_t kind, index;
  uint64_t ptr;
} delta_ref;

/* ---- kernel ops (argument use per kind; r = refs, i = ints, f = floats) ----
 *  COPY            r0 dst, r1 src, i0 bytes                      (D2D copy)
 *  CONV            conv, r0 x, r1 y, r2 stats (nullable)          (conv_fwd)
 *  CONV_EX         conv, r0 x, r1 y, r2 stats, i0 epi mode, i1 pool_hw,
 *                  i2 add_stride2, r3 add, r4 add_mask, r5 out_mask, r6 xc,
 *                  r7 mean, r8 invstd, r9 gamma, r10 beta      (fused epilogues)
 *  BN_STATS        r0 x, i0 M, i1 C, r1 ws, r2 mean, r3 invstd, r4 run_mean,
 *                  r5 run_var, f0 eps, f1 momentum
 *  BN_STATS_PARTS  r0 partials, i0 M, i1 C, i2 rows_per_part, r2..r5, f0, f1
 *  BN_APPLY        i0 mode, r0 x, r1 res, r2 y, i1 M, i2 C, r3..r10 mean,
 *                  invstd, gamma, beta, mean2, invstd2, gamma2, beta2
 *  BN_BWD          r0 up, i0 pool_hw, r1 mask, r2 x, r3 dx, i1 M, i2 C, r4 mean,
 *                  r5 invstd, r6 gamma, r7 dgamma, r8 dbeta, r9 ws
 *  BN_BWD_PARTS    r0 partials, r1 g, r2 x, r3 dx, i1 M, i2 C, r4 mean,
 *                  r5 invstd, r6 gamma, r7 dgamma, r8 dbeta
 *  ADD_GRAD        r0 a, r1 up, i0 pool_hw, r2 up_mask, r3 out_mask, r4 out,
 *                  i1 M, i2 C
 *  MAXPOOL_FWD     r0 x, r1 y, i0 N, i1 H, i2 W, i3 C
 *  MAXPOOL_BWD     r0 dy, r1 x, r2 dx, i0 N, i1 H, i2 W, i3 C, r3 ws
 *  AVGPOOL         r0 x, r1 y, i0 N, i1 HW, i2 C
 *  SOFTMAX_XENT    r0 logits, r1 labels, r2 loss, r3 dlogits, r4 row_ws, i0 N, i1 K
 *  HOST            i0 host op id (passed to the host callback)
 *  WGRAD           conv = a delta_wgrad*, r0 dy, r1 x, r2 dw (fp32 KRSC), r3 ws
 *  XENT_HEAD       r0 logits (bf16 [N][i2]), r1 bias, r2 labels, r3 loss,
 *                  r4 dlogits (fp32 [N][i1]), r5 dlogits (bf16 [N][i2]),
 *                  r6 dbias, r7 row_ws, i0 N, i1 K, i2 ld  (softmax_xent_head)
 *  CONV_EX with i0 = DELTA_EPI_SCATTER2: i3 = the parity class (2a + b)
 * transformer ops (delta_xformer.h; rng = device {seed, step}):
 *  LAYERNORM       r0 x, r1 y, r2 mean, r3 rstd, r4 gamma, r5 beta, i0 rows, i1 H, f0 eps
 *  LAYERNORM_BWD   r0 dy, r1 x, r2 dres, r3 dx, r4 mean, r5 rstd, r6 gamma, r7 dgamma,
 *                  r8 dbeta, r9 ws, i0 rows, i1 H
 *  GELU            r0 x, r1 y, i0 n
 *  ADD_DROPOUT     r0 a, r1 b, r2 y, r3 rng, i0 n, i1 tag, f0 p
 *  DROPOUT_BWD     r0 dy, r1 dx, r2 rng, i0 n, i1 tag, f0 p
 *  COLSUM          r0 x, r1 sel, r2 out, r3 ws, i0 rows, i1 cols, i2 sel_val, i3 accumulate
 *  EMBED           r0 ids, r1 types, r2 word, r3 pos, r4 type, r5 y, r6 rng, i0 B, i1 S,
 *                  i2 H, i3 tag, f0 p
 *  EMBED_GRADS     r0 dsum, r1 csr, r2 types, r3 dword, r4 dpos, r5 dtype, r6 ws, i0 B,
 *                  i1 S, i2 H, i3 vocab | n_types << 32
 *  SPAN_HEAD       r0 h, r1 w, r2 bias, r3 label, r4 logits, r5 dlogits, r6 row_loss,
 *                  r7 loss, i0 B, i1 S, i2 H
 *  SPAN_HEAD_BWD   r0 h, r1 dlogits, r2 w, r3 dh, r4 dw, r5 dbias, r6 ws, i0 T, i1 H
 *  ATTN            r0 qkv, r1 out, r2 lse, r3 rng, i0 B, i1 S, i2 heads, i3 tag, f0 p
 *  ATTN_BWD        r0 qkv, r1 out, r2 dout, r3 lse, r4 D, r5 dqkv, r6 rng, r7 dbias
 *                  (optional), r8 ws, i0 B, i1 S, i2 heads, i3 tag, f0 p
 *  STATS_SUM       r0 partials, r1 out, i0 C, i1 accumulate  (delta_stats_col_sum)
 *  LAYERNORM_BWD_DROP  as LAYERNORM_BWD, + r10 dxd, r11 dbias, r12 rng, i2 tag, f0 p
 *                  (delta_layernorm_bwd_drop)
 *  PARTS_MERGE     r0 ws, r1 out, i0 parts, i1 cols  (delta_parts_merge)
 */
enum {
  DELTA_K_COPY = 1,
  DELTA_K_CONV = 2,
  DELTA_K_CONV_EX = 3,
  DELTA_K_BN_STATS = 4,
  DELTA_K_BN_STATS_PARTS = 5,
  DELTA_K_BN_APPLY = 6,
  DELTA_K_BN_BWD = 7,
  DELTA_K_BN_BWD_PARTS = 8,
  DELTA_K_ADD_GRAD = 9,
  DELTA_K_MAXPOOL_FWD = 10,
  DELTA_K_MAXPOOL_BWD = 11,
  DELTA_K_AVGPOOL = 12,
  DELTA_K_SOFTMAX_XENT = 13,
  DELTA_K_HOST = 14,
  DELTA_K_WGRAD = 15,
  DELTA_K_XENT_HEAD = 16,
  DELTA_K_LAYERNORM = 17,
  DELTA_K_LAYERNORM_BWD = 18,
  DELTA_K_GELU = 19,
  DELTA_K_ADD_DROPOUT = 20,
  DELTA_K_DROPOUT_BWD = 21,
  DELTA_K_COLSUM = 22,
  DELTA_K_EMBED = 23,
  DELTA_K_EMBED_GRADS = 24,
  DELTA_K_SPAN_HEAD = 25,
  DELTA_K_SPAN_HEAD_BWD = 26,
  DELTA_K_ATTN = 27,
  DELTA_K_ATTN_BWD = 28,
  DELTA_K_STATS_SUM = 29,
  DELTA_K_LAYERNORM_BWD_DROP = 30,
  DELTA_K_PARTS_MERGE = 31
};
enum {
  DELTA_KOP_FIRST_ONLY = 1,     /* skipped when the node is recomputed        */
  DELTA_KOP_RECOMPUTE_ONLY = 2, /* run only when the node is recomputed       */
  DELTA_KOP_SIDE = 4,           /* with DELTA_SIDE_STREAM=1: run on the side
                                   compute stream, concurrent with the node's
                                   other ops, joined at the node's end        */
  DELTA_KOP_SIDE_ALWAYS = 8     /* on the side stream whatever DELTA_SIDE_STREAM
                                   says (an op placed there to fill another
                                   kernel's idle SMs), joined the same way   */
};

typedef struct delta_kop {
  uint32_t kind, flags;
  delta_conv* conv;
  int64_t i[4];
  float f[2];
  uint32_t pad;
  delta_ref r[14];
} delta_kop;

/* node -> its ops: kops[first .. first + count) */
typedef struct delta_recipe {
  uint64_t node;
  uint32_t first, count;
} delta_recipe;

/* host callback: enqueue library work for HOST op `host_op` of node `node`
 * on `stream`; `ins` = the node's input slot pointers.  Return a device
 * pointer (readable by the recipe's later ops as SCRATCH) or 0; set *status
 * nonzero to fail the step. */
typedef uint64_t (*delta_host_fn)(void* ctx, uint64_t node, int64_t host_op, uint64_t out,
                                  const uint64_t* ins, uint32_t n_ins, int32_t recompute,
                                  void* stream, int32_t* status);
/* per-action observer (tests, probes): called after an action is enqueued */
typedef void (*delta_action_fn)(void* ctx, uint64_t action, uint64_t node, uint64_t out,
                                void* stream);

typedef struct delta_rt delta_rt;

/* Arena: `arena` borrowed (caller-owned device memory of >= arena_bytes), or
 * NULL to allocate.  Pinned host slab of host_bytes and two high-priority
 * copy-engine streams (D2H, H2D) are owned. */
delta_status delta_rt_create(void* arena, uint64_t arena_bytes, uint64_t host_bytes,
                             delta_rt** out);
void* delta_rt_arena(const delta_rt* rt);
void* delta_rt_host_slab(const delta_rt* rt);
void* delta_rt_copy_stream(const delta_rt* rt, int32_t which); /* 1 D2H, 2 H2D */
/* Bind a program and the recipe table (copied; nodes without a recipe may
 * not be computed).  The program must fit the arena and slab. */
delta_status delta_rt_bind(delta_rt* rt, const delta_program* prog, const delta_kop* kops,
                           uint64_t n_kops, const delta_recipe* recipes, uint64_t n_recipes);
delta_status delta_rt_set_callbacks(delta_rt* rt, delta_host_fn host, delta_action_fn after,
                                    void* ctx);
/* Ready events for overlapping work with the step (data-parallel gradient
 * buckets): event i is recorded on the compute stream right after the
 * compute action of nodes[i] in every step; delta_rt_wait_ready makes
 * `stream` (e.g. a communication stream) wait for it.  Replaces any earlier
 * set. */
delta_status delta_rt_set_ready_nodes(delta_rt* rt, const uint64_t* nodes, uint32_t n);
delta_status delta_rt_wait_ready(delta_rt* rt, void* stream, uint32_t i);
/* Issue one step on `stream` (the compute stream); copy streams are joined
 * back into it at the end. */
delta_status delta_rt_step(delta_rt* rt, void* stream);
/* One step with every compute/recompute/offload/reload action bracketed by
 * timing events on its own stream; synchronizes, then writes per-action
 * start/end in ms from the step start (NaN for other actions).  The compute
 * stream is held by a ~50 ms spin kernel while the step is enqueued, so the
 * events time device execution, not host enqueue latency. */
delta_status delta_rt_step_timed(delta_rt* rt, void* stream, float* start_ms, float* end_ms,
                                 uint64_t n_actions);
/* One step with a DEVICE-side action log: every compute/recompute/offload/
 * reload action is bracketed on its own stream by a one-thread stamp kernel
 * that appends {%globaltimer ns, arrival index, action*2 + (0 head|1 tail),
 * node << 8 | action op} (4 x uint64) to a device log when the stream reaches
 * it.  Synchronizes and copies the log (arrival order) into `records`
 * (capacity `cap` records); *n_records = records written.  This is the
 * observed record of what the GPU ran and when (executed-timeline twin of
 * ref Timeline, include/deltasim/engine.hpp:44-70). */
delta_status delta_rt_step_observed(delta_rt* rt, void* stream, uint64_t* records, uint64_t cap,
                                    uint64_t* n_records);
/* GPU cost model (ref OpNode::compute_cost_us, trace.hpp:17): `iters` timed
 * steps; per node, the median over steps of its first compute action, in
 * whole microseconds (ceil, >= 1), written to cost_us[node index in the
 * program's trace order] for nodes with a compute action. */
delta_status delta_rt_measure_costs(delta_rt* rt, void* stream, uint32_t iters,
                                    uint64_t* cost_us, uint64_t n_nodes);
void delta_rt_destroy(delta_rt* rt);

#ifdef __cplusplus
}
#endif
#endif /* DELTA_DELTA_RT_H_ */
