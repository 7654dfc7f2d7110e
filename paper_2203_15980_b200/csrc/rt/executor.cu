// The step executor (include/delta/delta_rt.h): replays a lowered DELTA plan
// on the B200.  The reference's Engine::run (src/engine.cpp:84-121) walks the
// schedule on a logical clock; here the planner has already fixed every
// decision and the lowering (rt/lower.cpp) every arena offset and event edge,
// so a step is a straight walk over the action list:
//   COMPUTE / RECOMPUTE  -> the node's recipe ops on the compute stream
//   OFFLOAD / RELOAD     -> cudaMemcpyAsync on the D2H / H2D copy engines
//   RECORD / WAIT        -> cudaEventRecord / cudaStreamWaitEvent
// Nothing here allocates or synchronizes (except the timed variants), so a
// step can be captured into a CUDA graph.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "delta/delta_rt.h"
#include "kernels/xformer.hpp"
#include "kernels/kernels.hpp"
#include "rt/handles.hpp"

struct delta_rt {
  void* arena = nullptr;
  bool own_arena = false;
  uint64_t arena_bytes = 0;
  void* host = nullptr;
  uint64_t host_bytes = 0;
  cudaStream_t d2h = nullptr, h2d = nullptr;
  std::vector<cudaEvent_t> events;
  std::vector<delta_action> actions;
  std::vector<uint64_t> inputs;
  std::vector<delta_kop> kops;
  std::unordered_map<uint64_t, std::pair<uint32_t, uint32_t>> recipe;  // node -> (first, count)
  bool copy_used[3] = {false, false, false};
  cudaEvent_t join[3] = {nullptr, nullptr, nullptr};
  // side compute stream: ops flagged DELTA_KOP_SIDE run there, concurrently
  // with the rest of their node, and are joined back before the node ends
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, side_done = nullptr;
  bool side_enabled = false;  // DELTA_SIDE_STREAM=1 (measured neutral: both chains are
                              // bandwidth-bound full-grid kernels)
  delta_host_fn host_fn = nullptr;
  delta_action_fn after_fn = nullptr;
  void* ctx = nullptr;
  // ready events: recorded on the compute stream right after the compute
  // action of a node (e.g. the last weight gradient of a gradient bucket)
  std::unordered_map<uint64_t, uint32_t> ready_of;
  std::vector<cudaEvent_t> ready;
};

namespace {

// keeps the compute stream busy while the host enqueues a timed step, so the
// timing events measure device execution, not host enqueue latency
__global__ void k_spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

// Device-side action log of an observed step: one record per stamp, written
// by the device when the stream reaches it — {%globaltimer ns, global
// arrival order, action index * 2 + (0 head | 1 tail), node << 8 | op}.
__global__ void k_stamp(unsigned long long* log, unsigned int* count, unsigned int cap,
                        unsigned long long tag, unsigned long long what) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const unsigned int i = atomicAdd(count, 1u);
  if (i < cap) {
    log[4 * size_t(i) + 0] = t;
    log[4 * size_t(i) + 1] = i;
    log[4 * size_t(i) + 2] = tag;
    log[4 * size_t(i) + 3] = what;
  }
}

struct StampLog {
  unsigned long long* log = nullptr;
  unsigned int* count = nullptr;
  unsigned int cap = 0;
};

delta_status fail(delta_status code, const std::string& msg) {
  delta_set_error(msg);
  return code;
}
delta_status cuda_fail(cudaError_t e, const char* what) {
  return fail(DELTA_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define RT_CUDA(expr)                                  \
  do {                                                 \
    cudaError_t e_ = (expr);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
  } while (0)

struct Frame {  // operand resolution context of one compute action
  char* arena;
  uint64_t out;
  const uint64_t* in;  // input offsets
  uint32_t n_in;
  uint64_t scratch[8];
};

void* ref(const Frame& f, const delta_ref& r) {
  switch (r.kind) {
    case DELTA_REF_OUT: return f.arena + f.out;
    case DELTA_REF_IN: return r.index < f.n_in ? f.arena + f.in[r.index] : nullptr;
    case DELTA_REF_SCRATCH: return r.index < 8 ? reinterpret_cast<void*>(f.scratch[r.index]) : nullptr;
    default: return reinterpret_cast<void*>(r.ptr);
  }
}
template <class T>
T* rp(const Frame& f, const delta_ref& r) {
  return static_cast<T*>(ref(f, r));
}

delta_status run_kop(delta_rt* rt, const delta_kop& k, Frame& fr, uint64_t node, bool recompute,
                     cudaStream_t st, int& n_host) {
  cudaError_t e = cudaSuccess;
  const auto& r = k.r;
  const auto& i = k.i;
  switch (k.kind) {
    case DELTA_K_COPY:
      e = cudaMemcpyAsync(ref(fr, r[0]), ref(fr, r[1]), size_t(i[0]), cudaMemcpyDeviceToDevice, st);
      break;
    case DELTA_K_CONV:
      if (!k.conv) return fail(DELTA_E_ARGUMENT, "recipe: CONV without a conv handle");
      e = delta_k::conv_forward(k.conv->plan, ref(fr, r[0]), ref(fr, r[1]), rp<float>(fr, r[2]), st);
      break;
    case DELTA_K_CONV_EX: {
      if (!k.conv) return fail(DELTA_E_ARGUMENT, "recipe: CONV_EX without a conv handle");
      delta_k::ConvEpilogue ep{};
      ep.mode = int(i[0]);
      ep.pool_hw = int(i[1]);
      ep.add_stride2 = int(i[2]);
      ep.scatter = int(i[3]);
      ep.add = ref(fr, r[3]);
      ep.add_mask = ref(fr, r[4]);
      ep.out_mask = ref(fr, r[5]);
      ep.xc = ref(fr, r[6]);
      ep.mean = rp<const float>(fr, r[7]);
      ep.invstd = rp<const float>(fr, r[8]);
      ep.gamma = rp<const float>(fr, r[9]);
      ep.beta = rp<const float>(fr, r[10]);
      e = delta_k::conv_forward(k.conv->plan, ref(fr, r[0]), ref(fr, r[1]), rp<float>(fr, r[2]), st,
                                &ep);
      break;
    }
    case DELTA_K_BN_STATS:
      e = delta_k::bn_stats(ref(fr, r[0]), i[0], int(i[1]), rp<float>(fr, r[1]), rp<float>(fr, r[2]),
                            rp<float>(fr, r[3]), k.f[0], rp<float>(fr, r[4]), rp<float>(fr, r[5]),
                            k.f[1], st);
      break;
    case DELTA_K_BN_STATS_PARTS:
      e = delta_k::bn_stats_from_partials(rp<const float>(fr, r[0]), int(i[1]),
                                          rp<float>(fr, r[2]), rp<float>(fr, r[3]), k.f[0],
                                          rp<float>(fr, r[4]), rp<float>(fr, r[5]), k.f[1], st);
      break;
    case DELTA_K_BN_APPLY:
      e = delta_k::bn_apply(int(i[0]), ref(fr, r[0]), ref(fr, r[1]), ref(fr, r[2]), i[1], int(i[2]),
                            rp<const float>(fr, r[3]), rp<const float>(fr, r[4]),
                            rp<const float>(fr, r[5]), rp<const float>(fr, r[6]),
                            rp<const float>(fr, r[7]), rp<const float>(fr, r[8]),
                            rp<const float>(fr, r[9]), rp<const float>(fr, r[10]), st);
      break;
    case DELTA_K_BN_BWD:
      e = delta_k::bn_backward(ref(fr, r[0]), int(i[0]), ref(fr, r[1]), ref(fr, r[2]), ref(fr, r[3]),
                               i[1], int(i[2]), rp<const float>(fr, r[4]),
                               rp<const float>(fr, r[5]), rp<const float>(fr, r[6]),
                               rp<float>(fr, r[7]), rp<float>(fr, r[8]), rp<float>(fr, r[9]), st);
      break;
    case DELTA_K_BN_BWD_PARTS:
      e = delta_k::bn_backward_from_partials(rp<const float>(fr, r[0]), ref(fr, r[1]),
                                             ref(fr, r[2]), ref(fr, r[3]), i[1], int(i[2]),
                                             rp<const float>(fr, r[4]), rp<const float>(fr, r[5]),
                                             rp<const float>(fr, r[6]), rp<float>(fr, r[7]),
                                             rp<float>(fr, r[8]), st);
      break;
    case DELTA_K_ADD_GRAD:
      e = delta_k::add_grad(ref(fr, r[0]), ref(fr, r[1]), int(i[0]), ref(fr, r[2]), ref(fr, r[3]),
                            ref(fr, r[4]), i[1], int(i[2]), st);
      break;
    case DELTA_K_MAXPOOL_FWD:
      e = delta_k::maxpool3x3s2_fwd(ref(fr, r[0]), ref(fr, r[1]), int(i[0]), int(i[1]), int(i[2]),
                                    int(i[3]), st);
      break;
    case DELTA_K_MAXPOOL_BWD:
      e = delta_k::maxpool3x3s2_bwd(ref(fr, r[0]), ref(fr, r[1]), ref(fr, r[2]), int(i[0]),
                                    int(i[1]), int(i[2]), int(i[3]), ref(fr, r[3]), st);
      break;
    case DELTA_K_AVGPOOL:
      e = delta_k::avgpool_fwd(ref(fr, r[0]), ref(fr, r[1]), int(i[0]), int(i[1]), int(i[2]), st);
      break;
    case DELTA_K_SOFTMAX_XENT:
      e = delta_k::softmax_xent(rp<const float>(fr, r[0]), rp<const int64_t>(fr, r[1]),
                                rp<float>(fr, r[2]), rp<float>(fr, r[3]), rp<float>(fr, r[4]),
                                int(i[0]), int(i[1]), st);
      break;
    case DELTA_K_XENT_HEAD:
      e = delta_k::softmax_xent_head(ref(fr, r[0]), int(i[2]), rp<const float>(fr, r[1]),
                                     rp<const int64_t>(fr, r[2]), rp<float>(fr, r[3]),
                                     rp<float>(fr, r[4]), ref(fr, r[5]), rp<float>(fr, r[6]),
                                     rp<float>(fr, r[7]), int(i[0]), int(i[1]), st);
      break;
    case DELTA_K_WGRAD: {
      auto* w = reinterpret_cast<const delta_wgrad*>(k.conv);
      if (!w) return fail(DELTA_E_ARGUMENT, "recipe: WGRAD without a wgrad handle");
      e = delta_k::wgrad(w->plan, ref(fr, r[0]), ref(fr, r[1]), rp<float>(fr, r[2]),
                         rp<float>(fr, r[3]), st);
      break;
    }
    case DELTA_K_LAYERNORM:
      e = delta_k::layernorm_fwd(ref(fr, r[0]), ref(fr, r[1]), rp<float>(fr, r[2]), rp<float>(fr, r[3]),
                                 rp<const float>(fr, r[4]), rp<const float>(fr, r[5]), i[0],
                                 int(i[1]), k.f[0], st);
      break;
    case DELTA_K_LAYERNORM_BWD:
      e = delta_k::layernorm_bwd(ref(fr, r[0]), ref(fr, r[1]), ref(fr, r[2]), ref(fr, r[3]),
                                 rp<const float>(fr, r[4]), rp<const float>(fr, r[5]),
                                 rp<const float>(fr, r[6]), rp<float>(fr, r[7]), rp<float>(fr, r[8]),
                                 rp<float>(fr, r[9]), i[0], int(i[1]), st);
      break;
    case DELTA_K_LAYERNORM_BWD_DROP:
      e = delta_k::layernorm_bwd_drop(
          ref(fr, r[0]), ref(fr, r[1]), ref(fr, r[2]), ref(fr, r[3]), rp<const float>(fr, r[4]),
          rp<const float>(fr, r[5]), rp<const float>(fr, r[6]), rp<float>(fr, r[7]),
          rp<float>(fr, r[8]), rp<float>(fr, r[9]), i[0], int(i[1]), ref(fr, r[10]),
          rp<float>(fr, r[11]), k.f[0], rp<const uint64_t>(fr, r[12]), uint32_t(i[2]), st);
      break;
    case DELTA_K_GELU:
      e = delta_k::gelu_fwd(ref(fr, r[0]), ref(fr, r[1]), i[0], st);
      break;
    case DELTA_K_ADD_DROPOUT:
      e = delta_k::add_dropout(ref(fr, r[0]), ref(fr, r[1]), ref(fr, r[2]), i[0], k.f[0],
                               rp<const uint64_t>(fr, r[3]), uint32_t(i[1]), st);
      break;
    case DELTA_K_DROPOUT_BWD:
      e = delta_k::dropout_bwd(ref(fr, r[0]), ref(fr, r[1]), i[0], k.f[0],
                               rp<const uint64_t>(fr, r[2]), uint32_t(i[1]), st);
      break;
    case DELTA_K_COLSUM:
      e = delta_k::colsum(ref(fr, r[0]), i[0], int(i[1]), rp<const int32_t>(fr, r[1]), int(i[2]),
                          rp<float>(fr, r[2]), rp<float>(fr, r[3]), int(i[3]), st);
      break;
    case DELTA_K_EMBED:
      e = delta_k::embed_fwd(rp<const int32_t>(fr, r[0]), rp<const int32_t>(fr, r[1]), ref(fr, r[2]),
                             ref(fr, r[3]), ref(fr, r[4]), ref(fr, r[5]), int(i[0]), int(i[1]),
                             int(i[2]), k.f[0], rp<const uint64_t>(fr, r[6]), uint32_t(i[3]), st);
      break;
    case DELTA_K_EMBED_GRADS:
      e = delta_k::embed_grads(ref(fr, r[0]), rp<const int32_t>(fr, r[1]), rp<const int32_t>(fr, r[2]),
                               int(i[0]), int(i[1]), int(i[2]), int(i[3] & 0xFFFFFFFF),
                               int(i[3] >> 32), rp<float>(fr, r[3]), rp<float>(fr, r[4]),
                               rp<float>(fr, r[5]), rp<float>(fr, r[6]), st);
      break;
    case DELTA_K_SPAN_HEAD:
      e = delta_k::span_head_fwd(ref(fr, r[0]), rp<const float>(fr, r[1]), rp<const float>(fr, r[2]),
                                 rp<const int32_t>(fr, r[3]), rp<float>(fr, r[4]), rp<float>(fr, r[5]),
                                 rp<float>(fr, r[6]), rp<float>(fr, r[7]), int(i[0]), int(i[1]),
                                 int(i[2]), st);
      break;
    case DELTA_K_SPAN_HEAD_BWD:
      e = delta_k::span_head_bwd(ref(fr, r[0]), rp<const float>(fr, r[1]), rp<const float>(fr, r[2]),
                                 ref(fr, r[3]), rp<float>(fr, r[4]), rp<float>(fr, r[5]),
                                 rp<float>(fr, r[6]), i[0], int(i[1]), st);
      break;
    case DELTA_K_ATTN:
      e = delta_k::attention_fwd(ref(fr, r[0]), ref(fr, r[1]), rp<float>(fr, r[2]), int(i[0]),
                                 int(i[1]), int(i[2]), k.f[0], rp<const uint64_t>(fr, r[3]),
                                 uint32_t(i[3]), st);
      break;
    case DELTA_K_ATTN_BWD:
      e = delta_k::attention_bwd(ref(fr, r[0]), ref(fr, r[1]), ref(fr, r[2]), rp<const float>(fr, r[3]),
                                 rp<float>(fr, r[4]), ref(fr, r[5]), int(i[0]), int(i[1]), int(i[2]),
                                 k.f[0], rp<const uint64_t>(fr, r[6]), uint32_t(i[3]),
                                 rp<float>(fr, r[7]), rp<float>(fr, r[8]), st);
      break;
    case DELTA_K_PARTS_MERGE:
      e = delta_k::merge_parts(rp<const float>(fr, r[0]), int(i[0]), int(i[1]), rp<float>(fr, r[1]), st);
      break;
    case DELTA_K_STATS_SUM:
      e = delta_k::stats_col_sum(rp<const float>(fr, r[0]), int(i[0]), rp<float>(fr, r[1]), int(i[1]),
                                 st);
      break;
    case DELTA_K_HOST: {
      if (!rt->host_fn) return fail(DELTA_E_ARGUMENT, "recipe: HOST op without a host callback");
      std::vector<uint64_t> ins(fr.n_in);
      for (uint32_t j = 0; j < fr.n_in; ++j)
        ins[j] = reinterpret_cast<uint64_t>(fr.arena + fr.in[j]);
      int32_t status = 0;
      const uint64_t p = rt->host_fn(rt->ctx, node, i[0],
                                     reinterpret_cast<uint64_t>(fr.arena + fr.out),
                                     ins.data(), fr.n_in, recompute ? 1 : 0, st, &status);
      if (status != 0)
        return fail(DELTA_E_INTERNAL, "host op " + std::to_string(i[0]) + " of node " +
                                          std::to_string(node) + " failed");
      if (n_host < 8) fr.scratch[n_host] = p;
      ++n_host;
      return DELTA_OK;
    }
    default:
      return fail(DELTA_E_ARGUMENT, "recipe: unknown kernel op " + std::to_string(k.kind));
  }
  if (e != cudaSuccess)
    return cuda_fail(e, ("node " + std::to_string(node) + " op " + std::to_string(k.kind)).c_str());
  return DELTA_OK;
}

delta_status run_node(delta_rt* rt, const delta_action& a, cudaStream_t st) {
  auto it = rt->recipe.find(a.node);
  if (it == rt->recipe.end())
    return fail(DELTA_E_ARGUMENT, "no recipe for node " + std::to_string(a.node));
  Frame fr{};
  fr.arena = static_cast<char*>(rt->arena);
  fr.out = a.offset;
  fr.in = rt->inputs.data() + a.inputs_at;
  fr.n_in = a.n_inputs;
  const bool recompute = a.op == DELTA_ACT_RECOMPUTE;
  int n_host = 0;
  bool forked = false;
  for (uint32_t j = 0; j < it->second.second; ++j) {
    const delta_kop& k = rt->kops[it->second.first + j];
    if (recompute && (k.flags & DELTA_KOP_FIRST_ONLY)) continue;
    if (!recompute && (k.flags & DELTA_KOP_RECOMPUTE_ONLY)) continue;
    cudaStream_t ks = st;
    if (((k.flags & DELTA_KOP_SIDE) && rt->side_enabled) || (k.flags & DELTA_KOP_SIDE_ALWAYS)) {
      if (!forked) {  // the side stream starts after everything before this node
        RT_CUDA(cudaEventRecord(rt->fork, st));
        RT_CUDA(cudaStreamWaitEvent(rt->side, rt->fork, 0));
        forked = true;
      }
      ks = rt->side;
    }
    delta_status s = run_kop(rt, k, fr, a.node, recompute, ks, n_host);
    if (s) return s;
  }
  if (forked) {  // join: the node (and its arena reads) ends when both are done
    RT_CUDA(cudaEventRecord(rt->side_done, rt->side));
    RT_CUDA(cudaStreamWaitEvent(st, rt->side_done, 0));
  }
  return DELTA_OK;
}

// One pass over the actions.  `t0/t1` (optional) = per-action timing event
// pairs recorded around compute and copy actions on their own stream;
// `stamps` (optional) = device-logged head/tail stamps of the same actions.
delta_status issue(delta_rt* rt, cudaStream_t cs, cudaEvent_t* t0, cudaEvent_t* t1,
                   const StampLog* stamps = nullptr) {
  cudaStream_t streams[3] = {cs, rt->d2h, rt->h2d};
  char* arena = static_cast<char*>(rt->arena);
  char* host = static_cast<char*>(rt->host);
  for (uint64_t ai = 0; ai < rt->actions.size(); ++ai) {
    const delta_action& a = rt->actions[ai];
    cudaStream_t st = streams[a.stream < 3 ? a.stream : 0];
    const bool timed = t0 && (a.op == DELTA_ACT_COMPUTE || a.op == DELTA_ACT_RECOMPUTE ||
                              a.op == DELTA_ACT_OFFLOAD || a.op == DELTA_ACT_RELOAD);
    const bool work = a.op == DELTA_ACT_COMPUTE || a.op == DELTA_ACT_RECOMPUTE ||
                      a.op == DELTA_ACT_OFFLOAD || a.op == DELTA_ACT_RELOAD;
    const unsigned long long what = (static_cast<unsigned long long>(a.node) << 8) | a.op;
    if (stamps && work) {
      k_stamp<<<1, 1, 0, st>>>(stamps->log, stamps->count, stamps->cap, 2ull * ai, what);
      RT_CUDA(cudaGetLastError());
    }
    if (timed) RT_CUDA(cudaEventRecord(t0[ai], st));
    switch (a.op) {
      case DELTA_ACT_COMPUTE:
      case DELTA_ACT_RECOMPUTE: {
        delta_status s = run_node(rt, a, st);
        if (s) return s;
        break;
      }
      case DELTA_ACT_OFFLOAD:
        RT_CUDA(cudaMemcpyAsync(host + a.host_offset, arena + a.offset, a.bytes,
                                cudaMemcpyDeviceToHost, st));
        break;
      case DELTA_ACT_RELOAD:
        RT_CUDA(cudaMemcpyAsync(arena + a.offset, host + a.host_offset, a.bytes,
                                cudaMemcpyHostToDevice, st));
        break;
      case DELTA_ACT_RECORD:
        RT_CUDA(cudaEventRecord(rt->events.at(a.event), st));
        break;
      case DELTA_ACT_WAIT:
        RT_CUDA(cudaStreamWaitEvent(st, rt->events.at(a.event), 0));
        break;
      default:
        return fail(DELTA_E_ARGUMENT, "unknown action " + std::to_string(a.op));
    }
    if (timed) RT_CUDA(cudaEventRecord(t1[ai], st));
    if (stamps && work) {
      k_stamp<<<1, 1, 0, st>>>(stamps->log, stamps->count, stamps->cap, 2ull * ai + 1, what);
      RT_CUDA(cudaGetLastError());
    }
    if (a.op == DELTA_ACT_COMPUTE && !rt->ready_of.empty()) {
      auto r = rt->ready_of.find(a.node);
      if (r != rt->ready_of.end()) RT_CUDA(cudaEventRecord(rt->ready[r->second], st));
    }
    if (rt->after_fn && (a.op == DELTA_ACT_COMPUTE || a.op == DELTA_ACT_RECOMPUTE))
      rt->after_fn(rt->ctx, ai, a.node, reinterpret_cast<uint64_t>(arena + a.offset), st);
  }
  // join the copy streams that carried work back into the compute stream
  for (int s = 1; s < 3; ++s) {
    if (!rt->copy_used[s]) continue;
    RT_CUDA(cudaEventRecord(rt->join[s], streams[s]));
    RT_CUDA(cudaStreamWaitEvent(cs, rt->join[s], 0));
  }
  return DELTA_OK;
}

}  // namespace

extern "C" {

delta_status delta_rt_create(void* arena, uint64_t arena_bytes, uint64_t host_bytes,
                             delta_rt** out) {
  auto* rt = new delta_rt;
  rt->arena_bytes = arena_bytes;
  rt->host_bytes = host_bytes;
  cudaError_t e = cudaSuccess;
  if (arena) {
    rt->arena = arena;
  } else if (arena_bytes) {
    e = cudaMalloc(&rt->arena, arena_bytes);
    rt->own_arena = e == cudaSuccess;
  }
  if (e == cudaSuccess && host_bytes) e = cudaHostAlloc(&rt->host, host_bytes, cudaHostAllocPortable);
  int lo = 0, hi = 0;
  if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
  // copies get the high priority so a demand reload never queues behind compute
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&rt->d2h, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&rt->h2d, cudaStreamNonBlocking, hi);
  for (int s = 1; s < 3 && e == cudaSuccess; ++s)
    e = cudaEventCreateWithFlags(&rt->join[s], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&rt->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&rt->fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&rt->side_done, cudaEventDisableTiming);
  if (const char* v = std::getenv("DELTA_SIDE_STREAM")) rt->side_enabled = v[0] == '1';
  if (e != cudaSuccess) {
    delta_rt_destroy(rt);
    return cuda_fail(e, "delta_rt_create");
  }
  *out = rt;
  return DELTA_OK;
}

void* delta_rt_arena(const delta_rt* rt) { return rt->arena; }
void* delta_rt_host_slab(const delta_rt* rt) { return rt->host; }
void* delta_rt_copy_stream(const delta_rt* rt, int32_t which) {
  return which == 1 ? rt->d2h : which == 2 ? rt->h2d : nullptr;
}

delta_status delta_rt_bind(delta_rt* rt, const delta_program* prog, const delta_kop* kops,
                           uint64_t n_kops, const delta_recipe* recipes, uint64_t n_recipes) {
  delta_program_info info{};
  delta_status s = delta_program_info_get(prog, &info);
  if (s) return s;
  if (info.arena_bytes > rt->arena_bytes)
    return fail(DELTA_E_ARGUMENT, "delta_rt_bind: program arena " + std::to_string(info.arena_bytes) +
                                      " B exceeds the runtime's " + std::to_string(rt->arena_bytes));
  if (info.host_bytes > rt->host_bytes)
    return fail(DELTA_E_ARGUMENT, "delta_rt_bind: program host slab " +
                                      std::to_string(info.host_bytes) + " B exceeds the runtime's " +
                                      std::to_string(rt->host_bytes));
  uint64_t n = 0;
  const delta_action* acts = delta_program_actions(prog, &n);
  rt->actions.assign(acts, acts + n);
  const uint64_t* ins = delta_program_inputs(prog, &n);
  rt->inputs.assign(ins, ins + n);
  rt->kops.assign(kops, kops + n_kops);
  rt->recipe.clear();
  for (uint64_t j = 0; j < n_recipes; ++j) {
    if (uint64_t(recipes[j].first) + recipes[j].count > n_kops)
      return fail(DELTA_E_ARGUMENT, "delta_rt_bind: recipe past the op table");
    rt->recipe[recipes[j].node] = {recipes[j].first, recipes[j].count};
  }
  for (auto ev : rt->events) cudaEventDestroy(ev);
  rt->events.assign(info.n_events, nullptr);
  for (auto& ev : rt->events) RT_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  rt->copy_used[1] = rt->copy_used[2] = false;
  for (const auto& a : rt->actions)
    if (a.op == DELTA_ACT_OFFLOAD || a.op == DELTA_ACT_RELOAD) rt->copy_used[a.stream] = true;
  return DELTA_OK;
}

delta_status delta_rt_set_callbacks(delta_rt* rt, delta_host_fn host, delta_action_fn after,
                                    void* ctx) {
  rt->host_fn = host;
  rt->after_fn = after;
  rt->ctx = ctx;
  return DELTA_OK;
}

delta_status delta_rt_set_ready_nodes(delta_rt* rt, const uint64_t* nodes, uint32_t n) {
  for (auto ev : rt->ready) cudaEventDestroy(ev);
  rt->ready.assign(n, nullptr);
  rt->ready_of.clear();
  for (uint32_t i = 0; i < n; ++i) {
    RT_CUDA(cudaEventCreateWithFlags(&rt->ready[i], cudaEventDisableTiming));
    if (!rt->ready_of.emplace(nodes[i], i).second)
      return fail(DELTA_E_ARGUMENT, "delta_rt_set_ready_nodes: node listed twice");
  }
  return DELTA_OK;
}

delta_status delta_rt_wait_ready(delta_rt* rt, void* stream, uint32_t i) {
  if (i >= rt->ready.size()) return fail(DELTA_E_ARGUMENT, "delta_rt_wait_ready: no such event");
  RT_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), rt->ready[i], 0));
  return DELTA_OK;
}

delta_status delta_rt_step(delta_rt* rt, void* stream) {
  return issue(rt, static_cast<cudaStream_t>(stream), nullptr, nullptr);
}

delta_status delta_rt_step_timed(delta_rt* rt, void* stream, float* start_ms, float* end_ms,
                                 uint64_t n_actions) {
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  const uint64_t n = rt->actions.size();
  std::vector<cudaEvent_t> t0(n, nullptr), t1(n, nullptr);
  cudaEvent_t start = nullptr;
  delta_status s = DELTA_OK;
  cudaError_t e = cudaEventCreate(&start);
  for (uint64_t j = 0; j < n && e == cudaSuccess; ++j) {
    e = cudaEventCreate(&t0[j]);
    if (e == cudaSuccess) e = cudaEventCreate(&t1[j]);
  }
  if (e == cudaSuccess) {
    k_spin<<<1, 1, 0, cs>>>(100'000'000LL);  // ~50 ms at 1.9 GHz
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaEventRecord(start, cs);
  if (e != cudaSuccess) {
    s = cuda_fail(e, "delta_rt_step_timed events");
  } else {
    s = issue(rt, cs, t0.data(), t1.data());
  }
  if (!s) {
    e = cudaStreamSynchronize(cs);
    if (e != cudaSuccess) s = cuda_fail(e, "delta_rt_step_timed sync");
  }
  if (!s) {
    for (uint64_t j = 0; j < n && j < n_actions; ++j) {
      const auto op = rt->actions[j].op;
      float a = NAN, b = NAN;
      if (op == DELTA_ACT_COMPUTE || op == DELTA_ACT_RECOMPUTE || op == DELTA_ACT_OFFLOAD ||
          op == DELTA_ACT_RELOAD) {
        cudaEventElapsedTime(&a, start, t0[j]);
        cudaEventElapsedTime(&b, start, t1[j]);
      }
      if (start_ms) start_ms[j] = a;
      if (end_ms) end_ms[j] = b;
    }
  }
  for (auto ev : t0)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : t1)
    if (ev) cudaEventDestroy(ev);
  if (start) cudaEventDestroy(start);
  return s;
}

delta_status delta_rt_step_observed(delta_rt* rt, void* stream, uint64_t* records,
                                    uint64_t cap, uint64_t* n_records) {
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  StampLog sl;
  sl.cap = static_cast<unsigned int>(cap);
  void* mem = nullptr;
  const size_t bytes = 32 * size_t(cap) + 256;
  RT_CUDA(cudaMalloc(&mem, bytes));
  sl.log = static_cast<unsigned long long*>(mem);
  sl.count = reinterpret_cast<unsigned int*>(static_cast<char*>(mem) + 32 * size_t(cap));
  delta_status s = DELTA_OK;
  cudaError_t e = cudaMemsetAsync(sl.count, 0, 4, cs);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) s = cuda_fail(e, "delta_rt_step_observed setup");
  if (!s) s = issue(rt, cs, nullptr, nullptr, &sl);
  unsigned int n = 0;
  if (!s) {
    e = cudaStreamSynchronize(cs);
    if (e == cudaSuccess) e = cudaMemcpy(&n, sl.count, 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && n > cap) {
      s = fail(DELTA_E_ARGUMENT, "delta_rt_step_observed: " + std::to_string(n) +
                                     " records exceed the capacity " + std::to_string(cap));
    } else if (e == cudaSuccess) {
      e = cudaMemcpy(records, sl.log, 32 * size_t(n), cudaMemcpyDeviceToHost);
    }
    if (e != cudaSuccess && !s) s = cuda_fail(e, "delta_rt_step_observed readback");
  }
  cudaFree(mem);
  if (n_records) *n_records = s ? 0 : n;
  return s;
}

delta_status delta_rt_measure_costs(delta_rt* rt, void* stream, uint32_t iters, uint64_t* cost_us,
                                    uint64_t n_nodes) {
  const uint64_t n = rt->actions.size();
  std::vector<float> a(n), b(n);
  std::unordered_map<uint64_t, std::vector<float>> samples;
  for (uint32_t it = 0; it < iters + 1; ++it) {  // the first step warms up
    delta_status s = delta_rt_step_timed(rt, stream, a.data(), b.data(), n);
    if (s) return s;
    if (it == 0) continue;
    std::unordered_map<uint64_t, bool> seen;
    for (uint64_t j = 0; j < n; ++j) {
      const auto& act = rt->actions[j];
      if (act.op != DELTA_ACT_COMPUTE || seen[act.node]) continue;
      seen[act.node] = true;
      samples[act.node].push_back(b[j] - a[j]);
    }
  }
  for (auto& kv : samples) {
    if (kv.first >= n_nodes) continue;
    auto& v = kv.second;
    std::sort(v.begin(), v.end());
    const double us = double(v[v.size() / 2]) * 1e3;
    cost_us[kv.first] = std::max<uint64_t>(1, uint64_t(std::ceil(us)));
  }
  return DELTA_OK;
}

void delta_rt_destroy(delta_rt* rt) {
  if (!rt) return;
  for (auto ev : rt->ready)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : rt->events)
    if (ev) cudaEventDestroy(ev);
  for (int s = 1; s < 3; ++s)
    if (rt->join[s]) cudaEventDestroy(rt->join[s]);
  if (rt->side) cudaStreamDestroy(rt->side);
  if (rt->fork) cudaEventDestroy(rt->fork);
  if (rt->side_done) cudaEventDestroy(rt->side_done);
  if (rt->d2h) cudaStreamDestroy(rt->d2h);
  if (rt->h2d) cudaStreamDestroy(rt->h2d);
  if (rt->host) cudaFreeHost(rt->host);
  if (rt->own_arena && rt->arena) cudaFree(rt->arena);
  delete rt;
}

}  // extern "C"
