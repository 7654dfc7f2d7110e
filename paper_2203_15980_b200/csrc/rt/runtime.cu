// C ABI of the B200 execution side: kernel launchers, the swap engine (pinned
// slab + copy-engine streams) and the host-link probe of the cost model.
#include <cuda_runtime.h>

#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "delta/delta_kernels.h"
#include "kernels/kernels.hpp"
#include "rt/handles.hpp"

namespace delta_rt {
void set_error(const std::string& msg);  // capi.cpp
}

namespace {

delta_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DELTA_OK;
  delta_rt::set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return DELTA_E_CUDA;
}
#define DELTA_CUDA(expr) \
  do { delta_status s_ = cuda_status((expr), #expr); if (s_) return s_; } while (0)

inline cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }

}  // namespace

struct delta_swap {
  void* host = nullptr;
  uint64_t bytes = 0;
  cudaStream_t d2h = nullptr, h2d = nullptr;
};

struct delta_events {
  std::vector<cudaEvent_t> ev;
};

extern "C" {

delta_status delta_conv_create(int32_t N, int32_t H, int32_t W, int32_t C, int32_t K, int32_t R,
                               int32_t S_, int32_t stride, int32_t pad, const void* weight,
                               delta_conv** out) {
  return delta_conv_create_ex(N, H, W, C, K, R, S_, stride, pad, -1, -1, weight, out);
}

delta_status delta_conv_create_ex(int32_t N, int32_t H, int32_t W, int32_t C, int32_t K, int32_t R,
                                  int32_t S_, int32_t stride, int32_t pad, int32_t pad_end_h,
                                  int32_t pad_end_w, const void* weight, delta_conv** out) {
  auto* c = new delta_conv;
  std::memset(&c->plan, 0, sizeof(c->plan));
  c->plan.N = N; c->plan.H = H; c->plan.W = W; c->plan.C = C; c->plan.K = K;
  c->plan.R = R; c->plan.S = S_; c->plan.stride = stride; c->plan.pad = pad;
  c->plan.pad_end_h = pad_end_h; c->plan.pad_end_w = pad_end_w;
  c->weight = weight;
  int rc = delta_k::conv_plan_init(&c->plan, weight);
  if (rc != 0) {
    delete c;
    delta_rt::set_error(rc == 1 ? "conv: unsupported shape (need C%64==0 or C==4, K%8==0)"
                        : rc == 2 ? "conv: cuTensorMapEncodeTiled entry point unavailable"
                                  : "conv: tensor map encode failed");
    return rc == 1 ? DELTA_E_UNSUPPORTED : DELTA_E_CUDA;
  }
  *out = c;
  return DELTA_OK;
}

delta_status delta_conv_create_t(int32_t M, int32_t C, int32_t K, const void* weight_ck,
                                 delta_conv** out) {
  auto* c = new delta_conv;
  std::memset(&c->plan, 0, sizeof(c->plan));
  c->plan.N = M; c->plan.H = 1; c->plan.W = 1; c->plan.C = C; c->plan.K = K;
  c->plan.R = 1; c->plan.S = 1; c->plan.stride = 1; c->plan.pad = 0;
  c->plan.pad_end_h = -1; c->plan.pad_end_w = -1;
  c->plan.bmn = 1;
  c->weight = weight_ck;
  int rc = delta_k::conv_plan_init(&c->plan, weight_ck);
  if (rc != 0) {
    delete c;
    delta_rt::set_error(rc == 1 ? "conv_t: unsupported shape (need C%64==0, K%64==0)"
                                : "conv_t: tensor map encode failed");
    return rc == 1 ? DELTA_E_UNSUPPORTED : DELTA_E_CUDA;
  }
  *out = c;
  return DELTA_OK;
}

delta_status delta_conv_forward(const delta_conv* c, const void* x, void* y, float* stats,
                                void* stream) {
  return cuda_status(delta_k::conv_forward(c->plan, x, y, stats, S(stream)), "conv_forward");
}

static_assert(sizeof(delta_conv_epilogue) == sizeof(delta_k::ConvEpilogue),
              "C-ABI epilogue struct mirrors the kernel's");

delta_status delta_conv_forward_ex(const delta_conv* c, const void* x, void* y, float* stats,
                                   const delta_conv_epilogue* epi, void* stream) {
  delta_k::ConvEpilogue e{};
  if (epi) {
    e.mode = epi->mode;
    e.pool_hw = epi->pool_hw;
    e.add_stride2 = epi->add_stride2;
    e.scatter = epi->scatter;
    e.add = epi->add;
    e.add_mask = epi->add_mask;
    e.out_mask = epi->out_mask;
    e.xc = epi->xc;
    e.mean = epi->mean;
    e.invstd = epi->invstd;
    e.gamma = epi->gamma;
    e.beta = epi->beta;
  }
  return cuda_status(delta_k::conv_forward(c->plan, x, y, stats, S(stream), &e), "conv_forward_ex");
}

delta_status delta_wgrad_create(int32_t N, int32_t H, int32_t W, int32_t C, int32_t K, int32_t R,
                                int32_t S_, int32_t stride, int32_t pad, delta_wgrad** out) {
  auto* w = new delta_wgrad;
  std::memset(&w->plan, 0, sizeof(w->plan));
  w->plan.N = N; w->plan.H = H; w->plan.W = W; w->plan.C = C; w->plan.K = K;
  w->plan.R = R; w->plan.S = S_; w->plan.stride = stride; w->plan.pad = pad;
  if (delta_k::wgrad_plan_init(&w->plan) != 0) {
    delete w;
    delta_rt::set_error("wgrad: unsupported shape (need C%64==0 or the C==4 stem, K%64==0)");
    return DELTA_E_UNSUPPORTED;
  }
  *out = w;
  return DELTA_OK;
}

int32_t delta_wgrad_launches(const delta_wgrad* w) { return delta_k::wgrad_launches(w->plan); }

uint64_t delta_wgrad_workspace_bytes(const delta_wgrad* w) {
  return delta_k::wgrad_workspace_bytes(w->plan);
}

delta_status delta_wgrad_run(const delta_wgrad* w, const void* dy, const void* x, float* dw, void* ws,
                         void* stream) {
  return cuda_status(delta_k::wgrad(w->plan, dy, x, dw, static_cast<float*>(ws), S(stream)),
                     "wgrad");
}

void delta_wgrad_destroy(delta_wgrad* w) { delete w; }

delta_status delta_conv_set_tile_n(delta_conv* c, int32_t tile_n) {
  const int rc = delta_k::conv_plan_set_tile_n(&c->plan, tile_n, c->weight);
  if (rc == 0) return DELTA_OK;
  delta_rt::set_error(rc == 1 ? "conv: tile_n must be 64/128/256 and divide K"
                              : "conv: tensor map encode failed");
  return rc == 1 ? DELTA_E_UNSUPPORTED : DELTA_E_CUDA;
}


delta_status delta_conv_geometry(const delta_conv* c, int32_t* P, int32_t* Q, int32_t* kdim,
                                 int32_t* tile_n) {
  if (P) *P = c->plan.P;
  if (Q) *Q = c->plan.Q;
  if (kdim) *kdim = c->plan.kdim;
  if (tile_n) *tile_n = c->plan.bn;
  return DELTA_OK;
}

void delta_conv_destroy(delta_conv* c) { delete c; }

int64_t delta_bn_workspace_floats(int64_t M, int32_t C) { return delta_k::bn_workspace_floats(M, C); }

delta_status delta_bn_stats(const void* x, int64_t M, int32_t C, float* ws, float* mean,
                            float* invstd, float eps, float* rm, float* rv, float mom,
                            void* stream) {
  return cuda_status(delta_k::bn_stats(x, M, C, ws, mean, invstd, eps, rm, rv, mom, S(stream)),
                     "bn_stats");
}

int32_t delta_stats_parts(void) { return delta_k::stats_parts(); }

int64_t delta_stats_partials_floats(int32_t C) { return delta_k::stats_partials_floats(C); }

delta_status delta_stats_col_sum(const float* partials, int32_t C, float* out, int32_t accumulate,
                                 void* stream) {
  DELTA_CUDA(delta_k::stats_col_sum(partials, C, out, accumulate, S(stream)));
  return DELTA_OK;
}

delta_status delta_bn_stats_from_partials(const float* partials, int32_t C, float* mean,
                                          float* invstd, float eps, float* rm, float* rv,
                                          float mom, void* stream) {
  return cuda_status(
      delta_k::bn_stats_from_partials(partials, C, mean, invstd, eps, rm, rv, mom, S(stream)),
      "bn_stats_from_partials");
}

delta_status delta_sgd_step(float* w, float* mom, const float* g, void* wbf, int64_t n,
                            int64_t n_bf, float lr, float momentum, float weight_decay,
                            void* stream) {
  return cuda_status(
      delta_k::sgd_step(w, mom, g, wbf, n, n_bf, lr, momentum, weight_decay, S(stream)),
      "sgd_step");
}

delta_status delta_weight_views(const delta_weight_view* views_dev, int32_t n_views,
                                void* stream) {
  return cuda_status(delta_k::weight_views(views_dev, n_views, S(stream)), "weight_views");
}

delta_status delta_bn_apply(int32_t mode, const void* x, const void* res, void* y, int64_t M,
                            int32_t C, const float* mean, const float* invstd, const float* gamma,
                            const float* beta, const float* mean2, const float* invstd2,
                            const float* gamma2, const float* beta2, void* stream) {
  return cuda_status(delta_k::bn_apply(mode, x, res, y, M, C, mean, invstd, gamma, beta, mean2,
                                       invstd2, gamma2, beta2, S(stream)),
                     "bn_apply");
}

delta_status delta_bn_backward(const void* up, int32_t pool_hw, const void* mask, const void* x,
                               void* dx, int64_t M, int32_t C, const float* mean,
                               const float* invstd, const float* gamma, float* dgamma,
                               float* dbeta, float* ws, void* stream) {
  return cuda_status(delta_k::bn_backward(up, pool_hw, mask, x, dx, M, C, mean, invstd, gamma,
                                          dgamma, dbeta, ws, S(stream)),
                     "bn_backward");
}

delta_status delta_bn_backward_from_partials(const float* partials, const void* g, const void* x,
                                             void* dx, int64_t M, int32_t C, const float* mean,
                                             const float* invstd, const float* gamma,
                                             float* dgamma, float* dbeta, void* stream) {
  return cuda_status(delta_k::bn_backward_from_partials(partials, g, x, dx, M, C, mean, invstd,
                                                        gamma, dgamma, dbeta, S(stream)),
                     "bn_backward_from_partials");
}

delta_status delta_add_grad(const void* a, const void* up, int32_t pool_hw, const void* up_mask,
                            const void* out_mask, void* out, int64_t M, int32_t C, void* stream) {
  return cuda_status(delta_k::add_grad(a, up, pool_hw, up_mask, out_mask, out, M, C, S(stream)),
                     "add_grad");
}

delta_status delta_maxpool3x3s2_fwd(const void* x, void* y, int32_t N, int32_t H, int32_t W,
                                    int32_t C, void* stream) {
  return cuda_status(delta_k::maxpool3x3s2_fwd(x, y, N, H, W, C, S(stream)), "maxpool_fwd");
}

int64_t delta_maxpool_workspace_bytes(int32_t N, int32_t H, int32_t W, int32_t C) {
  return delta_k::maxpool_workspace_bytes(N, H, W, C);
}

delta_status delta_maxpool3x3s2_bwd(const void* dy, const void* x, void* dx, int32_t N, int32_t H,
                                    int32_t W, int32_t C, void* ws, void* stream) {
  return cuda_status(delta_k::maxpool3x3s2_bwd(dy, x, dx, N, H, W, C, ws, S(stream)),
                     "maxpool_bwd");
}

delta_status delta_avgpool_fwd(const void* x, void* y, int32_t N, int32_t HW, int32_t C,
                               void* stream) {
  return cuda_status(delta_k::avgpool_fwd(x, y, N, HW, C, S(stream)), "avgpool_fwd");
}

delta_status delta_softmax_xent_head(const void* logits, int32_t ld, const float* bias,
                                     const int64_t* labels, float* loss, float* dlogits,
                                     void* dlogits_bf16, float* dbias, float* row_ws, int32_t N,
                                     int32_t K, void* stream) {
  return cuda_status(delta_k::softmax_xent_head(logits, ld, bias, labels, loss, dlogits,
                                                dlogits_bf16, dbias, row_ws, N, K, S(stream)),
                     "softmax_xent_head");
}

delta_status delta_softmax_xent(const float* logits, const int64_t* labels, float* loss,
                                float* dlogits, float* row_ws, int32_t N, int32_t K,
                                void* stream) {
  return cuda_status(delta_k::softmax_xent(logits, labels, loss, dlogits, row_ws, N, K, S(stream)),
                     "softmax_xent");
}

// ---- swap engine ----
delta_status delta_swap_create(uint64_t host_bytes, delta_swap** out) {
  auto* s = new delta_swap;
  s->bytes = host_bytes;
  if (host_bytes) {
    cudaError_t e = cudaHostAlloc(&s->host, host_bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
      delete s;
      return cuda_status(e, "cudaHostAlloc(swap slab)");
    }
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  // copies get the high priority so a demand reload is never queued behind
  // compute; compute stays on the caller's stream.
  cudaError_t e1 = cudaStreamCreateWithPriority(&s->d2h, cudaStreamNonBlocking, hi);
  cudaError_t e2 = cudaStreamCreateWithPriority(&s->h2d, cudaStreamNonBlocking, hi);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    if (s->host) cudaFreeHost(s->host);
    delete s;
    return cuda_status(e1 != cudaSuccess ? e1 : e2, "cudaStreamCreate(swap)");
  }
  *out = s;
  return DELTA_OK;
}

void* delta_swap_host_ptr(const delta_swap* s) { return s->host; }
void* delta_swap_stream(const delta_swap* s, int32_t which) {
  return which == 1 ? s->d2h : which == 2 ? s->h2d : nullptr;
}

delta_status delta_swap_offload(delta_swap* s, const void* dev, uint64_t off, uint64_t bytes,
                                void* stream) {
  if (off + bytes > s->bytes) {
    delta_rt::set_error("swap offload past the host slab");
    return DELTA_E_ARGUMENT;
  }
  return cuda_status(cudaMemcpyAsync(static_cast<char*>(s->host) + off, dev, bytes,
                                     cudaMemcpyDeviceToHost, stream ? S(stream) : s->d2h),
                     "offload");
}

delta_status delta_swap_reload(delta_swap* s, void* dev, uint64_t off, uint64_t bytes,
                               void* stream) {
  if (off + bytes > s->bytes) {
    delta_rt::set_error("swap reload past the host slab");
    return DELTA_E_ARGUMENT;
  }
  return cuda_status(cudaMemcpyAsync(dev, static_cast<char*>(s->host) + off, bytes,
                                     cudaMemcpyHostToDevice, stream ? S(stream) : s->h2d),
                     "reload");
}

void delta_swap_destroy(delta_swap* s) {
  if (!s) return;
  if (s->d2h) cudaStreamDestroy(s->d2h);
  if (s->h2d) cudaStreamDestroy(s->h2d);
  if (s->host) cudaFreeHost(s->host);
  delete s;
}

// ---- cost model: host link ----
delta_status delta_probe_link(uint64_t bytes, int32_t iters, double* h2d, double* d2h,
                              double* duplex) {
  void *host = nullptr, *host2 = nullptr, *dev = nullptr, *dev2 = nullptr;
  cudaStream_t a = nullptr, b = nullptr;
  cudaEvent_t e0, e1, e2, e3;
  delta_status rc = DELTA_OK;
  auto fail = [&](cudaError_t e, const char* w) {
    if (rc == DELTA_OK && e != cudaSuccess) rc = cuda_status(e, w);
  };
  fail(cudaHostAlloc(&host, bytes, cudaHostAllocPortable), "probe host alloc");
  fail(cudaHostAlloc(&host2, bytes, cudaHostAllocPortable), "probe host alloc");
  fail(cudaMalloc(&dev, bytes), "probe dev alloc");
  fail(cudaMalloc(&dev2, bytes), "probe dev alloc");
  fail(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking), "probe stream");
  fail(cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking), "probe stream");
  cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2); cudaEventCreate(&e3);
  if (rc == DELTA_OK) {
    std::memset(host, 1, bytes);
    std::memset(host2, 2, bytes);
    for (int w = 0; w < 2; ++w) {  // warm-up
      cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, a);
      cudaMemcpyAsync(host2, dev2, bytes, cudaMemcpyDeviceToHost, b);
    }
    cudaDeviceSynchronize();
    float ms = 0.f;
    cudaEventRecord(e0, a);
    for (int i = 0; i < iters; ++i) cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, a);
    cudaEventRecord(e1, a);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    *h2d = double(bytes) * iters / (ms * 1e-3) / 1e9;
    cudaEventRecord(e0, b);
    for (int i = 0; i < iters; ++i) cudaMemcpyAsync(host2, dev2, bytes, cudaMemcpyDeviceToHost, b);
    cudaEventRecord(e1, b);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    *d2h = double(bytes) * iters / (ms * 1e-3) / 1e9;
    // both directions at once (two copy engines)
    cudaEventRecord(e0, a);
    cudaStreamWaitEvent(b, e0, 0);
    for (int i = 0; i < iters; ++i) {
      cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, a);
      cudaMemcpyAsync(host2, dev2, bytes, cudaMemcpyDeviceToHost, b);
    }
    cudaEventRecord(e2, b);
    cudaStreamWaitEvent(a, e2, 0);
    cudaEventRecord(e3, a);
    cudaEventSynchronize(e3);
    cudaEventElapsedTime(&ms, e0, e3);
    *duplex = 2.0 * double(bytes) * iters / (ms * 1e-3) / 1e9;
    fail(cudaGetLastError(), "probe copies");
  }
  cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2); cudaEventDestroy(e3);
  if (a) cudaStreamDestroy(a);
  if (b) cudaStreamDestroy(b);
  if (dev) cudaFree(dev);
  if (dev2) cudaFree(dev2);
  if (host) cudaFreeHost(host);
  if (host2) cudaFreeHost(host2);
  return rc;
}

// ---- events ----
delta_status delta_events_create(uint32_t n, delta_events** out) {
  auto* e = new delta_events;
  e->ev.resize(n, nullptr);
  for (uint32_t i = 0; i < n; ++i) {
    cudaError_t r = cudaEventCreateWithFlags(&e->ev[i], cudaEventDisableTiming);
    if (r != cudaSuccess) {
      for (uint32_t j = 0; j < i; ++j) cudaEventDestroy(e->ev[j]);
      delete e;
      return cuda_status(r, "cudaEventCreate");
    }
  }
  *out = e;
  return DELTA_OK;
}

delta_status delta_event_record(delta_events* e, uint32_t i, void* stream) {
  return cuda_status(cudaEventRecord(e->ev.at(i), S(stream)), "cudaEventRecord");
}

delta_status delta_event_wait(delta_events* e, uint32_t i, void* stream) {
  return cuda_status(cudaStreamWaitEvent(S(stream), e->ev.at(i), 0), "cudaStreamWaitEvent");
}

void delta_events_destroy(delta_events* e) {
  if (!e) return;
  for (cudaEvent_t x : e->ev) cudaEventDestroy(x);
  delete e;
}

}  // extern "C"
