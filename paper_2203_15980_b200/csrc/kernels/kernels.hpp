// Internal launch interface of the sm_100a kernels (wrapped by capi_kernels.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "delta/delta_kernels.h"

namespace delta_k {

// ---- implicit-GEMM convolution (conv_fwd.cu) ----
struct ConvPlan {
  int N, H, W, C, K, R, S, stride, pad;
  int pad_end_h, pad_end_w;  // padding after the last row / column (conv_plan_init: -1 = pad)
  int P, Q, kdim, bn;
  int halo, halo_slot, halo_rows;  // 3x3 stride-1: input halo staged per tile (conv_halo.cu)
  int stem_rows;                   // C=4 stem: one output row per tile (conv_fwd.cu MODE_STEMROW)
  const void* wptr;                // the weights (pair mode encodes its half-tile map per launch)
  int bmn;                         // 1x1 only: weights stored [kdim][K] (read MN-major; e.g. an
                                   // input gradient straight from the forward's [out][in])
  alignas(64) unsigned char wmap[128];  // CUtensorMap over the [K][kdim] weight matrix
};
// Fused epilogues (the backward pass runs input-gradient convolutions through
// the same kernel with transposed/flipped weights):
//   EPI_STORE    y = bf16(acc)                                  [+ BN-stats partials]
//   EPI_ADD_MASK y = bf16((acc + add') * [out_mask > 0]),  add' = add or pooled
//                add / pool_hw, times [add_mask > 0]             (gradient adds)
//   EPI_BN_BWD   y = g = bf16(acc) * [relu(bn(xc)) > 0], partials (sum g,
//                sum g*xc) per 128-row tile                     (BN+ReLU backward)
//   EPI_SCATTER2 y[n][2p+a][2q+b][k] = bf16(acc) into a [N][2P][2Q][K] tensor,
//                (a, b) = (scatter >> 1, scatter & 1): one parity class of a
//                stride-2 input gradient (sub-pixel decomposition)
//   EPI_BIAS     y = bf16(acc + beta[k])                        (linear layers)
//   EPI_GELU_BWD y = bf16(acc * gelu'(xc)), xc the [M][K] pre-activation
constexpr int EPI_STORE = 0, EPI_ADD_MASK = 1, EPI_BN_BWD = 2, EPI_SCATTER2 = 3, EPI_BIAS = 4,
              EPI_GELU_BWD = 5;
struct ConvEpilogue {
  int mode;
  int pool_hw;
  int add_stride2;  // EPI_ADD_MASK: `add` is given at the even rows/columns only,
                    // as a [N][P/2][Q/2][K] tensor (zero elsewhere)
  int scatter;      // EPI_SCATTER2: parity class a*2 + b
  const void* add;
  const void* add_mask;
  const void* out_mask;
  const void* xc;
  const float* mean;
  const float* invstd;
  const float* gamma;
  const float* beta;
};
// 0 ok, 1 unsupported shape, 2 no driver entry point, 3 tensor-map encode failed
int conv_plan_init(ConvPlan* cp, const void* w);
// conv_halo.cu: the 3x3 stride-1 halo path (plain epilogue + BN statistics)
bool conv_halo_eligible(const ConvPlan& cp);
bool conv_halo_default(const ConvPlan& cp);  // the shapes it is dispatched for by default
void conv_halo_shape(ConvPlan* cp);
cudaError_t conv_halo_forward(const ConvPlan& cp, const void* x, void* y, float* stats,
                              cudaStream_t st);
// choose the N tile (64/128/256, dividing K; fused epilogues need <= 128)
int conv_plan_set_tile_n(ConvPlan* cp, int bn, const void* w);
// stats (optional, nullptr = off): [ceil(M/128)][K] float2 (mean, M2) of the
// bf16 outputs of each 128-row tile — the BN statistics partials.
cudaError_t conv_forward(const ConvPlan& cp, const void* x, void* y, float* stats,
                         cudaStream_t st, const ConvEpilogue* epi = nullptr);

// ---- optimizer step + weight views (optim.cu) ----
cudaError_t sgd_step(float* w, float* mom, const float* g, void* wbf, int64_t n, int64_t n_bf,
                     float lr, float m, float wd, cudaStream_t st);
cudaError_t weight_views(const delta_weight_view* views_dev, int n_views, cudaStream_t st);

// ---- weight gradient (wgrad.cu) ----
struct WgradPlan {
  int N, H, W, C, K, R, S, stride, pad;  // the forward conv (C == 4: the pair-view stem)
  int P, Q, mode, bn, taps, tiles, splits, kb_per_split;
  int mt;  // 128-row output-channel blocks per tile (2: two accumulators share each B tile)
  int pair;  // 256-channel tiles on a CTA pair (cta_group::2)
};
// 0 ok, 1 unsupported shape
int wgrad_plan_init(WgradPlan* wp);
size_t wgrad_workspace_bytes(const WgradPlan& wp);
int wgrad_launches(const WgradPlan& wp);  // 1, or 2 with the separate split reduce
// dw: fp32 [K][R][S][C] (overwritten); ws: wgrad_workspace_bytes of scratch
cudaError_t wgrad(const WgradPlan& wp, const void* dy, const void* x, float* dw, float* ws,
                  cudaStream_t st);

// ---- batch norm / elementwise / pooling (bn_pool.cu) ----
int64_t bn_workspace_floats(int64_t M, int C);
cudaError_t bn_stats(const void* x, int64_t M, int C, float* ws, float* mean, float* invstd,
                     float eps, float* run_mean, float* run_var, float momentum, cudaStream_t st);
// Finish BN statistics from the conv epilogue's per-CTA partial rows
// (stats_cta.cuh: stats_parts() rows of float4 (count, mean, M2) per channel),
// merged in a fixed order by one launch.  `partials` holds
// stats_partials_floats(C) floats.
int stats_parts();
int64_t stats_partials_floats(int C);
cudaError_t bn_stats_from_partials(const float* partials, int C, float* mean, float* invstd,
                                   float eps, float* run_mean, float* run_var, float momentum,
                                   cudaStream_t st);

// out[c] (=|+=) sum over the rows of count * mean: column sums of the
// outputs a conv/GEMM epilogue reduced into statistics partials
cudaError_t stats_col_sum(const float* partials, int C, float* out, int accumulate,
                          cudaStream_t st);

// mode 0: y = relu(bn(x)); 1: y = relu(bn(x) + res); 2: y = relu(bn(x) + bn2(res))
cudaError_t bn_apply(int mode, const void* x, const void* res, void* y, int64_t M, int C,
                     const float* mean, const float* invstd, const float* gamma, const float* beta,
                     const float* mean2, const float* invstd2, const float* gamma2,
                     const float* beta2, cudaStream_t st);

// BN(+ReLU) backward.  g = up * (mask > 0) (mask may be null: g = up), where `up` is a full [M,C] bf16
// gradient (pool_hw == 0) or a pooled [N,C] bf16 gradient broadcast over
// pool_hw pixels and scaled by 1/pool_hw.  Writes dx (bf16) and the
// parameter gradients dgamma, dbeta (fp32).
cudaError_t bn_backward(const void* up, int pool_hw, const void* mask, const void* x, void* dx,
                        int64_t M, int C, const float* mean, const float* invstd,
                        const float* gamma, float* dgamma, float* dbeta, float* ws,
                        cudaStream_t st);

// BN(+ReLU) backward whose reductions were fused into the producing conv's
// EPI_BN_BWD epilogue: `partials` = per-CTA rows (sum g, sum g*x) of g (already
// masked), sized stats_partials_floats(C).  Writes dgamma, dbeta and
// dx = BN-backward(g, x).
cudaError_t bn_backward_from_partials(const float* partials, const void* g, const void* x,
                                      void* dx, int64_t M, int C, const float* mean,
                                      const float* invstd, const float* gamma, float* dgamma,
                                      float* dbeta, cudaStream_t st);

// out = (a + g) * [out_mask > 0], g = up * [up_mask > 0] (up full or pooled as
// above; a null mask means no masking)
cudaError_t add_grad(const void* a, const void* up, int pool_hw, const void* up_mask,
                     const void* out_mask, void* out, int64_t M, int C, cudaStream_t st);

cudaError_t maxpool3x3s2_fwd(const void* x, void* y, int N, int H, int W, int C, cudaStream_t st);
int64_t maxpool_workspace_bytes(int N, int H, int W, int C);
cudaError_t maxpool3x3s2_bwd(const void* dy, const void* x, void* dx, int N, int H, int W, int C,
                             void* ws, cudaStream_t st);
cudaError_t avgpool_fwd(const void* x, void* y, int N, int HW, int C, cudaStream_t st);

// loss = mean_i -log softmax(logits_i)[label_i]; dlogits = (softmax - onehot) / N
cudaError_t softmax_xent(const float* logits, const int64_t* labels, float* loss, float* dlogits,
                         float* row_loss_ws, int N, int K, cudaStream_t st);
// classifier head on bf16 GEMM logits [N][ld] (+ fp32 bias): loss, dlogits
// fp32 [N][K], its bf16 copy [N][ld] (zero pad columns), dbias = column sums
cudaError_t softmax_xent_head(const void* logits, int ld, const float* bias,
                              const int64_t* labels, float* loss, float* dlogits, void* dl_bf16,
                              float* dbias, float* row_loss_ws, int N, int K, cudaStream_t st);

}  // namespace delta_k
