/* delta-b200 C ABI — the B200 execution side of the DELTA runtime.
 *
 * The reference simulates these subsystems (include/deltasim/device.hpp:17-74
 * MemoryPool / Stream / Clock; OpNode::compute_cost_us at trace.hpp:17 as the
 * "recompute" of a tensor; policy.cpp:58-64 as the "swap").  Here they are
 * real:
 *   recompute engine : sm_100a kernels that (re)produce every activation
 *                      (tcgen05 implicit-GEMM conv; HBM-bound BN/ReLU/add/pool),
 *   swap engine      : pinned host slab + D2H/H2D copy-engine streams + events,
 *   cost model       : device-timed op latencies and a host-link probe.
 * All tensors are device pointers (NHWC bf16 activations unless stated);
 * `stream` is a cudaStream_t passed as void*.  Every call is asynchronous on
 * `stream`; errors are reported as delta_status (delta.h), never thrown.
 */
#ifndef DELTA_DELTA_KERNELS_H_
#define DELTA_DELTA_KERNELS_H_

#include <stdint.h>

#include "delta/delta.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- recompute engine: convolution (ConvForward, ref src/trace.cpp:403) ----
 * Weights are [K][R][S][C] bf16.  C == 4 is the 7x7/2 pad-3 stem over an
 * even-width image, computed as a 7x4 conv over pixel pairs: weights
 * [K][256] bf16, column (r*4 + j)*8 + e*4 + c holds W[k][r][2j+e-1][c]
 * (zero for 2j+e-1 < 0 and for columns >= 224).  The handle caches the TMA
 * descriptor of the weights. */
typedef struct delta_conv delta_conv;
delta_status delta_conv_create(int32_t N, int32_t H, int32_t W, int32_t C, int32_t K,
                               int32_t R, int32_t S, int32_t stride, int32_t pad,
                               const void* weight, delta_conv** out);
/* As delta_conv_create with `pad` before the first row/column and
 * pad_end_h / pad_end_w after the last (-1 = pad): P = H + pad + pad_end_h -
 * R + 1 (stride 1 only).  The sub-pixel convolutions of a stride-2 input
 * gradient are R', S' in {1, 2} with pad 0 and pad_end = R'-1, S'-1. */
delta_status delta_conv_create_ex(int32_t N, int32_t H, int32_t W, int32_t C, int32_t K,
                                  int32_t R, int32_t S, int32_t stride, int32_t pad,
                                  int32_t pad_end_h, int32_t pad_end_w, const void* weight,
                                  delta_conv** out);
/* A 1x1 GEMM y[M][K] = x[M][C] . W with the weights stored [C][K] (read
 * through MN-major descriptors): e.g. a linear layer's input gradient straight
 * from its forward weights [out][in], no transposed copy.  Plain
 * (DELTA_EPI_STORE) and DELTA_EPI_GELU_BWD epilogues. */
delta_status delta_conv_create_t(int32_t M, int32_t C, int32_t K, const void* weight_ck,
                                 delta_conv** out);
/* `stats` (nullable): [ceil(N*P*Q/128)][K] float2 (mean, M2) per 128-row tile
 * of the bf16 outputs — BatchNorm statistics partials fused in the epilogue. */
delta_status delta_conv_forward(const delta_conv* c, const void* x, void* y, float* stats,
                                void* stream);
/* Fused epilogues.  The backward pass runs input-gradient (dgrad) convolutions
 * of stride-1 layers through the same kernel: x = dY [N][P][Q][K], weights
 * transposed (1x1: [C][K]) or flipped and transposed (RxS: [C][R][S][K] with
 * W'[c][r][s][k] = W[k][R-1-r][S-1-s][c]).
 *   DELTA_EPI_ADD_MASK: y = bf16((acc + add') * [out_mask > 0]); add' = add
 *       ([M][K]), or with pool_hw > 0 the pooled add ([N][K]) / pool_hw *
 *       [add_mask > 0] (add_mask is read only with a pooled add).  With
 *       add_stride2 = 1 the full add is the input gradient of a stride-2 1x1
 *       conv: given as [N][P/2][Q/2][K] at the even rows/columns, zero elsewhere.
 *       Null pointers are skipped.  (The residual-branch gradient sum.)
 *       With a full add, out_mask, xc and `stats` all given (1x1, tile_n 64):
 *       `stats` also receives the per-CTA (sum y, sum y*xc) rows of the BN
 *       backward that consumes y (xc = that BN's input), for
 *       delta_bn_backward_from_partials — its partial pass is skipped.
 *   DELTA_EPI_BN_BWD: y = g = bf16(acc) * [relu(bn(xc)) > 0] with the saved
 *       statistics (the forward's exact arithmetic), and `stats` receives the
 *       per-CTA (sum g, sum g*xc) partial rows for delta_bn_backward_from_partials.
 *   DELTA_EPI_SCATTER2: the input gradient of a stride-2 3x3 (pad 1) conv
 *       as four sub-pixel stride-1 convolutions over dY (parity class (a, b),
 *       scatter = 2a + b, with the class's taps of the flipped weights,
 *       delta_weight_view DELTA_VIEW_DGRAD_S2): output pixel (p, q) of class
 *       (a, b) is written to y[n][2p+a][2q+b][:] of the [N][2P][2Q][K]
 *       gradient.  The four classes tile y exactly once.
 *   DELTA_EPI_BIAS: y = bf16(acc + beta[k]) — a linear layer (1x1, stride 1:
 *       x = [tokens][in], weights [out][in]) with its bias (`beta`).
 *   DELTA_EPI_GELU_BWD: y = bf16(acc * gelu'(xc)), xc = the [M][K] GELU input
 *       (erf GELU): the MLP input gradient through the GELU (1x1 only,
 *       tile_n <= 128).
 * Output channels must be a multiple of 32 for the fused modes. */
enum {
  DELTA_EPI_STORE = 0,
  DELTA_EPI_ADD_MASK = 1,
  DELTA_EPI_BN_BWD = 2,
  DELTA_EPI_SCATTER2 = 3,
  DELTA_EPI_BIAS = 4,
  DELTA_EPI_GELU_BWD = 5
};
typedef struct delta_conv_epilogue {
  int32_t mode;
  int32_t pool_hw;
  int32_t add_stride2;
  int32_t scatter;
  const void* add;
  const void* add_mask;
  const void* out_mask;
  const void* xc;
  const float* mean;
  const float* invstd;
  const float* gamma;
  const float* beta;
} delta_conv_epilogue;
delta_status delta_conv_forward_ex(const delta_conv* c, const void* x, void* y, float* stats,
                                   const delta_conv_epilogue* epi, void* stream);
/* Override the output-channel tile (64, 128 or 256, dividing K).  The fused
 * epilogues require tile_n <= 128, except DELTA_EPI_BN_BWD (256 allowed). */
delta_status delta_conv_set_tile_n(delta_conv* c, int32_t tile_n);
delta_status delta_conv_geometry(const delta_conv* c, int32_t* P, int32_t* Q, int32_t* kdim,
                                 int32_t* tile_n);
void delta_conv_destroy(delta_conv* c);

/* ---- backward: convolution weight gradient ----
 * dW[k][r][s][c] = sum over output pixels of dY[n,p,q,k] * X[n, p*st-pad+r,
 * q*st-pad+s, c]; fp32 KRSC output (overwritten), deterministic split-K over
 * pixels (tcgen05, MN-major operands): the last split of each tile to land
 * sums the tile's partials in split order (one launch, no atomics on data).
 * C == 4 is the 7x7/2 stem (input channel 3 is the zero pad).  `ws` must hold
 * delta_wgrad_workspace_bytes and be ZEROED once at allocation (it carries
 * self-resetting per-tile split counters); one launch at a time per `ws`. */
typedef struct delta_wgrad delta_wgrad;
delta_status delta_wgrad_create(int32_t N, int32_t H, int32_t W, int32_t C, int32_t K, int32_t R,
                                int32_t S, int32_t stride, int32_t pad, delta_wgrad** out);
uint64_t delta_wgrad_workspace_bytes(const delta_wgrad* w);
/* kernel launches one delta_wgrad_run issues (1, or 2 with a separate split
 * reduce: the stem, and tiles split more than 4-way over the pixels) */
int32_t delta_wgrad_launches(const delta_wgrad* w);
delta_status delta_wgrad_run(const delta_wgrad* w, const void* dy, const void* x, float* dw, void* ws,
                         void* stream);
void delta_wgrad_destroy(delta_wgrad* w);

/* ---- recompute engine: BatchNorm (BNForward, ref src/trace.cpp:405) ---- */
/* BN workspace (floats): a few words of grid-barrier state at its head,
 * then partial rows.  Zero it once at allocation; every kernel leaves the
 * barrier words in a reusable state. */
int64_t delta_bn_workspace_floats(int64_t M, int32_t C);
/* training-mode statistics; run_mean/run_var may be NULL (recompute never
 * touches them) */
delta_status delta_bn_stats(const void* x, int64_t M, int32_t C, float* ws, float* mean,
                            float* invstd, float eps, float* run_mean, float* run_var,
                            float momentum, void* stream);
/* BN statistics from a conv's epilogue partials.  A conv launched with a
 * `stats` buffer writes one partial row per CTA — delta_stats_parts() rows
 * (one CTA per SM) of float4 (count, mean, M2) per channel, merged tile by
 * tile in the CTA's fixed tile order — and one launch reduces the rows in a
 * fixed order.  The buffer holds delta_stats_partials_floats(C) floats. */
int32_t delta_stats_parts(void);
int64_t delta_stats_partials_floats(int32_t C);
delta_status delta_bn_stats_from_partials(const float* partials, int32_t C, float* mean,
                                          float* invstd, float eps, float* run_mean,
                                          float* run_var, float momentum, void* stream);
/* out[c] (=, or += with accumulate) = the column sums of the bf16 outputs a
 * conv launched with a `stats` buffer reduced: sum over the partial rows of
 * count * mean, fixed order (a bias gradient without another pass) */
delta_status delta_stats_col_sum(const float* partials, int32_t C, float* out, int32_t accumulate,
                                 void* stream);
/* mode 0 relu(bn(x)), 1 relu(bn(x)+res), 2 relu(bn(x)+bn2(res)) */
delta_status delta_bn_apply(int32_t mode, const void* x, const void* res, void* y, int64_t M,
                            int32_t C, const float* mean, const float* invstd,
                            const float* gamma, const float* beta, const float* mean2,
                            const float* invstd2, const float* gamma2, const float* beta2,
                            void* stream);
/* Training-mode BN backward (dgamma, dbeta, dx) of g = up [* (mask > 0)]; up
 * full [M][C] or pooled [N][C] / pool_hw.  One persistent launch of
 * co-resident CTAs (a cooperative launch) with two grid-wide barriers
 * (partial sums -> fixed-order per-channel merge -> apply); deterministic.
 * `ws`: delta_bn_workspace_floats floats, zeroed at allocation; the barrier
 * state lives in it, so launches on different streams need different
 * workspaces.  If the cooperative launch is refused, or with
 * DELTA_BN_BWD_GRID=0, the three-launch path runs instead. */
delta_status delta_bn_backward(const void* up, int32_t pool_hw, const void* mask, const void* x,
                               void* dx, int64_t M, int32_t C, const float* mean,
                               const float* invstd, const float* gamma, float* dgamma,
                               float* dbeta, float* ws, void* stream);
/* BN(+ReLU) backward after a DELTA_EPI_BN_BWD conv: `partials` are that
 * conv's per-CTA (sum g, sum g*x) rows (delta_stats_partials_floats(C)
 * floats), g its masked output.  Writes dgamma, dbeta, dx. */
delta_status delta_bn_backward_from_partials(const float* partials, const void* g, const void* x,
                                             void* dx, int64_t M, int32_t C, const float* mean,
                                             const float* invstd, const float* gamma,
                                             float* dgamma, float* dbeta, void* stream);
/* out = (a + up*[up_mask>0]) * [out_mask>0]; null masks are not applied;
 * pool_hw > 0: `up` is [N,C] broadcast over pool_hw pixels / pool_hw */
delta_status delta_add_grad(const void* a, const void* up, int32_t pool_hw, const void* up_mask,
                            const void* out_mask, void* out, int64_t M, int32_t C, void* stream);

/* ---- pooling / head ---- */
delta_status delta_maxpool3x3s2_fwd(const void* x, void* y, int32_t N, int32_t H, int32_t W,
                                    int32_t C, void* stream);
/* `ws`: delta_maxpool_workspace_bytes() of scratch (argmax bytes) */
int64_t delta_maxpool_workspace_bytes(int32_t N, int32_t H, int32_t W, int32_t C);
delta_status delta_maxpool3x3s2_bwd(const void* dy, const void* x, void* dx, int32_t N,
                                    int32_t H, int32_t W, int32_t C, void* ws, void* stream);
delta_status delta_avgpool_fwd(const void* x, void* y, int32_t N, int32_t HW, int32_t C,
                               void* stream);
delta_status delta_softmax_xent(const float* logits, const int64_t* labels, float* loss,
                                float* dlogits, float* row_ws, int32_t N, int32_t K,
                                void* stream);
/* The classifier head after the tensor-core FC GEMM (a 1x1 delta_conv over
 * the pooled features, bf16 logits [N][ld], ld >= K the padded class count):
 * z = logits + bias (fp32); loss = mean_i (logsumexp z_i - z_i[label_i]);
 * dlogits = (softmax(z) - onehot) / N as fp32 [N][K] and as bf16 [N][ld]
 * with zero pad columns (the operand of the head's dgrad and wgrad GEMMs);
 * dbias = column sums of dlogits in row order.  K <= 1024. */
delta_status delta_softmax_xent_head(const void* logits, int32_t ld, const float* bias,
                                     const int64_t* labels, float* loss, float* dlogits,
                                     void* dlogits_bf16, float* dbias, float* row_ws, int32_t N,
                                     int32_t K, void* stream);

/* ---- optimizer step and the per-step weight views (optim.cu) ---- */
/* SGD with momentum and weight decay over flat fp32 buffers (n floats, 16 B
 * aligned): mom = mom*momentum + g + weight_decay*w; w -= lr*mom; and the
 * first n_bf elements of w rounded to bf16 into wbf (the conv weights). */
delta_status delta_sgd_step(float* w, float* mom, const float* g, void* wbf, int64_t n,
                            int64_t n_bf, float lr, float momentum, float weight_decay,
                            void* stream);
/* Derived bf16 weight tensors from bf16 [K][R][S][C] conv weights, one launch
 * for a device-resident table of views:
 *   DELTA_VIEW_DGRAD: dst[c][r][s][k] = src[k][R-1-r][S-1-s][c] (input-gradient
 *                     convs through our kernel)
 *   DELTA_VIEW_STEM:  dst[k][256] pixel-pair stem layout (C = 4, 7x7): column
 *                     (r*4+j)*8 + e*4 + c = src[k][r][2j+e-1][c], zero elsewhere
 *   DELTA_VIEW_DGRAD_S2: (3x3 source) the weights of parity class (a, b) =
 *                     (reserved >> 1, reserved & 1) of the stride-2 input
 *                     gradient: dst[c][r'][s'][k], r' < 1+a, s' < 1+b, =
 *                     src[k][ra(r')][sb(s')][c] with ra = 1 for a = 0 and
 *                     ra(r') = 2 - 2r' for a = 1 (sub-tap r' reads dY row
 *                     i + r'); same for columns */
enum { DELTA_VIEW_DGRAD = 0, DELTA_VIEW_STEM = 1, DELTA_VIEW_DGRAD_S2 = 2 };
typedef struct delta_weight_view {
  int32_t kind, K, R, S, C, reserved;
  const void* src;
  void* dst;
} delta_weight_view;
delta_status delta_weight_views(const delta_weight_view* views_dev, int32_t n_views,
                                void* stream);

/* ---- swap engine (Offload/Reload, ref src/engine.cpp:312-331, 396-419,
 *      533-585): pinned host slab + dedicated copy-engine streams ---- */
typedef struct delta_swap delta_swap;
/* Allocates `host_bytes` of pinned host memory and creates two
 * non-blocking copy streams (D2H, H2D). */
delta_status delta_swap_create(uint64_t host_bytes, delta_swap** out);
void* delta_swap_host_ptr(const delta_swap* s);
void* delta_swap_stream(const delta_swap* s, int32_t which); /* 1 D2H, 2 H2D */
delta_status delta_swap_offload(delta_swap* s, const void* dev, uint64_t host_off,
                                uint64_t bytes, void* stream);
delta_status delta_swap_reload(delta_swap* s, void* dev, uint64_t host_off, uint64_t bytes,
                               void* stream);
void delta_swap_destroy(delta_swap* s);

/* ---- cost model: host-link probe (GB/s) with pinned memory ---- */
delta_status delta_probe_link(uint64_t bytes, int32_t iters, double* h2d_gbs, double* d2h_gbs,
                              double* duplex_gbs);

/* ---- events for program replay ---- */
typedef struct delta_events delta_events;
delta_status delta_events_create(uint32_t n, delta_events** out);
delta_status delta_event_record(delta_events* e, uint32_t i, void* stream);
delta_status delta_event_wait(delta_events* e, uint32_t i, void* stream);
void delta_events_destroy(delta_events* e);

#ifdef __cplusplus
}
#endif
#endif /* DELTA_DELTA_KERNELS_H_ */
