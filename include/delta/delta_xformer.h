/* delta-b200 C ABI — the transformer (BERT) side of the recompute engine.
 *
 * The reference's transformer trace (src/trace.cpp:422-466,
 * gen_transformer_like) registers per layer LayerNorm1, QKVProj, Attention,
 * OutProj, AddResid1, LayerNorm2, MlpUp, MlpDown, AddResid2 behind an
 * uncomputable Embedding; its OpNode::compute_cost_us (trace.hpp:17) stands in
 * for the op.  These are the real ops on a B200, all re-runnable with
 * bit-identical output (the recompute engine's contract, ref
 * src/engine.cpp:423-454):
 *   - linear layers: delta_conv 1x1 over [tokens][features] with
 *     DELTA_EPI_BIAS / DELTA_EPI_GELU_BWD (delta_kernels.h), weight gradients
 *     with delta_wgrad, bias gradients with delta_colsum;
 *   - attention: tcgen05 kernels (S <= 512, head dim 64) with dropout;
 *   - LayerNorm, GELU, residual add + dropout, embeddings, the SQuAD span
 *     head, AdamW: HBM-bound kernels.
 * Dropout masks are counter-based (Philox4x32-10): element e of site `tag`
 * in step `step` is kept iff byte (e mod 16) of Philox((e/16, tag, step),
 * seed) >= round(256 p), with rng = device pointer to {seed, step}; a
 * recompute (same step) redraws the same mask.  The drop probability is thus
 * quantised to 1/256 (scale = 256 / (256 - round(256 p))).
 * Activations are bf16 row-major [rows][H]; H a multiple of 256 (<= 1024 for
 * LayerNorm backward and the span head).  All calls are asynchronous on
 * `stream`; deterministic (fixed-order reductions, no atomics). */
#ifndef DELTA_DELTA_XFORMER_H_
#define DELTA_DELTA_XFORMER_H_

#include <stdint.h>

#include "delta/delta.h"

#ifdef __cplusplus
extern "C" {
#endif

/* y = (x - mean) * rstd * gamma + beta per row; mean/rstd saved (fp32 [rows]) */
delta_status delta_layernorm_fwd(const void* x, void* y, float* mean, float* rstd,
                                 const float* gamma, const float* beta, int64_t rows, int32_t H,
                                 float eps, void* stream);
int64_t delta_layernorm_bwd_workspace_floats(int64_t rows, int32_t H);
/* dx = LN-backward(dy) (+ dres if non-null: the residual branch's gradient);
 * dgamma, dbeta overwritten; ws: delta_layernorm_bwd_workspace_floats */
delta_status delta_layernorm_bwd(const void* dy, const void* x, const void* dres, void* dx,
                                 const float* mean, const float* rstd, const float* gamma,
                                 float* dgamma, float* dbeta, float* ws, int64_t rows, int32_t H,
                                 void* stream);
/* delta_layernorm_bwd, and the gradient through the dropout (p, tag) of the
 * residual branch that fed this LayerNorm's input, in the same pass:
 * dxd = dropout mask * scale * dx (bf16, the mask of delta_add_dropout(tag))
 * and dbias = its column sums (fp32 [H], overwritten: that branch's bias
 * gradient).  ws: delta_layernorm_bwd_workspace_floats. */
delta_status delta_layernorm_bwd_drop(const void* dy, const void* x, const void* dres, void* dx,
                                      const float* mean, const float* rstd, const float* gamma,
                                      float* dgamma, float* dbeta, float* ws, int64_t rows,
                                      int32_t H, void* dxd, float* dbias, float p,
                                      const uint64_t* rng, uint32_t tag, void* stream);
/* y = x * Phi(x) (erf GELU), n a multiple of 8 */
delta_status delta_gelu_fwd(const void* x, void* y, int64_t n, void* stream);
/* y = a + dropout(b) (n a multiple of 16) — AddResid */
delta_status delta_add_dropout(const void* a, const void* b, void* y, int64_t n, float p,
                               const uint64_t* rng, uint32_t tag, void* stream);
/* dx = dropout mask * scale * dy, the same mask as delta_add_dropout(tag) */
delta_status delta_dropout_bwd(const void* dy, void* dx, int64_t n, float p, const uint64_t* rng,
                               uint32_t tag, void* stream);
int64_t delta_colsum_workspace_floats(int64_t rows, int32_t cols);
/* out[c] (=|+=) sum over rows r (with sel[r] == sel_val if sel) of x[r][c] */
delta_status delta_colsum(const void* x, int64_t rows, int32_t cols, const int32_t* sel,
                          int32_t sel_val, float* out, float* ws, int32_t accumulate,
                          void* stream);
/* y[t] = dropout(word[ids[t]] + pos[t % S] + type[types[t]]) (bf16 tables) */
delta_status delta_embed_fwd(const int32_t* ids, const int32_t* types, const void* word,
                             const void* pos, const void* type, void* y, int32_t B, int32_t S,
                             int32_t H, float p, const uint64_t* rng, uint32_t tag, void* stream);
/* Embedding-table gradients (fp32, overwritten) from dsum = the gradient of
 * the pre-dropout sum.  csr (int32, built by the host with the batch): [0] =
 * U unique ids, [1, 1+T) the ids, [1+T, 2+2T) segment offsets, [2+2T, 2+3T)
 * token indices grouped by id (ascending within a group).  ws:
 * delta_colsum_workspace_floats(T, H). */
delta_status delta_embed_grads(const void* dsum, const int32_t* csr, const int32_t* types,
                               int32_t B, int32_t S, int32_t H, int32_t vocab, int32_t n_types,
                               float* dword, float* dpos, float* dtype, float* ws, void* stream);
/* SQuAD span head: logits [T][2] = h . w^T + bias (w fp32 [2][H]); loss =
 * mean over sequences of (CE(start) + CE(end)) / 2 over the S positions
 * (label [B][2]); dlogits fp32 [T][2]; row_loss fp32 [B] */
delta_status delta_span_head_fwd(const void* h, const float* w, const float* bias,
                                 const int32_t* label, float* logits, float* dlogits,
                                 float* row_loss, float* loss, int32_t B, int32_t S, int32_t H,
                                 void* stream);
int64_t delta_span_head_workspace_floats(int64_t T, int32_t H);
/* dh = dlogits . w (bf16 [T][H]); dw [2][H], dbias [2] overwritten */
delta_status delta_span_head_bwd(const void* h, const float* dlogits, const float* w, void* dh,
                                 float* dw, float* dbias, float* ws, int64_t T, int32_t H,
                                 void* stream);
/* attention over qkv [B*S][3*heads*64] (Q | K | V thirds, head h at columns
 * h*64 of each) -> out [B*S][heads*64]; lse fp32 [B*heads][S] saved for the
 * backward.  S a multiple of 128, <= 512; dropout p on the probabilities. */
delta_status delta_attention_fwd(const void* qkv, void* out, float* lse, int32_t B, int32_t S,
                                 int32_t heads, float p, const uint64_t* rng, uint32_t tag,
                                 void* stream);
/* dqkv [B*S][3*heads*64] from dout; D: fp32 [B*heads][S] scratch.  dbias
 * (optional, fp32 [3*heads*64], overwritten): the column sums of dqkv — the
 * QKV projection's bias gradient — reduced inside the kernel per sequence
 * into ws (fp32 [B][3*heads*64]) and merged in sequence order. */
delta_status delta_attention_bwd(const void* qkv, const void* out, const void* dout,
                                 const float* lse, float* D, void* dqkv, int32_t B, int32_t S,
                                 int32_t heads, float p, const uint64_t* rng, uint32_t tag,
                                 float* dbias, float* ws, void* stream);
/* debugging aid (libraries built with -DDELTA_ATTN_DEBUG; a no-op
 * otherwise): the backward kernel writes progress words (32 per CTA) to this
 * mapped host buffer (NULL = off) */
delta_status delta_attention_debug(void* host_words);
/* out[c] = sum over p < parts of ws[p * cols + c], summed in order of p
 * (partial rows of a column reduction, e.g. DELTA_EPI_GELU_BWD's) */
delta_status delta_parts_merge(const float* ws, int32_t parts, int32_t cols, float* out,
                               void* stream);
/* AdamW over flat fp32 buffers (decoupled weight decay on the first n_bf
 * elements, which are also written as bf16 to wbf), bias correction with step
 * rng[1] + 1; then rng[1] += 1 (the next step's dropout masks). */
delta_status delta_adamw_step(float* w, float* m, float* v, const float* g, void* wbf, int64_t n,
                              int64_t n_bf, float lr, float beta1, float beta2, float eps,
                              float weight_decay, uint64_t* rng, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DELTA_DELTA_XFORMER_H_ */
