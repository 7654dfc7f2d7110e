// C ABI of the transformer (BERT) kernels (include/delta/delta_xformer.h).
#include <cuda_runtime.h>

#include <string>

#include "delta/delta_xformer.h"
#include "kernels/xformer.hpp"

namespace delta_rt {
void set_error(const std::string& msg);  // capi.cpp
}

namespace {
delta_status st_(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DELTA_OK;
  delta_rt::set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorInvalidValue ? DELTA_E_UNSUPPORTED : DELTA_E_CUDA;
}
inline cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }
}  // namespace

extern "C" {

delta_status delta_layernorm_fwd(const void* x, void* y, float* mean, float* rstd,
                                 const float* gamma, const float* beta, int64_t rows, int32_t H,
                                 float eps, void* stream) {
  return st_(delta_k::layernorm_fwd(x, y, mean, rstd, gamma, beta, rows, H, eps, S(stream)),
             "layernorm_fwd");
}
int64_t delta_layernorm_bwd_workspace_floats(int64_t rows, int32_t H) {
  return delta_k::layernorm_bwd_workspace_floats(rows, H);
}
delta_status delta_layernorm_bwd(const void* dy, const void* x, const void* dres, void* dx,
                                 const float* mean, const float* rstd, const float* gamma,
                                 float* dgamma, float* dbeta, float* ws, int64_t rows, int32_t H,
                                 void* stream) {
  return st_(delta_k::layernorm_bwd(dy, x, dres, dx, mean, rstd, gamma, dgamma, dbeta, ws, rows, H,
                                    S(stream)),
             "layernorm_bwd");
}
delta_status delta_layernorm_bwd_drop(const void* dy, const void* x, const void* dres, void* dx,
                                      const float* mean, const float* rstd, const float* gamma,
                                      float* dgamma, float* dbeta, float* ws, int64_t rows,
                                      int32_t H, void* dxd, float* dbias, float p,
                                      const uint64_t* rng, uint32_t tag, void* stream) {
  return st_(delta_k::layernorm_bwd_drop(dy, x, dres, dx, mean, rstd, gamma, dgamma, dbeta, ws, rows,
                                         H, dxd, dbias, p, rng, tag, S(stream)),
             "layernorm_bwd_drop");
}
delta_status delta_gelu_fwd(const void* x, void* y, int64_t n, void* stream) {
  return st_(delta_k::gelu_fwd(x, y, n, S(stream)), "gelu_fwd");
}
delta_status delta_add_dropout(const void* a, const void* b, void* y, int64_t n, float p,
                               const uint64_t* rng, uint32_t tag, void* stream) {
  return st_(delta_k::add_dropout(a, b, y, n, p, rng, tag, S(stream)), "add_dropout");
}
delta_status delta_dropout_bwd(const void* dy, void* dx, int64_t n, float p, const uint64_t* rng,
                               uint32_t tag, void* stream) {
  return st_(delta_k::dropout_bwd(dy, dx, n, p, rng, tag, S(stream)), "dropout_bwd");
}
int64_t delta_colsum_workspace_floats(int64_t rows, int32_t cols) {
  return delta_k::colsum_workspace_floats(rows, cols);
}
delta_status delta_colsum(const void* x, int64_t rows, int32_t cols, const int32_t* sel,
                          int32_t sel_val, float* out, float* ws, int32_t accumulate,
                          void* stream) {
  return st_(delta_k::colsum(x, rows, cols, sel, sel_val, out, ws, accumulate, S(stream)),
             "colsum");
}
delta_status delta_embed_fwd(const int32_t* ids, const int32_t* types, const void* word,
                             const void* pos, const void* type, void* y, int32_t B, int32_t S_,
                             int32_t H, float p, const uint64_t* rng, uint32_t tag, void* stream) {
  return st_(delta_k::embed_fwd(ids, types, word, pos, type, y, B, S_, H, p, rng, tag, S(stream)),
             "embed_fwd");
}
delta_status delta_embed_grads(const void* dsum, const int32_t* csr, const int32_t* types,
                               int32_t B, int32_t S_, int32_t H, int32_t vocab, int32_t n_types,
                               float* dword, float* dpos, float* dtype, float* ws, void* stream) {
  return st_(delta_k::embed_grads(dsum, csr, types, B, S_, H, vocab, n_types, dword, dpos, dtype, ws,
                                  S(stream)),
             "embed_grads");
}
delta_status delta_span_head_fwd(const void* h, const float* w, const float* bias,
                                 const int32_t* label, float* logits, float* dlogits,
                                 float* row_loss, float* loss, int32_t B, int32_t S_, int32_t H,
                                 void* stream) {
  return st_(delta_k::span_head_fwd(h, w, bias, label, logits, dlogits, row_loss, loss, B, S_, H,
                                    S(stream)),
             "span_head_fwd");
}
int64_t delta_span_head_workspace_floats(int64_t T, int32_t H) {
  return delta_k::span_head_workspace_floats(T, H);
}
delta_status delta_span_head_bwd(const void* h, const float* dlogits, const float* w, void* dh,
                                 float* dw, float* dbias, float* ws, int64_t T, int32_t H,
                                 void* stream) {
  return st_(delta_k::span_head_bwd(h, dlogits, w, dh, dw, dbias, ws, T, H, S(stream)),
             "span_head_bwd");
}
delta_status delta_attention_fwd(const void* qkv, void* out, float* lse, int32_t B, int32_t S_,
                                 int32_t heads, float p, const uint64_t* rng, uint32_t tag,
                                 void* stream) {
  return st_(delta_k::attention_fwd(qkv, out, lse, B, S_, heads, p, rng, tag, S(stream)),
             "attention_fwd");
}
delta_status delta_attention_bwd(const void* qkv, const void* out, const void* dout,
                                 const float* lse, float* D, void* dqkv, int32_t B, int32_t S_,
                                 int32_t heads, float p, const uint64_t* rng, uint32_t tag,
                                 float* dbias, float* ws, void* stream) {
  return st_(delta_k::attention_bwd(qkv, out, dout, lse, D, dqkv, B, S_, heads, p, rng, tag, dbias,
                                    ws, S(stream)),
             "attention_bwd");
}
delta_status delta_attention_debug(void* host_words) {
  return st_(delta_k::attention_debug(host_words), "attention_debug");
}
delta_status delta_parts_merge(const float* ws, int32_t parts, int32_t cols, float* out,
                               void* stream) {
  if (parts <= 0 || cols <= 0) {
    delta_rt::set_error("parts_merge: empty");
    return DELTA_E_ARGUMENT;
  }
  return st_(delta_k::merge_parts(ws, parts, cols, out, S(stream)), "parts_merge");
}
delta_status delta_adamw_step(float* w, float* m, float* v, const float* g, void* wbf, int64_t n,
                              int64_t n_bf, float lr, float beta1, float beta2, float eps,
                              float weight_decay, uint64_t* rng, void* stream) {
  return st_(delta_k::adamw_step(w, m, v, g, wbf, n, n_bf, lr, beta1, beta2, eps, weight_decay, rng,
                                 S(stream)),
             "adamw_step");
}

}  // extern "C"
