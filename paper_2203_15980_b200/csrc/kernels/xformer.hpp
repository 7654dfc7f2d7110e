// Internal launch interface of the transformer (BERT) kernels: xformer.cu
// (HBM-bound ops) and attention.cu (tcgen05 attention).  Wrapped by the C ABI
// in rt/xformer_capi.cpp (include/delta/delta_xformer.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace delta_k {

// activations: bf16 [rows][H] row-major, H a multiple of 256 (<= 1024 for
// the LayerNorm backward and the span head)
cudaError_t layernorm_fwd(const void* x, void* y, float* mean, float* rstd, const float* gamma,
                          const float* beta, int64_t rows, int H, float eps, cudaStream_t st);
int64_t layernorm_bwd_workspace_floats(int64_t rows, int H);
cudaError_t layernorm_bwd(const void* dy, const void* x, const void* dres, void* dx,
                          const float* mean, const float* rstd, const float* gamma, float* dgamma,
                          float* dbeta, float* ws, int64_t rows, int H, cudaStream_t st);
// the same, and the gradient through the dropout(p, tag) of the residual
// branch feeding this LayerNorm: dxd = mask * scale * dx (bf16), dbias = its
// column sums (the branch's bias gradient, overwritten)
cudaError_t layernorm_bwd_drop(const void* dy, const void* x, const void* dres, void* dx,
                               const float* mean, const float* rstd, const float* gamma,
                               float* dgamma, float* dbeta, float* ws, int64_t rows, int H,
                               void* dxd, float* dbias, float p, const uint64_t* rng, uint32_t tag,
                               cudaStream_t st);
cudaError_t gelu_fwd(const void* x, void* y, int64_t n, cudaStream_t st);
cudaError_t add_dropout(const void* a, const void* b, void* y, int64_t n, float p,
                        const uint64_t* rng, uint32_t tag, cudaStream_t st);
cudaError_t dropout_bwd(const void* dy, void* dx, int64_t n, float p, const uint64_t* rng,
                        uint32_t tag, cudaStream_t st);
int64_t colsum_workspace_floats(int64_t rows, int cols);
cudaError_t colsum(const void* x, int64_t rows, int cols, const int32_t* sel, int sel_val,
                   float* out, float* ws, int accumulate, cudaStream_t st);
cudaError_t embed_fwd(const int32_t* ids, const int32_t* types, const void* word, const void* pos,
                      const void* type, void* y, int B, int S, int H, float p, const uint64_t* rng,
                      uint32_t tag, cudaStream_t st);
cudaError_t embed_grads(const void* dsum, const int32_t* csr, const int32_t* types, int B, int S,
                        int H, int vocab, int n_types, float* dword, float* dpos, float* dtype,
                        float* ws, cudaStream_t st);
cudaError_t span_head_fwd(const void* h, const float* w, const float* bias, const int32_t* label,
                          float* logits, float* dlogits, float* row_loss, float* loss, int B,
                          int S, int H, cudaStream_t st);
int64_t span_head_workspace_floats(int64_t T, int H);
cudaError_t span_head_bwd(const void* h, const float* dlogits, const float* w, void* dh, float* dw,
                          float* dbias, float* ws, int64_t T, int H, cudaStream_t st);
cudaError_t attn_dvec(const void* o, const void* dout, int64_t T, int S, int heads, float* D,
                      cudaStream_t st);
// out[c] = sum over p < parts of ws[p * cols + c], in order of p
cudaError_t merge_parts(const float* ws, int parts, int cols, float* out, cudaStream_t st);
cudaError_t adamw_step(float* w, float* m, float* v, const float* g, void* wbf, int64_t n,
                       int64_t n_bf, float lr, float b1, float b2, float eps, float wd,
                       uint64_t* rng, cudaStream_t st);

// attention.cu: softmax(Q K^T / sqrt(64)) with dropout, V; head dim 64,
// S a multiple of 128 and <= 512.  qkv [B*S][3*heads*64] (Q | K | V, head h
// at columns h*64 of each third); out [B*S][heads*64]; lse [B*heads][S] in
// log2 units of the scaled scores.
cudaError_t attention_fwd(const void* qkv, void* out, float* lse, int B, int S, int heads,
                          float p, const uint64_t* rng, uint32_t tag, cudaStream_t st);
// debug: progress words of the backward kernel in mapped host memory (32 per CTA)
cudaError_t attention_debug(void* host_words);
// dqkv [B*S][3*heads*64]; D = rowsum(dO * O) scratch [B*heads][S]; if dbias
// (fp32 [3*heads*64], overwritten): the column sums of dqkv, per-sequence
// partials in ws [B][3*heads*64] merged in sequence order
cudaError_t attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                          float* D, void* dqkv, int B, int S, int heads, float p,
                          const uint64_t* rng, uint32_t tag, float* dbias, float* ws,
                          cudaStream_t st);

}  // namespace delta_k
