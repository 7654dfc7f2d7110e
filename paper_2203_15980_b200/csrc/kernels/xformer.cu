// Transformer (BERT) ops of the recompute engine, the layers of the
// reference's transformer trace (ref src/trace.cpp:422-466: Embedding,
// LayerNorm1/2, QKVProj, Attention, OutProj, AddResid1/2, MlpUp, MlpDown).
// The linear layers are the tcgen05 GEMM (conv_fwd.cu, a 1x1 conv over the
// [tokens][features] matrix, bias / GELU-backward epilogues) and attention is
// attention.cu; this file holds the HBM-bound rest:
//
//   k_layernorm_fwd / k_layernorm_bwd(+merge)  one warp per row, two-pass
//       statistics in registers; per-CTA (dgamma, dbeta) partial rows merged
//       in a fixed order (deterministic, so a recomputed LayerNorm output and
//       the step's gradients reproduce bit for bit)
//   k_gelu_fwd                                 erf GELU (BERT), the Gelu node
//   k_add_dropout / k_dropout_bwd              AddResid = x + dropout(y), masks
//       from philox.cuh (replayed on recompute and in the backward pass)
//   k_colsum(+merge)                           bias gradients (column sums),
//       optionally over the rows of one token type
//   k_embed_*                                  word + position + type gather,
//       dropout; the word-embedding gradient as a segmented sum over a host-
//       built CSR of the batch's token ids (no atomics)
//   k_span_head_*                              SQuAD span head: start/end
//       logits, the per-sequence softmax cross-entropy and its backward
//   k_attn_dvec                                D = rowsum(dO * O), attention
//       backward preprocessing
//   k_adamw / k_rng_advance                    AdamW over the flat fp32
//       buffers (+ bf16 weight copies), then the dropout step counter
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels/gelu.cuh"
#include "kernels/launch.hpp"
#include "kernels/philox.cuh"
#include "kernels/sm100_common.cuh"
#include "kernels/xformer.hpp"

namespace delta_k {

namespace {

using namespace dsm100;
using bf16 = __nv_bfloat16;

__device__ __forceinline__ void unpack8(uint4 u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint32_t pk2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint4 pack8(const float* f) {
  return make_uint4(pk2(f[0], f[1]), pk2(f[2], f[3]), pk2(f[4], f[5]), pk2(f[6], f[7]));
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

int g_sms = 0;
int sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

// ---------------------------------------------------------------- LayerNorm
// Row r = one warp; lane owns NV 16-byte chunks at columns (v*32 + lane)*8.
// Warp w of block b takes rows b*8 + w + i*(8*gridDim), each arriving by a
// bulk copy (TMA) LNF_ST rows ahead into the warp's shared-memory stages;
// gamma / beta are staged once per block.
constexpr int LNF_ST = 3;
template <int NV>
constexpr size_t ln_fwd_smem() {
  return size_t(NV) * 256 * 8 + size_t(8) * LNF_ST * NV * 256 * 2;
}
template <int NV>
__global__ void __launch_bounds__(256)
    k_layernorm_fwd(const bf16* __restrict__ x, bf16* __restrict__ y, float* __restrict__ mean,
                    float* __restrict__ rstd, const float* __restrict__ gamma,
                    const float* __restrict__ beta, int64_t rows, float eps) {
  constexpr int H = NV * 256;
  constexpr uint32_t RB = H * 2;
  extern __shared__ __align__(128) uint8_t lnf_smem[];
  __shared__ uint64_t bar[8][LNF_ST];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* sg = reinterpret_cast<float*>(lnf_smem);
  float* sb = sg + H;
  uint8_t* stage0 = lnf_smem + H * 8 + size_t(warp) * LNF_ST * RB;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < LNF_ST; ++s) mbar_init(&bar[warp][s], 1);
    fence_mbar_init();
  }
  pdl_wait();
  pdl_trigger();
  for (int c = threadIdx.x; c < H; c += 256) {
    sg[c] = __ldg(gamma + c);
    sb[c] = __ldg(beta + c);
  }
  __syncthreads();
  const int64_t stride = int64_t(gridDim.x) * 8;
  const int64_t r0 = int64_t(blockIdx.x) * 8 + warp;
  const int n = r0 < rows ? int((rows - r0 + stride - 1) / stride) : 0;
  auto issue = [&](int it) {
    uint64_t* b = &bar[warp][it % LNF_ST];
    mbar_arrive_expect_tx(b, RB);
    bulk_load(smem_u32(stage0 + size_t(it % LNF_ST) * RB), x + (r0 + it * stride) * H, RB, b);
  };
  if (lane == 0)
    for (int it = 0; it < min(n, LNF_ST); ++it) issue(it);
  for (int it = 0; it < n; ++it) {
    const int64_t r = r0 + it * stride;
    const int s = it % LNF_ST;
    mbar_wait(&bar[warp][s], uint32_t(it / LNF_ST) & 1u);
    const uint4* sx = reinterpret_cast<const uint4*>(stage0 + size_t(s) * RB);
    float v[NV][8];
#pragma unroll
    for (int k = 0; k < NV; ++k) unpack8(sx[k * 32 + lane], v[k]);
    __syncwarp();  // the row is in registers: refill its stage
    if (lane == 0 && it + LNF_ST < n) issue(it + LNF_ST);
    float sum = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) sum += v[k][i];
    const float mu = warp_sum(sum) * (1.f / H);
    float q = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = v[k][i] - mu;
        q = fmaf(d, d, q);
      }
    const float rs = rsqrtf(warp_sum(q) * (1.f / H) + eps);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int c = (k * 32 + lane) * 8;
      float g[8], b[8], o[8];
      *reinterpret_cast<float4*>(g) = *reinterpret_cast<const float4*>(sg + c);
      *reinterpret_cast<float4*>(g + 4) = *reinterpret_cast<const float4*>(sg + c + 4);
      *reinterpret_cast<float4*>(b) = *reinterpret_cast<const float4*>(sb + c);
      *reinterpret_cast<float4*>(b + 4) = *reinterpret_cast<const float4*>(sb + c + 4);
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = fmaf((v[k][i] - mu) * rs, g[i], b[i]);
      reinterpret_cast<uint4*>(y + r * H)[k * 32 + lane] = pack8(o);
    }
    if (lane == 0) {
      mean[r] = mu;
      rstd[r] = rs;
    }
  }
}

// The optional second output of the LayerNorm backward: the gradient that
// flows on through the dropout of the residual branch feeding this
// LayerNorm's input (dxd = mask * scale * bf16(dx), the same mask as
// add_dropout(tag)), whose column sums are that branch's bias gradient.
struct LnDrop {
  bf16* dxd;
  uint32_t thr;
  float scale;
  const uint64_t* rng;
  uint32_t tag;
};

// dx = rstd * (g - mean(g) - xhat * mean(g * xhat)) + dres, g = dy * gamma.
// Block b owns rows [b*chunk, (b+1)*chunk), one row per warp at a time (warps
// interleaved).  The rows a warp reads (dy, x, dres: 2 KB each at H = 1024)
// arrive by bulk copies (TMA) LN_ST rows ahead into the warp's own shared-
// memory stages, so every warp keeps several rows of loads in flight without
// holding them in registers; the two passes over a row (its statistics, then
// dx) both read the staged row.  Each block writes one partial row per reduced
// quantity (sum dy*xhat, sum dy[, sum dxd]) per column to ws[b][NQ][H].
constexpr int LN_ST = 3;
template <int NV>
constexpr size_t ln_bwd_smem() {
  return size_t(NV) * 256 * 4 + size_t(8) * LN_ST * 3 * NV * 256 * 2;
}

template <int NV, bool DROP>
__global__ void __launch_bounds__(256, 1)
    k_layernorm_bwd(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                    const bf16* __restrict__ dres, bf16* __restrict__ dx,
                    const float* __restrict__ mean, const float* __restrict__ rstd,
                    const float* __restrict__ gamma, float* __restrict__ ws, int64_t rows,
                    int64_t chunk, const LnDrop dr) {
  constexpr int H = NV * 256;
  constexpr uint32_t RB = H * 2;  // bytes per bf16 row
  constexpr int NQ = DROP ? 3 : 2;
  extern __shared__ __align__(128) uint8_t ln_smem[];
  __shared__ float red[8][NQ][256];  // per warp, per chunk pass
  __shared__ uint64_t bar[8][LN_ST];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* sgam = reinterpret_cast<float*>(ln_smem);
  uint8_t* stage0 = ln_smem + H * 4 + size_t(warp) * LN_ST * 3 * RB;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < LN_ST; ++s) mbar_init(&bar[warp][s], 1);
    fence_mbar_init();
  }
  pdl_wait();
  pdl_trigger();
  for (int c = threadIdx.x; c < H; c += 256) sgam[c] = __ldg(gamma + c);
  __syncthreads();

  float acc_g[NV][8], acc_b[NV][8], acc_d[DROP ? NV : 1][8];
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc_g[k][i] = acc_b[k][i] = 0.f;
#pragma unroll
  for (int k = 0; k < (DROP ? NV : 1); ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc_d[k][i] = 0.f;
  uint64_t seed = 0, step = 0;
  if (DROP) seed = dr.rng[0], step = dr.rng[1];

  const int64_t rbeg = int64_t(blockIdx.x) * chunk + warp;
  const int64_t rend = min(rows, int64_t(blockIdx.x + 1) * chunk);
  const int n = rbeg < rend ? int((rend - rbeg + 7) / 8) : 0;
  const uint32_t nbytes = (dres ? 3 : 2) * RB;
  auto issue = [&](int it) {
    const int s = it % LN_ST;
    const int64_t r = rbeg + 8 * int64_t(it);
    uint64_t* b = &bar[warp][s];
    const uint32_t d = smem_u32(stage0 + size_t(s) * 3 * RB);
    mbar_arrive_expect_tx(b, nbytes);
    bulk_load(d, dy + r * H, RB, b);
    bulk_load(d + RB, x + r * H, RB, b);
    if (dres) bulk_load(d + 2 * RB, dres + r * H, RB, b);
  };
  if (lane == 0)
    for (int it = 0; it < min(n, LN_ST); ++it) issue(it);

  float mu_l = 0.f, rs_l = 0.f;  // lane j: mean / rstd of row it + j of the next 32
  for (int it = 0; it < n; ++it) {
    const int64_t r = rbeg + 8 * int64_t(it);
    const int s = it % LN_ST;
    if ((it & 31) == 0 && it + lane < n) {
      mu_l = __ldg(mean + r + 8 * lane);
      rs_l = __ldg(rstd + r + 8 * lane);
    }
    const float mu = __shfl_sync(0xFFFFFFFFu, mu_l, it & 31);
    const float rs = __shfl_sync(0xFFFFFFFFu, rs_l, it & 31);
    mbar_wait(&bar[warp][s], uint32_t(it / LN_ST) & 1u);
    const uint4* sdy = reinterpret_cast<const uint4*>(stage0 + size_t(s) * 3 * RB);
    const uint4* sx = sdy + RB / 16;
    const uint4* sres = sdy + 2 * (RB / 16);
    float sg = 0.f, sgx = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float d[8], xv[8], gm[8];
      unpack8(sdy[k * 32 + lane], d);
      unpack8(sx[k * 32 + lane], xv);
      const float4* gp = reinterpret_cast<const float4*>(sgam + (k * 32 + lane) * 8);
      *reinterpret_cast<float4*>(gm) = gp[0];
      *reinterpret_cast<float4*>(gm + 4) = gp[1];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (xv[i] - mu) * rs;
        const float g = d[i] * gm[i];
        sg += g;
        sgx = fmaf(g, xh, sgx);
        acc_g[k][i] = fmaf(d[i], xh, acc_g[k][i]);
        acc_b[k][i] += d[i];
      }
    }
    const float a = warp_sum(sg) * (1.f / H);
    const float b = warp_sum(sgx) * (1.f / H);
    // dropout keep bits of this lane's 8 columns per chunk k: element
    // e = r*H + (k*32 + lane)*8 is in Philox block r*H/16 + k*16 + lane/2,
    // half lane & 1.  Lanes 2m and 2m+1 share each block: each draws the
    // block of one chunk of a chunk pair and they swap.
    // dropout keep masks of this lane's 8 columns per chunk k (2 words of byte
    // masks): element e = r*H + (k*32 + lane)*8 is in Philox block
    // r*H/16 + k*16 + lane/2, half lane & 1.  Lanes 2m and 2m+1 share each
    // block: each draws the block of one chunk of a chunk pair and they swap
    // the halves the other needs.
    uint2 keep[DROP ? NV : 1];
    if (DROP) {
      const uint64_t blk0 = uint64_t(r) * (H / 16) + uint64_t(lane >> 1);
      const int odd = lane & 1;
      const uint4 all = make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
      for (int k = 0; k + 1 < NV; k += 2) {
        const uint4 mine =
            dr.thr ? keep_mask_bytes(drop_block(seed, step, dr.tag, blk0 + uint64_t(k + odd) * 16),
                                     dr.thr)
                   : all;
        // even lane: block k (keeps words 0,1; sends 2,3); odd: block k+1 (keeps 2,3; sends 0,1)
        const uint32_t s0 = odd ? mine.x : mine.z, s1 = odd ? mine.y : mine.w;
        const uint32_t g0 = __shfl_xor_sync(0xFFFFFFFFu, s0, 1);
        const uint32_t g1 = __shfl_xor_sync(0xFFFFFFFFu, s1, 1);
        keep[DROP ? k : 0] = odd ? make_uint2(g0, g1) : make_uint2(mine.x, mine.y);
        keep[DROP ? k + 1 : 0] = odd ? make_uint2(mine.z, mine.w) : make_uint2(g0, g1);
      }
      if (NV & 1) {
        const uint4 w =
            dr.thr ? keep_mask_bytes(drop_block(seed, step, dr.tag, blk0 + uint64_t(NV - 1) * 16),
                                     dr.thr)
                   : all;
        keep[DROP ? NV - 1 : 0] = odd ? make_uint2(w.z, w.w) : make_uint2(w.x, w.y);
      }
    }
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float d[8], xv[8], gm[8], rr[8], o[8];
      unpack8(sdy[k * 32 + lane], d);
      unpack8(sx[k * 32 + lane], xv);
      const float4* gp = reinterpret_cast<const float4*>(sgam + (k * 32 + lane) * 8);
      *reinterpret_cast<float4*>(gm) = gp[0];
      *reinterpret_cast<float4*>(gm + 4) = gp[1];
      if (dres) {
        unpack8(sres[k * 32 + lane], rr);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) rr[i] = 0.f;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float xh = (xv[i] - mu) * rs;
        o[i] = fmaf(rs, d[i] * gm[i] - a - xh * b, rr[i]);
      }
      const uint4 packed = pack8(o);
      reinterpret_cast<uint4*>(dx + r * H)[k * 32 + lane] = packed;
      if (DROP) {
        float q[8];
        unpack8(packed, q);  // the stored (bf16) gradient, as a separate pass would read it
#pragma unroll
        for (int i = 0; i < 8; ++i)
          q[i] = __uint_as_float(__float_as_uint(q[i] * dr.scale) &
                                 keep_mask_elem(i < 4 ? keep[DROP ? k : 0].x : keep[DROP ? k : 0].y,
                                                i & 3));
        const uint4 pd = pack8(q);
        reinterpret_cast<uint4*>(dr.dxd + r * H)[k * 32 + lane] = pd;
        unpack8(pd, q);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc_d[DROP ? k : 0][i] += q[i];
      }
    }
    __syncwarp();  // every lane has read stage s: refill it
    if (lane == 0 && it + LN_ST < n) issue(it + LN_ST);
  }
  // fixed-order reduction over the 8 warps, 256 columns at a time
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      red[warp][0][lane * 8 + i] = acc_g[k][i];
      red[warp][1][lane * 8 + i] = acc_b[k][i];
      if (DROP) red[warp][NQ - 1][lane * 8 + i] = acc_d[DROP ? k : 0][i];
    }
    __syncthreads();
    for (int t = threadIdx.x; t < NQ * 256; t += 256) {
      const int which = t >> 8, c = t & 255;
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += red[w][which][c];
      // column (k*32 + c/8)*8 + c%8 of the row
      ws[(int64_t(blockIdx.x) * NQ + which) * H + k * 256 + c] = s;
    }
    __syncthreads();
  }
}

// out[c] (=|+=) sum over p < parts of ws[p * pstride + c], in p order: block
// = 32 columns x 8 warps, warp w sums parts w, w+8, ... (coalesced 128-byte
// rows), the 8 warp sums combined in warp order (deterministic)
__global__ void __launch_bounds__(256)
    k_parts_merge(const float* __restrict__ ws, int parts, int64_t pstride, int cols,
                  float* __restrict__ out, int accumulate, int64_t ws_y, float* __restrict__ out_y,
                  float* __restrict__ out_z) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.y) {
    ws += ws_y * blockIdx.y;
    out = blockIdx.y == 1 ? out_y : out_z;
  }
  __shared__ float red[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (c < cols) {
    // four loads in flight, summed in the same order as one at a time
    int p = w;
    for (; p + 24 < parts; p += 32) {
      const float a0 = ws[int64_t(p) * pstride + c], a1 = ws[int64_t(p + 8) * pstride + c];
      const float a2 = ws[int64_t(p + 16) * pstride + c], a3 = ws[int64_t(p + 24) * pstride + c];
      s += a0;
      s += a1;
      s += a2;
      s += a3;
    }
    for (; p < parts; p += 8) s += ws[int64_t(p) * pstride + c];
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < cols) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += red[k][lane];
    out[c] = accumulate ? out[c] + t : t;
  }
}

// out (and with out_y, a second merge: ws + ws_y -> out_y; with out_z a third,
// ws + 2 ws_y -> out_z) in one launch
cudaError_t parts_merge(const float* ws, int parts, int64_t pstride, int cols, float* out,
                        int accumulate, cudaStream_t st, int64_t ws_y = 0, float* out_y = nullptr,
                        float* out_z = nullptr) {
  return launch_k(k_parts_merge, dim3((cols + 31) / 32, out_z ? 3 : out_y ? 2 : 1), dim3(256), 0,
                  st, ws, parts, pstride, cols, out, accumulate, ws_y, out_y, out_z);
}

// ---------------------------------------------------------------- GELU
__global__ void __launch_bounds__(256)
    k_gelu_fwd(const uint4* __restrict__ x, uint4* __restrict__ y, int64_t n8) {
  pdl_wait();
  pdl_trigger();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += int64_t(gridDim.x) * blockDim.x) {
    float v[8];
    unpack8(__ldg(x + i), v);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = gelu_fwd1(v[k]);
    y[i] = pack8(v);
  }
}

// ---------------------------------------------------------------- dropout
// thread = one Philox block = 16 elements (two 16-byte vectors)
template <bool BWD>
__global__ void __launch_bounds__(256)
    k_dropout(const uint4* __restrict__ a, const uint4* __restrict__ b, uint4* __restrict__ y,
              int64_t n16, uint32_t thr, float scale, const uint64_t* __restrict__ rng,
              uint32_t tag) {
  pdl_wait();
  pdl_trigger();
  const uint64_t seed = rng[0], step = rng[1];
  for (int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; g < n16;
       g += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t keep = thr ? keep16(drop_block(seed, step, tag, uint64_t(g)), thr) : 0xFFFFu;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float vb[8], o[8];
      unpack8(__ldg(b + 2 * g + h), vb);
      if (BWD) {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = (keep >> (h * 8 + i)) & 1u ? vb[i] * scale : 0.f;
      } else {
        float va[8];
        unpack8(__ldg(a + 2 * g + h), va);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          o[i] = (keep >> (h * 8 + i)) & 1u ? fmaf(vb[i], scale, va[i]) : va[i];
      }
      y[2 * g + h] = pack8(o);
    }
  }
}

// ---------------------------------------------------------------- column sums
// ws[part][cols]: part p sums rows [p*chunk, (p+1)*chunk) (rows with
// sel[r] == sel_val only, when sel is given); thread = 8 columns.
// thread (g, c8): 8 columns c8*8.., rows r0 + g, r0 + g + RG, ... of the
// block's chunk (RG = 256 / (cols/8) row groups when cols < 2048, 4 rows in
// flight); the RG group sums are combined in smem in group order.
__global__ void __launch_bounds__(256)
    k_colsum_part(const bf16* __restrict__ x, int64_t rows, int cols, const int32_t* __restrict__ sel,
                  int sel_val, int64_t chunk, float* __restrict__ ws) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[256 * 8];
  const int vecs = cols / 8;
  const int vb = vecs < 256 ? vecs : 256;       // vectors per block
  const int RG = 256 / vb;                      // row groups
  const int g = threadIdx.x / vb;
  const int c8 = blockIdx.y * vb + threadIdx.x % vb;
  const bool on = g < RG && c8 < vecs;
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (on) {
    const int64_t r0 = int64_t(blockIdx.x) * chunk, r1 = min(rows, r0 + chunk);
    const uint4* xp = reinterpret_cast<const uint4*>(x) + c8;
    int64_t r = r0 + g;
    if (!sel) {
      for (; r + 3 * RG < r1; r += 4 * RG) {
        uint4 u[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) u[k] = __ldg(xp + (r + k * RG) * vecs);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float v[8];
          unpack8(u[k], v);
#pragma unroll
          for (int i = 0; i < 8; ++i) s[i] += v[i];
        }
      }
    }
    for (; r < r1; r += RG) {
      if (sel && __ldg(sel + r) != sel_val) continue;
      float v[8];
      unpack8(__ldg(xp + r * vecs), v);
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i] += v[i];
    }
  }
  if (RG > 1) {
#pragma unroll
    for (int i = 0; i < 8; ++i) red[threadIdx.x * 8 + i] = s[i];
    __syncthreads();
    if (g == 0 && on) {
      for (int q = 1; q < RG; ++q)
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] += red[(q * vb + threadIdx.x) * 8 + i];
    }
  }
  if (g == 0 && on) {
    float4* o = reinterpret_cast<float4*>(ws + int64_t(blockIdx.x) * cols + c8 * 8);
    o[0] = make_float4(s[0], s[1], s[2], s[3]);
    o[1] = make_float4(s[4], s[5], s[6], s[7]);
  }
}

// ---------------------------------------------------------------- embeddings
// y[t] = dropout(word[id[t]] + pos[t % S] + type[tt[t]]); warp per token,
// a lane pair shares each Philox block (16 columns).
template <int NV>
__global__ void __launch_bounds__(256)
    k_embed_fwd(const int32_t* __restrict__ ids, const int32_t* __restrict__ types,
                const bf16* __restrict__ word, const bf16* __restrict__ pos,
                const bf16* __restrict__ type, bf16* __restrict__ y, int64_t T, int S,
                uint32_t thr, float scale, const uint64_t* __restrict__ rng, uint32_t tag) {
  pdl_wait();
  pdl_trigger();
  constexpr int H = NV * 256;
  const int lane = threadIdx.x & 31;
  const int64_t t = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const uint64_t seed = rng[0], step = rng[1];
  const int64_t id = __ldg(ids + t), tt = types ? __ldg(types + t) : 0, s = t % S;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int v = k * 32 + lane;
    float a[8], b[8], c[8], o[8];
    unpack8(__ldg(reinterpret_cast<const uint4*>(word + id * H) + v), a);
    unpack8(__ldg(reinterpret_cast<const uint4*>(pos + s * H) + v), b);
    unpack8(__ldg(reinterpret_cast<const uint4*>(type + tt * H) + v), c);
    const uint64_t e = uint64_t(t) * H + uint64_t(v) * 8;  // first element
    const uint32_t keep =
        thr ? (keep16(drop_block(seed, step, tag, e >> 4), thr) >> (e & 15)) : 0xFFu;
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = (keep >> i) & 1u ? (a[i] + b[i] + c[i]) * scale : 0.f;
    reinterpret_cast<uint4*>(y + t * H)[v] = pack8(o);
  }
}

// word-embedding gradient: block u sums the rows of unique id uniq[u] in
// token order (perm[seg[u] .. seg[u+1])) into dword[uniq[u]] (fp32, rows of
// ids absent from the batch were zeroed by the caller)
__global__ void __launch_bounds__(128)
    k_embed_word_grad(const bf16* __restrict__ d, const int32_t* __restrict__ csr, int T, int H,
                      float* __restrict__ dword) {
  pdl_wait();
  pdl_trigger();
  const int u = blockIdx.x;
  if (u >= __ldg(csr)) return;
  const int32_t* uniq = csr + 1;
  const int32_t* seg = csr + 1 + T;
  const int32_t* perm = csr + 2 + 2 * T;
  const int id = __ldg(uniq + u), b = __ldg(seg + u), e = __ldg(seg + u + 1);
  for (int c8 = threadIdx.x; c8 * 8 < H; c8 += blockDim.x) {
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int j = b; j < e; ++j) {
      float v[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(d + int64_t(__ldg(perm + j)) * H) + c8), v);
#pragma unroll
      for (int i = 0; i < 8; ++i) s[i] += v[i];
    }
    float4* o = reinterpret_cast<float4*>(dword + int64_t(id) * H + c8 * 8);
    o[0] = make_float4(s[0], s[1], s[2], s[3]);
    o[1] = make_float4(s[4], s[5], s[6], s[7]);
  }
}

// position-embedding gradient: dpos[s] = sum over the batch in order
__global__ void __launch_bounds__(128)
    k_embed_pos_grad(const bf16* __restrict__ d, int B, int S, int H, float* __restrict__ dpos) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.x;
  for (int c8 = threadIdx.x; c8 * 8 < H; c8 += blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int b = 0; b < B; ++b) {
      float v[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(d + (int64_t(b) * S + s) * H) + c8), v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += v[i];
    }
    float4* o = reinterpret_cast<float4*>(dpos + int64_t(s) * H + c8 * 8);
    o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
    o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
  }
}

// ---------------------------------------------------------------- span head
// Block b = sequence b: logits z[t][j] = h[t] . w[j] + bias[j] (j = start,
// end), log-softmax over the S positions, loss_b = (CE_start + CE_end) / 2,
// dlogits = (softmax - onehot) / (2B).
template <int NV>
__global__ void __launch_bounds__(256)
    k_span_head_fwd(const bf16* __restrict__ h, const float* __restrict__ w,
                    const float* __restrict__ bias, const int32_t* __restrict__ label, int S,
                    int B, float* __restrict__ logits, float* __restrict__ dlogits,
                    float* __restrict__ row_loss) {
  pdl_wait();
  pdl_trigger();
  constexpr int H = NV * 256;
  extern __shared__ float z[];  // [S][2]
  __shared__ float red[2][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x;
  float w0[NV][8], w1[NV][8];
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      w0[k][i] = __ldg(w + (k * 32 + lane) * 8 + i);
      w1[k][i] = __ldg(w + H + (k * 32 + lane) * 8 + i);
    }
  const float b0 = __ldg(bias), b1 = __ldg(bias + 1);
  for (int s = warp; s < S; s += 8) {
    const int64_t t = int64_t(b) * S + s;
    float d0 = 0.f, d1 = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float v[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(h + t * H) + k * 32 + lane), v);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        d0 = fmaf(v[i], w0[k][i], d0);
        d1 = fmaf(v[i], w1[k][i], d1);
      }
    }
    d0 = warp_sum(d0) + b0;
    d1 = warp_sum(d1) + b1;
    if (lane == 0) {
      z[2 * s] = d0;
      z[2 * s + 1] = d1;
      logits[2 * t] = d0;
      logits[2 * t + 1] = d1;
    }
  }
  __syncthreads();
  if (warp < 2) {
    const int j = warp;
    float m = -INFINITY;
    for (int s = lane; s < S; s += 32) m = fmaxf(m, z[2 * s + j]);
    m = warp_max(m);
    float l = 0.f;
    for (int s = lane; s < S; s += 32) l += __expf(z[2 * s + j] - m);
    l = warp_sum(l);
    const float lse = m + __logf(l);
    const int y = __ldg(label + 2 * b + j);
    const float inv = 0.5f / float(B);
    for (int s = lane; s < S; s += 32)
      dlogits[2 * (int64_t(b) * S + s) + j] = (__expf(z[2 * s + j] - lse) - (s == y ? 1.f : 0.f)) * inv;
    if (lane == 0) red[j][0] = lse - z[2 * y + j];
  }
  __syncthreads();
  if (threadIdx.x == 0) row_loss[b] = 0.5f * (red[0][0] + red[1][0]);
}

__global__ void k_mean_loss(const float* __restrict__ row_loss, int B, float* __restrict__ loss) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int b = 0; b < B; ++b) s += row_loss[b];
    loss[0] = s / float(B);
  }
}

// dh[t] = dl[t][0] w[0] + dl[t][1] w[1]; partial dw over the block's token
// chunk (fixed warp order) to ws[blk][2][H]
template <int NV>
__global__ void __launch_bounds__(256)
    k_span_head_bwd(const bf16* __restrict__ h, const float* __restrict__ dl,
                    const float* __restrict__ w, bf16* __restrict__ dh, float* __restrict__ ws,
                    int64_t T, int64_t chunk) {
  pdl_wait();
  pdl_trigger();
  constexpr int H = NV * 256;
  __shared__ float red[8][2][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float w0[NV][8], w1[NV][8], a0[NV][8], a1[NV][8];
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      w0[k][i] = __ldg(w + (k * 32 + lane) * 8 + i);
      w1[k][i] = __ldg(w + H + (k * 32 + lane) * 8 + i);
      a0[k][i] = a1[k][i] = 0.f;
    }
  const int64_t t0 = int64_t(blockIdx.x) * chunk, t1 = min(T, t0 + chunk);
  for (int64_t t = t0 + warp; t < t1; t += 8) {
    const float g0 = __ldg(dl + 2 * t), g1 = __ldg(dl + 2 * t + 1);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float v[8], o[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(h + t * H) + k * 32 + lane), v);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        o[i] = fmaf(g0, w0[k][i], g1 * w1[k][i]);
        a0[k][i] = fmaf(g0, v[i], a0[k][i]);
        a1[k][i] = fmaf(g1, v[i], a1[k][i]);
      }
      reinterpret_cast<uint4*>(dh + t * H)[k * 32 + lane] = pack8(o);
    }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      red[warp][0][lane * 8 + i] = a0[k][i];
      red[warp][1][lane * 8 + i] = a1[k][i];
    }
    __syncthreads();
    for (int x = threadIdx.x; x < 512; x += 256) {
      const int which = x >> 8, c = x & 255;
      float s = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += red[q][which][c];
      ws[(int64_t(blockIdx.x) * 2 + which) * H + k * 256 + c] = s;
    }
    __syncthreads();
  }
}

// dbias[j] = sum_t dl[t][j] in token order (one warp per j, fixed lane
// partition, xor-tree combine)
__global__ void k_span_dbias(const float* __restrict__ dl, int64_t T, float* __restrict__ dbias) {
  pdl_wait();
  pdl_trigger();
  const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (j >= 2) return;
  float s = 0.f;
  for (int64_t t = lane; t < T; t += 32) s += dl[2 * t + j];
  s = warp_sum(s);
  if (lane == 0) dbias[j] = s;
}

// ---------------------------------------------------------------- attention prep
// D[(b*heads + hd)*S + s] = sum_d dO[t][hd*64 + d] * O[t][hd*64 + d]; warp per
// token
__global__ void __launch_bounds__(256)
    k_attn_dvec(const bf16* __restrict__ o, const bf16* __restrict__ d, int64_t T, int S, int heads,
                float* __restrict__ D) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int64_t t = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const int H = heads * 64;
  const int64_t bb = t / S, ss = t % S;
  // lane-interleaved 16-byte chunks (each load instruction reads 512
  // contiguous bytes): chunk u covers columns [u*256, u*256 + 256), four heads,
  // lane l its 8 columns u*256 + 8 l; a head's sum is an 8-lane reduction
  for (int u = 0; u * 256 < H; ++u) {
    const int c0 = u * 256 + lane * 8;
    float s = 0.f;
    if (c0 < H) {
      float a[8], b[8];
      unpack8(__ldg(reinterpret_cast<const uint4*>(o + t * H + c0)), a);
      unpack8(__ldg(reinterpret_cast<const uint4*>(d + t * H + c0)), b);
#pragma unroll
      for (int i = 0; i < 8; ++i) s = fmaf(a[i], b[i], s);
    }
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 4);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 2);
    s += __shfl_xor_sync(0xFFFFFFFFu, s, 1);
    if (c0 < H && (lane & 7) == 0) D[(bb * heads + c0 / 64) * S + ss] = s;
  }
}

// ---------------------------------------------------------------- optimizer
// AdamW (decoupled weight decay on the first n_bf elements: the matrices and
// embedding tables), bias-corrected with the device step counter rng[1] + 1;
// the leading n_bf fp32 masters also written as bf16 (the GEMM operands).
__device__ __forceinline__ void adamw1(float& w, float& m, float& v, float g, bool decay, float lr,
                                       float b1, float b2, float eps, float wd, float c1, float c2) {
  m = fmaf(b1, m, (1.f - b1) * g);
  v = fmaf(b2, v, (1.f - b2) * g * g);
  const float upd = (m * c1) / (sqrtf(v * c2) + eps) + (decay ? wd * w : 0.f);
  w = fmaf(-lr, upd, w);
}

__global__ void __launch_bounds__(256)
    k_adamw(float* __restrict__ w, float* __restrict__ m, float* __restrict__ v,
            const float* __restrict__ g, bf16* __restrict__ wbf, int64_t n, int64_t n_bf, float lr,
            float b1, float b2, float eps, float wd, const uint64_t* __restrict__ rng) {
  pdl_wait();
  pdl_trigger();
  const float t = float(rng[1] + 1);
  const float c1 = 1.f / (1.f - powf(b1, t)), c2 = 1.f / (1.f - powf(b2, t));
  const int64_t n4 = n >> 2, stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 wv = reinterpret_cast<const float4*>(w)[i];
    float4 mv = reinterpret_cast<const float4*>(m)[i];
    float4 vv = reinterpret_cast<const float4*>(v)[i];
    const float4 gv = __ldg(reinterpret_cast<const float4*>(g) + i);
    const int64_t e = 4 * i;
    adamw1(wv.x, mv.x, vv.x, gv.x, e < n_bf, lr, b1, b2, eps, wd, c1, c2);
    adamw1(wv.y, mv.y, vv.y, gv.y, e + 1 < n_bf, lr, b1, b2, eps, wd, c1, c2);
    adamw1(wv.z, mv.z, vv.z, gv.z, e + 2 < n_bf, lr, b1, b2, eps, wd, c1, c2);
    adamw1(wv.w, mv.w, vv.w, gv.w, e + 3 < n_bf, lr, b1, b2, eps, wd, c1, c2);
    reinterpret_cast<float4*>(w)[i] = wv;
    reinterpret_cast<float4*>(m)[i] = mv;
    reinterpret_cast<float4*>(v)[i] = vv;
    if (e + 3 < n_bf) {
      reinterpret_cast<uint2*>(wbf)[i] = make_uint2(pk2(wv.x, wv.y), pk2(wv.z, wv.w));
    } else if (e < n_bf) {
      const float f[4] = {wv.x, wv.y, wv.z, wv.w};
      for (int k = 0; k < 4 && e + k < n_bf; ++k) wbf[e + k] = __float2bfloat16_rn(f[k]);
    }
  }
  for (int64_t i = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    float wi = w[i], mi = m[i], vi = v[i];
    adamw1(wi, mi, vi, g[i], i < n_bf, lr, b1, b2, eps, wd, c1, c2);
    w[i] = wi;
    m[i] = mi;
    v[i] = vi;
    if (i < n_bf) wbf[i] = __float2bfloat16_rn(wi);
  }
}

__global__ void k_rng_advance(uint64_t* rng) {
  if (threadIdx.x == 0) rng[1] += 1;
}

int grid_for(int64_t work, int per_block) {
  const int64_t b = (work + per_block - 1) / per_block;
  return int(std::max<int64_t>(1, std::min<int64_t>(b, int64_t(sms()) * 16)));
}

}  // namespace

cudaError_t merge_parts(const float* ws, int parts, int cols, float* out, cudaStream_t st) {
  return parts_merge(ws, parts, cols, cols, out, 0, st);
}

// ================================================================ launchers
#define DELTA_NV_SWITCH(H, ...)       \
  switch ((H) / 256) {                \
    case 1: { constexpr int NV = 1; __VA_ARGS__; break; } \
    case 2: { constexpr int NV = 2; __VA_ARGS__; break; } \
    case 3: { constexpr int NV = 3; __VA_ARGS__; break; } \
    case 4: { constexpr int NV = 4; __VA_ARGS__; break; } \
    case 8: { constexpr int NV = 8; __VA_ARGS__; break; } \
    default: return cudaErrorInvalidValue;        \
  }

bool xf_width_ok(int H) { return H % 256 == 0 && (H / 256 <= 4 || H / 256 == 8); }

cudaError_t layernorm_fwd(const void* x, void* y, float* mean, float* rstd, const float* gamma,
                          const float* beta, int64_t rows, int H, float eps, cudaStream_t st) {
  if (!xf_width_ok(H) || rows <= 0) return cudaErrorInvalidValue;
  // two blocks per SM, each warp walking rows (ln_fwd_smem: 56 KB at H = 1024)
  const dim3 grid(unsigned(std::min<int64_t>((rows + 7) / 8, 2 * int64_t(sms()))));
  DELTA_NV_SWITCH(H, {
    static bool attr = false;
    if (!attr) {
      if (cudaError_t e = cudaFuncSetAttribute(k_layernorm_fwd<NV>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               int(ln_fwd_smem<NV>())))
        return e;
      attr = true;
    }
    if (cudaError_t e = launch_k(k_layernorm_fwd<NV>, grid, dim3(256), ln_fwd_smem<NV>(), st,
                                 static_cast<const bf16*>(x), static_cast<bf16*>(y), mean, rstd,
                                 gamma, beta, rows, eps))
      return e;
  });
  return cudaGetLastError();
}

// one wave of one block per SM (the staged rows keep the loads in flight)
int ln_bwd_parts(int64_t rows) {
  return int(std::max<int64_t>(1, std::min<int64_t>((rows + 63) / 64, sms())));
}
template <int NV, bool DROP, typename... Args>
cudaError_t ln_bwd_launch(int parts, cudaStream_t st, Args... args) {
  static bool attr = false;
  if (!attr) {
    if (cudaError_t e = cudaFuncSetAttribute(k_layernorm_bwd<NV, DROP>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(ln_bwd_smem<NV>())))
      return e;
    attr = true;
  }
  return launch_k(k_layernorm_bwd<NV, DROP>, dim3(parts), dim3(256), ln_bwd_smem<NV>(), st,
                  args...);
}
int64_t layernorm_bwd_workspace_floats(int64_t rows, int H) {
  return int64_t(4 * sms()) * 3 * H;
}

cudaError_t layernorm_bwd(const void* dy, const void* x, const void* dres, void* dx,
                          const float* mean, const float* rstd, const float* gamma, float* dgamma,
                          float* dbeta, float* ws, int64_t rows, int H, cudaStream_t st) {
  return layernorm_bwd_drop(dy, x, dres, dx, mean, rstd, gamma, dgamma, dbeta, ws, rows, H,
                            nullptr, nullptr, 0.f, nullptr, 0, st);
}

cudaError_t layernorm_bwd_drop(const void* dy, const void* x, const void* dres, void* dx,
                               const float* mean, const float* rstd, const float* gamma,
                               float* dgamma, float* dbeta, float* ws, int64_t rows, int H,
                               void* dxd, float* dbias, float p, const uint64_t* rng, uint32_t tag,
                               cudaStream_t st) {
  if (!xf_width_ok(H) || rows <= 0 || H / 256 > 4) return cudaErrorInvalidValue;
  if (dxd && (!dbias || !rng)) return cudaErrorInvalidValue;
  const int parts = ln_bwd_parts(rows);
  const int64_t chunk = (rows + parts - 1) / parts;
  const DropParams dp = drop_params(p);
  const LnDrop dr{static_cast<bf16*>(dxd), dp.thr, dp.scale, rng, tag};
  const auto* dy_ = static_cast<const bf16*>(dy);
  const auto* x_ = static_cast<const bf16*>(x);
  const auto* dres_ = static_cast<const bf16*>(dres);
  auto* dx_ = static_cast<bf16*>(dx);
  if (dxd) {
    DELTA_NV_SWITCH(H, if (cudaError_t e = ln_bwd_launch<NV, true>(parts, st, dy_, x_, dres_, dx_,
                                                                   mean, rstd, gamma, ws, rows,
                                                                   chunk, dr)) return e);
    if (cudaError_t e = parts_merge(ws, parts, 3 * int64_t(H), H, dgamma, 0, st, H, dbeta, dbias))
      return e;
  } else {
    DELTA_NV_SWITCH(H, if (cudaError_t e = ln_bwd_launch<NV, false>(parts, st, dy_, x_, dres_, dx_,
                                                                    mean, rstd, gamma, ws, rows,
                                                                    chunk, dr)) return e);
    if (cudaError_t e = parts_merge(ws, parts, 2 * int64_t(H), H, dgamma, 0, st, H, dbeta))
      return e;
  }
  return cudaGetLastError();
}

cudaError_t gelu_fwd(const void* x, void* y, int64_t n, cudaStream_t st) {
  if (n % 8) return cudaErrorInvalidValue;
  if (cudaError_t e = launch_k(k_gelu_fwd, dim3(grid_for(n / 8, 256)), dim3(256), 0, st,
                               static_cast<const uint4*>(x), static_cast<uint4*>(y), n / 8))
    return e;
  return cudaGetLastError();
}

cudaError_t add_dropout(const void* a, const void* b, void* y, int64_t n, float p,
                        const uint64_t* rng, uint32_t tag, cudaStream_t st) {
  if (n % 16) return cudaErrorInvalidValue;
  const DropParams dp = drop_params(p);
  if (cudaError_t e = launch_k(k_dropout<false>, dim3(grid_for(n / 16, 256)), dim3(256), 0, st,
                               static_cast<const uint4*>(a), static_cast<const uint4*>(b),
                               static_cast<uint4*>(y), n / 16, dp.thr, dp.scale, rng, tag))
    return e;
  return cudaGetLastError();
}

cudaError_t dropout_bwd(const void* dy, void* dx, int64_t n, float p, const uint64_t* rng,
                        uint32_t tag, cudaStream_t st) {
  if (n % 16) return cudaErrorInvalidValue;
  const DropParams dp = drop_params(p);
  if (cudaError_t e = launch_k(k_dropout<true>, dim3(grid_for(n / 16, 256)), dim3(256), 0, st,
                               static_cast<const uint4*>(nullptr), static_cast<const uint4*>(dy),
                               static_cast<uint4*>(dx), n / 16, dp.thr, dp.scale, rng, tag))
    return e;
  return cudaGetLastError();
}

int colsum_parts(int64_t rows) {
  return int(std::max<int64_t>(1, std::min<int64_t>((rows + 31) / 32, 2 * sms())));
}
int64_t colsum_workspace_floats(int64_t rows, int cols) {
  return int64_t(2 * sms()) * cols;
}

cudaError_t colsum(const void* x, int64_t rows, int cols, const int32_t* sel, int sel_val,
                   float* out, float* ws, int accumulate, cudaStream_t st) {
  if (cols % 8 || rows <= 0) return cudaErrorInvalidValue;
  const int parts = colsum_parts(rows);
  const int64_t chunk = (rows + parts - 1) / parts;
  const dim3 grid(parts, unsigned((cols / 8 + 255) / 256));  // vectors per block: min(cols/8, 256)
  if (cudaError_t e = launch_k(k_colsum_part, grid, dim3(256), 0, st, static_cast<const bf16*>(x),
                               rows, cols, sel, sel_val, chunk, ws))
    return e;
  if (cudaError_t e = parts_merge(ws, parts, cols, cols, out, accumulate, st)) return e;
  return cudaGetLastError();
}

cudaError_t embed_fwd(const int32_t* ids, const int32_t* types, const void* word, const void* pos,
                      const void* type, void* y, int B, int S, int H, float p, const uint64_t* rng,
                      uint32_t tag, cudaStream_t st) {
  if (!xf_width_ok(H)) return cudaErrorInvalidValue;
  const int64_t T = int64_t(B) * S;
  const DropParams dp = drop_params(p);
  DELTA_NV_SWITCH(H, if (cudaError_t e = launch_k(k_embed_fwd<NV>, dim3(unsigned((T + 7) / 8)),
                                                  dim3(256), 0, st, ids, types,
                                                  static_cast<const bf16*>(word),
                                                  static_cast<const bf16*>(pos),
                                                  static_cast<const bf16*>(type),
                                                  static_cast<bf16*>(y), T, S, dp.thr, dp.scale,
                                                  rng, tag)) return e);
  return cudaGetLastError();
}

cudaError_t embed_grads(const void* dsum, const int32_t* csr, const int32_t* types, int B, int S,
                        int H, int vocab, int n_types, float* dword, float* dpos, float* dtype,
                        float* ws, cudaStream_t st) {
  const int T = B * S;
  if (H % 8) return cudaErrorInvalidValue;
  if (cudaError_t e = cudaMemsetAsync(dword, 0, size_t(vocab) * H * 4, st)) return e;
  if (cudaError_t e = launch_k(k_embed_word_grad, dim3(T), dim3(128), 0, st,
                               static_cast<const bf16*>(dsum), csr, T, H, dword))
    return e;
  if (cudaError_t e = launch_k(k_embed_pos_grad, dim3(S), dim3(128), 0, st,
                               static_cast<const bf16*>(dsum), B, S, H, dpos))
    return e;
  for (int j = 0; j < n_types; ++j)
    if (cudaError_t e = colsum(dsum, T, H, types, j, dtype + int64_t(j) * H, ws, 0, st)) return e;
  return cudaGetLastError();
}

cudaError_t span_head_fwd(const void* h, const float* w, const float* bias, const int32_t* label,
                          float* logits, float* dlogits, float* row_loss, float* loss, int B,
                          int S, int H, cudaStream_t st) {
  if (!xf_width_ok(H) || H / 256 > 4) return cudaErrorInvalidValue;
  const size_t smem = size_t(S) * 2 * sizeof(float);
  DELTA_NV_SWITCH(H, if (cudaError_t e = launch_k(k_span_head_fwd<NV>, dim3(B), dim3(256), smem,
                                                  st, static_cast<const bf16*>(h), w, bias, label,
                                                  S, B, logits, dlogits, row_loss)) return e);
  if (cudaError_t e = launch_k(k_mean_loss, dim3(1), dim3(32), 0, st,
                               static_cast<const float*>(row_loss), B, loss))
    return e;
  return cudaGetLastError();
}

int64_t span_head_workspace_floats(int64_t T, int H) { return int64_t(4 * sms()) * 2 * H; }

cudaError_t span_head_bwd(const void* h, const float* dlogits, const float* w, void* dh, float* dw,
                          float* dbias, float* ws, int64_t T, int H, cudaStream_t st) {
  if (!xf_width_ok(H) || H / 256 > 4) return cudaErrorInvalidValue;
  const int parts = ln_bwd_parts(T);
  const int64_t chunk = (T + parts - 1) / parts;
  DELTA_NV_SWITCH(H, if (cudaError_t e = launch_k(k_span_head_bwd<NV>, dim3(parts), dim3(256), 0,
                                                  st, static_cast<const bf16*>(h), dlogits, w,
                                                  static_cast<bf16*>(dh), ws, T, chunk)) return e);
  if (cudaError_t e = parts_merge(ws, parts, 2 * int64_t(H), H, dw, 0, st, H, dw + H)) return e;
  if (cudaError_t e = launch_k(k_span_dbias, dim3(1), dim3(64), 0, st, dlogits, T, dbias))
    return e;
  return cudaGetLastError();
}

cudaError_t attn_dvec(const void* o, const void* dout, int64_t T, int S, int heads, float* D,
                      cudaStream_t st) {
  if (cudaError_t e = launch_k(k_attn_dvec, dim3(unsigned((T + 7) / 8)), dim3(256), 0, st,
                               static_cast<const bf16*>(o), static_cast<const bf16*>(dout), T, S,
                               heads, D))
    return e;
  return cudaGetLastError();
}

cudaError_t adamw_step(float* w, float* m, float* v, const float* g, void* wbf, int64_t n,
                       int64_t n_bf, float lr, float b1, float b2, float eps, float wd,
                       uint64_t* rng, cudaStream_t st) {
  if (cudaError_t e = launch_k(k_adamw, dim3(grid_for(n, 256)), dim3(256), 0, st, w, m, v, g,
                               static_cast<bf16*>(wbf), n, n_bf, lr, b1, b2, eps, wd,
                               static_cast<const uint64_t*>(rng)))
    return e;
  if (cudaError_t e = launch_k(k_rng_advance, dim3(1), dim3(32), 0, st, rng)) return e;
  return cudaGetLastError();
}

}  // namespace delta_k
