// Per-CTA BN statistics partials written by the conv epilogues (conv_fwd.cu,
// conv_halo.cu): row blockIdx.x of a [gridDim.x][K] float4 table, one row per
// persistent CTA (launches that produce statistics always use one CTA per SM,
// idle CTAs leave a zero row).  Every tile of the CTA is merged into its row
// in the CTA's static tile order, so the result is deterministic:
//   EPI_STORE   (count, mean, M2, 0) of the stored bf16 outputs (Chan's merge)
//   EPI_BN_BWD  (sum g, sum g*xc, 0, 0)
//   EPI_ADD_MASK with xc (conv_fwd.cu EV_ADD_OM_ST): (sum y, sum y*xc, 0, 0)
//               of its output, the sums of the BN backward that consumes it
// One merge launch then reduces the (at most SM-count) rows per channel in a
// fixed order (bn_pool.cu) — no per-tile partials, no grouping pass.
#pragma once
#include <cuda_runtime.h>

namespace delta_k {

// zero this CTA's row; thread `et` of `nt` owns columns n0 + c, c = et mod nt
// (the same mapping stats_merge_tile is called with), so no barrier is needed
__device__ __forceinline__ void stats_row_zero(float4* stats, int K, int BN, int et, int nt) {
  float4* row = stats + size_t(blockIdx.x) * K;
  for (int n0 = 0; n0 < K; n0 += BN)
    for (int c = et; c < BN && n0 + c < K; c += nt) row[n0 + c] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// fold (n_t rows, sum S, sum of squares / cross term Q) into `a`: a
// (count, mean, M2) running value, or (sum g, sum g*xc) sums for SUMS
template <bool SUMS>
__device__ __forceinline__ float4 stats_merge_tile(float4 a, float n_t, float S, float Q) {
  if (SUMS) {
    a.x += S;
    a.y += Q;
  } else {
    // fast reciprocal: deterministic, ~2 ulp, and off the epilogue's critical path
    const float mu_t = __fdividef(S, n_t);
    const float m2_t = fmaxf(Q - S * mu_t, 0.f);
    const float n = a.x + n_t;
    const float w = __fdividef(n_t, n);
    const float d = mu_t - a.y;
    a.y = fmaf(d, w, a.y);
    a.z += m2_t + d * d * (a.x * w);
    a.x = n;
  }
  return a;
}

// Chan merge of two (count, mean, M2) triples
__device__ __forceinline__ float4 stats_merge_pair(float4 a, float4 b) {
  if (b.x <= 0.f) return a;
  const float n = a.x + b.x;
  const float d = b.y - a.y;
  a.y = fmaf(d, b.x / n, a.y);
  a.z += b.z + d * d * (a.x * b.x / n);
  a.x = n;
  return a;
}

// ... the same, read-modify-write of this CTA's row in the table
template <bool SUMS>
__device__ __forceinline__ void stats_fold_tile(float4* stats, int K, int col, float n_t, float S,
                                                float Q) {
  float4* p = stats + size_t(blockIdx.x) * K + col;
  *p = stats_merge_tile<SUMS>(*p, n_t, S, Q);
}

// Column sums of a 32x32 bf16 block staged with the 64B swizzle (row r at
// byte r*64, its 16 B chunk c at ((c ^ ((r >> 1) & 3)) << 4)) — the epilogue's
// TMA-store staging layout.  Lane c returns (sum of column c, sum of column c
// times the same column of `obuf` (CROSS: BN backward's sum g*xc) or of
// itself (sum of squares)) over the rows set in `rowmask`.  Each lane walks a
// column PAIR over every other row with packed fp32 math (FADD2/FFMA2), the
// two row parities are combined by one xor shuffle and the pairs spread back
// to one column per lane: fixed order, deterministic.
template <bool CROSS>
__device__ __forceinline__ float2 column_sums32(uint32_t buf, uint32_t obuf, uint32_t rowmask,
                                                int lane) {
  const int pr = lane >> 4;        // row parity
  const uint32_t cp = lane & 15;   // columns 2cp, 2cp + 1
  const uint32_t cb = (cp & 3u) * 4u, c16 = cp >> 2;
  float2 s = make_float2(0.f, 0.f), q = make_float2(0.f, 0.f);
#pragma unroll 8
  for (int i = 0; i < 16; ++i) {
    const int rr = 2 * i + pr;
    const uint32_t off = rr * 64 + ((c16 ^ ((rr >> 1) & 3)) << 4) + cb;
    uint32_t w;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(buf + off));
    if (!((rowmask >> rr) & 1u)) w = 0u;
    const float2 f = make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
    s = __fadd2_rn(s, f);
    if (CROSS) {
      uint32_t wx;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(wx) : "r"(obuf + off));
      const float2 x = make_float2(__uint_as_float(wx << 16), __uint_as_float(wx & 0xFFFF0000u));
      q = __ffma2_rn(f, x, q);
    } else {
      q = __ffma2_rn(f, f, q);
    }
  }
  s.x += __shfl_xor_sync(0xffffffffu, s.x, 16);
  s.y += __shfl_xor_sync(0xffffffffu, s.y, 16);
  q.x += __shfl_xor_sync(0xffffffffu, q.x, 16);
  q.y += __shfl_xor_sync(0xffffffffu, q.y, 16);
  const int src = lane >> 1;
  const float s0 = __shfl_sync(0xffffffffu, s.x, src), s1 = __shfl_sync(0xffffffffu, s.y, src);
  const float q0 = __shfl_sync(0xffffffffu, q.x, src), q1 = __shfl_sync(0xffffffffu, q.y, src);
  return (lane & 1) ? make_float2(s1, q1) : make_float2(s0, q0);
}

}  // namespace delta_k
