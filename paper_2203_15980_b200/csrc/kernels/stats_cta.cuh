// Per-CTA BN statistics partials written by the conv epilogues (conv_fwd.cu,
// conv_halo.cu): row blockIdx.x of a [gridDim.x][K] float4 table, one row per
// persistent CTA (launches that produce statistics always use one CTA per SM,
// idle CTAs leave a zero row).  Every tile of the CTA is merged into its row
// in the CTA's static tile order, so the result is deterministic:
//   EPI_STORE   (count, mean, M2, 0) of the stored bf16 outputs (Chan's merge)
//   EPI_BN_BWD  (sum g, sum g*xc, 0, 0)
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

}  // namespace delta_k
