// Optimizer step and the per-step weight views, as two launches instead of
// one torch op per tensor (the SGD update was 5 full passes over the flat
// fp32 buffers plus ~40 small strided copies for the bf16 / transposed /
// pixel-pair weight views every step).
//
//   k_sgd_step:     mom = mom*m + g + wd*w ; w -= lr*mom ; wbf = bf16(w)  (conv slice)
//                   — one pass over the flat fp32 master/grad/momentum buffers
//                   (torch.optim.SGD's momentum/weight-decay order, not its
//                   in-place op sequence: fp32 FMA contraction may differ in
//                   the last bit).
//   k_weight_views: every derived bf16 weight tensor from the bf16 conv
//                   weights [K][R][S][C], one table entry per tensor:
//                   DELTA_VIEW_DGRAD  W'[c][r][s][k] = W[k][R-1-r][S-1-s][c]
//                                     (input-gradient convs on our kernel)
//                   DELTA_VIEW_DGRAD_S2 the taps of one parity class of a
//                                     stride-2 3x3 input gradient (sub-pixel)
//                   DELTA_VIEW_STEM   [K][256] pixel-pair stem layout, column
//                                     (r*4+j)*8 + e*4 + c = W[k][r][2j+e-1][c]
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "kernels/kernels.hpp"
#include "kernels/launch.hpp"

namespace delta_k {

namespace {

using bf16 = __nv_bfloat16;

__global__ void __launch_bounds__(256)
    k_sgd_step(float* __restrict__ w, float* __restrict__ mom, const float* __restrict__ g,
               bf16* __restrict__ wbf, int64_t n, int64_t n_bf, float lr, float m, float wd) {
  pdl_wait();
  pdl_trigger();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t n4 = n >> 2;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 wv = reinterpret_cast<const float4*>(w)[i];
    float4 mv = reinterpret_cast<const float4*>(mom)[i];
    const float4 gv = __ldg(reinterpret_cast<const float4*>(g) + i);
    mv.x = fmaf(wd, wv.x, mv.x * m + gv.x);
    mv.y = fmaf(wd, wv.y, mv.y * m + gv.y);
    mv.z = fmaf(wd, wv.z, mv.z * m + gv.z);
    mv.w = fmaf(wd, wv.w, mv.w * m + gv.w);
    wv.x = fmaf(-lr, mv.x, wv.x);
    wv.y = fmaf(-lr, mv.y, wv.y);
    wv.z = fmaf(-lr, mv.z, wv.z);
    wv.w = fmaf(-lr, mv.w, wv.w);
    reinterpret_cast<float4*>(mom)[i] = mv;
    reinterpret_cast<float4*>(w)[i] = wv;
    if (4 * i + 3 < n_bf) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(wv.x, wv.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(wv.z, wv.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      reinterpret_cast<uint2*>(wbf)[i] = pk;
    } else if (4 * i < n_bf) {
      const float e[4] = {wv.x, wv.y, wv.z, wv.w};
      for (int k = 0; k < 4 && 4 * i + k < n_bf; ++k) wbf[4 * i + k] = __float2bfloat16_rn(e[k]);
    }
  }
  // tail (n % 4)
  for (int64_t i = 4 * n4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float mv = fmaf(wd, w[i], mom[i] * m + g[i]);
    mom[i] = mv;
    w[i] = fmaf(-lr, mv, w[i]);
    if (i < n_bf) wbf[i] = __float2bfloat16_rn(w[i]);
  }
}

__global__ void __launch_bounds__(256)
    k_weight_views(const delta_weight_view* __restrict__ views, int n_views) {
  pdl_wait();
  pdl_trigger();
  const delta_weight_view v = views[blockIdx.y];
  const bf16* src = static_cast<const bf16*>(v.src);
  bf16* dst = static_cast<bf16*>(v.dst);
  const int K = v.K, R = v.R, S = v.S, C = v.C;
  if (v.kind == DELTA_VIEW_DGRAD || v.kind == DELTA_VIEW_DGRAD_S2) {
    // per destination filter tap (r, s): dst_tap[c][k] = src_tap'[k][c] — a
    // K x C transpose in 32 x 32 tiles through shared memory (both sides
    // coalesced); 256 threads = 32 columns x 8 rows, 4 rows each.
    //   DGRAD:    R x S taps, tap' = (R-1-r, S-1-s)
    //   DGRAD_S2: parity class (a, b) = (reserved >> 1, reserved & 1) of a
    //             stride-2 3x3 conv: (1+a) x (1+b) taps; sub-pixel tap t of a
    //             class reads dY at offset +t and weight row s2(a, t) with
    //             s2(0, 0) = 1, s2(1, 0) = 2, s2(1, 1) = 0 (same for columns)
    __shared__ bf16 tile[32][33];
    const bool s2 = v.kind == DELTA_VIEW_DGRAD_S2;
    const int pa = v.reserved >> 1, pb = v.reserved & 1;
    const int Rd = s2 ? 1 + pa : R, Sd = s2 ? 1 + pb : S;
    const int taps = Rd * Sd, tk = (K + 31) >> 5, tc = (C + 31) >> 5;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < taps * tk * tc; t += gridDim.x) {
      const int tap = t / (tk * tc), rem = t - tap * (tk * tc);
      const int k0 = (rem / tc) * 32, c0 = (rem % tc) * 32;
      const int r = tap / Sd, s = tap - r * Sd;
      const int src_tap = s2 ? (pa ? 2 - 2 * r : 1) * S + (pb ? 2 - 2 * s : 1)
                             : (R - 1 - r) * S + (S - 1 - s);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = k0 + ty + 8 * i, c = c0 + tx;
        if (k < K && c < C) tile[ty + 8 * i][tx] = src[(int64_t(k) * R * S + src_tap) * C + c];
      }
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int c = c0 + ty + 8 * i, k = k0 + tx;
        if (k < K && c < C) dst[(int64_t(c) * taps + tap) * K + k] = tile[tx][ty + 8 * i];
      }
      __syncthreads();
    }
  } else {  // DELTA_VIEW_STEM: C = 4, 7x7 -> [K][256]
    const int64_t total = int64_t(K) * 256;
    for (int64_t o = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; o < total;
         o += int64_t(gridDim.x) * blockDim.x) {
      const int k = int(o >> 8), col = int(o & 255);
      const int tap = col >> 3, e = (col >> 2) & 1, c = col & 3;
      const int r = tap >> 2, j = tap & 3, s = 2 * j + e - 1;
      const bool ok = tap < 28 && s >= 0 && s < 7;
      dst[o] = ok ? src[((int64_t(k) * 7 + r) * 7 + s) * 4 + c] : __float2bfloat16_rn(0.f);
    }
  }
}

}  // namespace

cudaError_t sgd_step(float* w, float* mom, const float* g, void* wbf, int64_t n, int64_t n_bf,
                     float lr, float m, float wd, cudaStream_t st) {
  if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(mom) |
       reinterpret_cast<uintptr_t>(g)) & 15)
    return cudaErrorInvalidValue;
  if (n_bf > 0 && (reinterpret_cast<uintptr_t>(wbf) & 7)) return cudaErrorInvalidValue;
  const int64_t blocks = std::min<int64_t>((n / 4 + 255) / 256 + 1, 148 * 8);
  return launch_k(k_sgd_step, dim3(unsigned(blocks)), dim3(256), 0, st, w, mom, g,
                  static_cast<bf16*>(wbf), n, n_bf, lr, m, wd);
}

cudaError_t weight_views(const delta_weight_view* views_dev, int n_views, cudaStream_t st) {
  if (n_views <= 0) return cudaSuccess;
  return launch_k(k_weight_views, dim3(128, unsigned(n_views)), dim3(256), 0, st, views_dev,
                  n_views);
}

}  // namespace delta_k
