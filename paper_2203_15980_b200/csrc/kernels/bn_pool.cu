// HBM-bound kernels of the recompute engine and the backward pass:
// BatchNorm statistics / apply (fused ReLU, fused residual add, fused second
// BN on the shortcut), BN backward, gradient adds, max/avg pooling and the
// softmax cross-entropy head.
//
// Layout: NHWC bf16 viewed as [M = N*H*W rows][C channels], C a power of two
// (64..2048).  Each thread moves 8 channels (16 B) per access.  Every
// reduction is deterministic: per-chunk partials in a fixed grid position,
// merged in a fixed order (no atomics), so the forward statistics — and hence
// every recomputed activation — are reproducible bit for bit.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels/kernels.hpp"
#include "kernels/launch.hpp"

namespace delta_k {

using bf16 = __nv_bfloat16;

namespace {

constexpr int SLICE = 64;   // channel granularity (C is a power of two, 64..2048)
// Streaming loops issue UNROLL vectors' loads of every input before any math
// (memory-level parallelism: 2-3 input streams need ~100+ KB in flight per SM
// to reach HBM speed; a load-use loop kept only ~60 KB and ran at ~4.4 TB/s).
constexpr int UNROLL = 4;

// Rows per reduction partial.  A reduction block covers ALL C channels of its
// rows (C/8 threads per row, 2048/C rows per step: every warp reads whole
// contiguous rows), so there are M / rows partials: ~8 per SM, merged in a
// fixed order by the two-level merge.  A multiple of 16.
int64_t chunk_rows(int64_t M, int C) {
  const int64_t target_ctas = 148 * 8;
  int64_t rows = (M + target_ctas - 1) / target_ctas;
  rows = (rows + 15) / 16 * 16;
  return rows < 16 ? 16 : rows;
}

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// coherent streaming load: for data the same kernel also writes (in place)
__device__ __forceinline__ uint4 ld_coherent(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p)
               : "memory");
  return r;
}
__device__ __forceinline__ void unpack8(uint4 u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

int grid_for(int64_t work_items, int threads) {
  int64_t blocks = (work_items + threads - 1) / threads;
  int64_t cap = 148 * 16;
  return int(blocks < cap ? (blocks < 1 ? 1 : blocks) : cap);
}

// Chan et al. parallel merge of (n, mean, M2).
__device__ __forceinline__ void merge(float& n, float& mu, float& m2, float nb, float mub,
                                      float m2b) {
  if (nb == 0.f) return;
  float nn = n + nb;
  float d = mub - mu;
  mu += d * (nb / nn);
  m2 += m2b + d * d * (n * nb / nn);
  n = nn;
}

// ---------------------------------------------------------------- BN stats
// Per-chunk (mean, M2) of every channel.  Thread layout: tx = channel group
// (8 channels, 16 B), ty = row phase; rows r0+ty, r0+ty+RPI, ... (RPI =
// 256 / (C/8)).  Row-phase partials are combined in smem (fixed order).
__global__ void __launch_bounds__(256, 4) k_bn_stats_partial(const bf16* __restrict__ x, int64_t M,
                                                          int C, int64_t chunk,
                                                          float2* __restrict__ ws) {
  pdl_wait();
  pdl_trigger();
  const int tpr = C >> 3, rpi = 256 / tpr;
  const int tx = threadIdx.x % tpr, ty = threadIdx.x / tpr;
  const int c0 = tx * 8;
  const int64_t r0 = int64_t(blockIdx.x) * chunk;
  const int64_t r1 = min(M, r0 + chunk);
  float s[8] = {0}, q[8] = {0};
  for (int64_t rb = r0 + ty; rb < r1; rb += 2 * UNROLL * rpi) {
    uint4 xv[2 * UNROLL];
#pragma unroll
    for (int u = 0; u < 2 * UNROLL; ++u)
      if (rb + u * rpi < r1) xv[u] = ld_stream(x + (rb + u * rpi) * C + c0);
#pragma unroll
    for (int u = 0; u < 2 * UNROLL; ++u) {
      if (rb + u * rpi >= r1) break;
      float f[8];
      unpack8(xv[u], f);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s[i] += f[i];
        q[i] = fmaf(f[i], f[i], q[i]);
      }
    }
  }
  __shared__ float ss[2048], sq[2048];  // [rpi][C]
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    ss[ty * C + c0 + i] = s[i];
    sq[ty * C + c0 + i] = q[i];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += 256) {
    float S = 0.f, Q = 0.f;
    for (int j = 0; j < rpi; ++j) {
      S += ss[j * C + c];
      Q += sq[j * C + c];
    }
    const float n = float(r1 - r0);
    const float mu = S / n;
    ws[int64_t(blockIdx.x) * C + c] = make_float2(mu, fmaxf(Q - S * mu, 0.f));
  }
}

// Merge per-chunk (mean, M2) partials of `rows_per` rows (last chunk shorter)
// into the channel statistics.  Warp per channel, two passes without
// dependent divisions: (1) total sum -> mean; (2) M2 = sum_i M2_i +
// n_i (mean_i - mean)^2.  Lane-strided accumulation then a fixed xor
// butterfly: deterministic.
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order column sums over partial rows for the 8 channels c0..c0+7 of a
// block: thread t takes channel t&7 of rows t>>3, (t>>3)+32, ... (each warp
// reads 4 rows x 8 adjacent channels: coalesced), then warp 0 adds the 32
// stripes in order.  Returns the sums in thread ch < 8 of warp 0.
template <typename T, typename F>
__device__ __forceinline__ float2 rows_sum8(const T* __restrict__ ws, int rows, int C, int c0,
                                            F&& term) {
  __shared__ float2 part[32][9];
  const int ch = threadIdx.x & 7, stripe = threadIdx.x >> 3;
  float2 acc = make_float2(0.f, 0.f);
  if (c0 + ch < C) {
    // RB rows in flight per thread (the loop is load-latency bound), summed
    // in the same k order as one row at a time
    constexpr int RB = 8;
    for (int k0 = stripe; k0 < rows; k0 += 32 * RB) {
      T v[RB];
#pragma unroll
      for (int b = 0; b < RB; ++b)
        if (k0 + b * 32 < rows) v[b] = ws[int64_t(k0 + b * 32) * C + c0 + ch];
#pragma unroll
      for (int b = 0; b < RB; ++b)
        if (k0 + b * 32 < rows) {
          const float2 t = term(v[b]);
          acc.x += t.x;
          acc.y += t.y;
        }
    }
  }
  part[stripe][ch] = acc;
  __syncthreads();
  float2 r = make_float2(0.f, 0.f);
  if (threadIdx.x < 8)
    for (int k = 0; k < 32; ++k) {
      r.x += part[k][threadIdx.x].x;
      r.y += part[k][threadIdx.x].y;
    }
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256)
    k_bn_stats_merge(const float2* __restrict__ ws, int parts, int64_t rows_per, int64_t M, int C,
                     float* mean, float* invstd, float eps, float* rm, float* rv, float mom) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= C) return;
  const float n_last = float(M - int64_t(parts - 1) * rows_per);
  const float n_full = float(rows_per);
  float s = 0.f;
  for (int k = lane; k < parts; k += 32)
    s = fmaf(k == parts - 1 ? n_last : n_full, ws[int64_t(k) * C + c].x, s);
  const float mu = warp_sum(s) / float(M);
  float m2 = 0.f;
  for (int k = lane; k < parts; k += 32) {
    const float2 p = ws[int64_t(k) * C + c];
    const float d = p.x - mu;
    m2 += fmaf(k == parts - 1 ? n_last : n_full, d * d, p.y);
  }
  m2 = warp_sum(m2);
  if (lane == 0) {
    const float var = m2 / float(M);
    mean[c] = mu;
    invstd[c] = rsqrtf(var + eps);
    if (rm) {
      rm[c] = (1.f - mom) * rm[c] + mom * mu;
      rv[c] = (1.f - mom) * rv[c] + mom * (M > 1 ? m2 / float(M - 1) : var);
    }
  }
}

// Statistics from the conv epilogues' per-CTA rows (stats_cta.cuh): float4
// (count, mean, M2) per (CTA, channel), at most a few hundred rows — one warp
// per channel, lane-strided then a fixed butterfly, so the order is fixed.
__global__ void __launch_bounds__(256)
    k_bn_stats_merge_cta(const float4* __restrict__ ws, int parts, int C, float* mean,
                         float* invstd, float eps, float* rm, float* rv, float mom) {
  pdl_wait();
  pdl_trigger();
  __shared__ float mu_s[8];
  const int c0 = blockIdx.x * 8;
  // pass 1: count and sum(count * mean) -> the channel mean
  const float2 sn = rows_sum8(ws, parts, C, c0,
                              [](float4 p) { return make_float2(p.x * p.y, p.x); });
  if (threadIdx.x < 8) mu_s[threadIdx.x] = sn.y > 0.f ? sn.x / sn.y : 0.f;
  __syncthreads();
  // pass 2: sum(M2 + count * (mean - mu)^2)
  const float mu_c = mu_s[threadIdx.x & 7];
  const float2 m2 = rows_sum8(ws, parts, C, c0, [mu_c](float4 p) {
    const float d = p.y - mu_c;
    return make_float2(fmaf(p.x, d * d, p.z), 0.f);
  });
  const int c = c0 + threadIdx.x;
  if (threadIdx.x < 8 && c < C) {
    const float n = sn.y, mu = mu_s[threadIdx.x];
    const float var = m2.x / n;
    mean[c] = mu;
    invstd[c] = rsqrtf(var + eps);
    if (rm) {
      rm[c] = (1.f - mom) * rm[c] + mom * mu;
      rv[c] = (1.f - mom) * rv[c] + mom * (n > 1.f ? m2.x / (n - 1.f) : var);
    }
  }
}

// Column sums from the per-CTA statistics rows (count, mean, M2): sum =
// sum over rows of count * mean, fixed order — a bias gradient from the
// statistics a GEMM epilogue already reduced (no separate pass over dY)
__global__ void __launch_bounds__(256)
    k_stats_col_sum(const float4* __restrict__ ws, int parts, int C, float* out, int accumulate) {
  pdl_wait();
  pdl_trigger();
  const int c0 = blockIdx.x * 8;
  const float2 sn = rows_sum8(ws, parts, C, c0,
                              [](float4 p) { return make_float2(p.x * p.y, 0.f); });
  const int c = c0 + threadIdx.x;
  if (threadIdx.x < 8 && c < C) out[c] = accumulate ? out[c] + sn.x : sn.x;
}

// BN backward reductions from the per-CTA rows (sum g, sum g*xc): dbeta,
// dgamma per channel, fixed order
__global__ void __launch_bounds__(256)
    k_bn_bwd_final_cta(const float4* __restrict__ ws, int parts, int C, const float* mean,
                       const float* invstd, float* dgamma, float* dbeta) {
  pdl_wait();
  pdl_trigger();
  const int c0 = blockIdx.x * 8;
  const float2 AB = rows_sum8(ws, parts, C, c0, [](float4 p) { return make_float2(p.x, p.y); });
  const int c = c0 + threadIdx.x;
  if (threadIdx.x < 8 && c < C) {
    dbeta[c] = AB.x;
    dgamma[c] = invstd[c] * (AB.y - mean[c] * AB.x);
  }
}

// First level of a two-level merge when there are many partials: thread per
// (channel, group of GROUP consecutive partials) -> one (mean, M2) partial of
// the group's rows.  The group's partials are loaded up front (one memory
// round trip, not GROUP dependent ones), then two passes over registers
// (sum -> mean, then M2) in a fixed order.
constexpr int GROUP = 16;
// a grouping pass only above this many partials: the streaming passes write
// ~148*8 chunk partials, which one warp per channel reduces directly (~2 us)
// faster than a second launch would
int group_above() {
  static const int v = [] {
    const char* e = std::getenv("DELTA_BN_GROUP_ABOVE");
    return e ? std::atoi(e) : 4096;
  }();
  return v;
}
__global__ void __launch_bounds__(256)
    k_bn_stats_group(const float2* __restrict__ ws, int parts, int64_t rows_per, int64_t M, int C,
                     float2* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int k0 = blockIdx.y * GROUP;
  const float n_last = float(M - int64_t(parts - 1) * rows_per);
  const float n_full = float(rows_per);
  float2 p[GROUP];
  float nk[GROUP];
#pragma unroll
  for (int j = 0; j < GROUP; ++j) {
    const int k = k0 + j;
    p[j] = k < parts ? ws[int64_t(k) * C + c] : make_float2(0.f, 0.f);
    nk[j] = k < parts ? (k == parts - 1 ? n_last : n_full) : 0.f;
  }
  float s = 0.f, n = 0.f;
#pragma unroll
  for (int j = 0; j < GROUP; ++j) {
    s = fmaf(nk[j], p[j].x, s);
    n += nk[j];
  }
  const float mu = s / n;
  float m2 = 0.f;
#pragma unroll
  for (int j = 0; j < GROUP; ++j) {
    const float d = p[j].x - mu;
    m2 += fmaf(nk[j], d * d, p[j].y);
  }
  out[int64_t(blockIdx.y) * C + c] = make_float2(mu, m2);
}

// ---------------------------------------------------------------- BN apply
// blockDim (256) is a multiple of C/8 for every C <= 2048, so with a grid
// stride that is a multiple of the block, each thread always touches the SAME
// 8 channels: their scale/shift live in registers, not shared memory.

template <int MODE>
__global__ void __launch_bounds__(256)
    k_bn_apply(const bf16* __restrict__ x, const bf16* __restrict__ res, bf16* __restrict__ y,
               int64_t vecs, int cmask, const float* __restrict__ mean,
               const float* __restrict__ invstd, const float* __restrict__ gamma,
               const float* __restrict__ beta, const float* __restrict__ mean2,
               const float* __restrict__ invstd2, const float* __restrict__ gamma2,
               const float* __restrict__ beta2) {
  // per-channel scale / shift of all C (<= 2048) channels, once per block with
  // coalesced loads (a thread's 8 channels read back from shared memory: the
  // per-thread scattered loads of 4 x 8 parameters cost ~30 us per launch)
  __shared__ __align__(16) float s_sc[2048], s_sh[2048];
  __shared__ __align__(16) float s_sc2[MODE == 2 ? 2048 : 1], s_sh2[MODE == 2 ? 2048 : 1];
  pdl_wait();
  pdl_trigger();
  for (int c = threadIdx.x; c <= cmask; c += blockDim.x) {
    // explicit FMAs: the dgrad BN-backward epilogue (conv_fwd.cu) recomputes
    // this ReLU mask with the identical arithmetic
    const float a = invstd[c] * gamma[c];
    s_sc[c] = a;
    s_sh[c] = fmaf(-mean[c], a, beta[c]);
    if (MODE == 2) {
      const float a2 = invstd2[c] * gamma2[c];
      s_sc2[MODE == 2 ? c : 0] = a2;
      s_sh2[MODE == 2 ? c : 0] = fmaf(-mean2[c], a2, beta2[c]);
    }
  }
  __syncthreads();
  const int64_t first = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c0 = int(first * 8) & cmask;
  float sc[8], sh[8], sc2[8], sh2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sc[j] = s_sc[c0 + j];
    sh[j] = s_sh[c0 + j];
    if (MODE == 2) {
      sc2[j] = s_sc2[MODE == 2 ? c0 + j : 0];
      sh2[j] = s_sh2[MODE == 2 ? c0 + j : 0];
    }
  }
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i0 = first; i0 < vecs; i0 += UNROLL * stride) {
    uint4 xv[UNROLL], rv[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < vecs) {
        xv[u] = ld_stream(x + i * 8);
        if (MODE >= 1) rv[u] = ld_stream(res + i * 8);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= vecs) break;
      float f[8], r[8];
      unpack8(xv[u], f);
      if (MODE >= 1) unpack8(rv[u], r);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float v = fmaf(f[j], sc[j], sh[j]);
        if (MODE == 1) v += r[j];
        if (MODE == 2) v += fmaf(r[j], sc2[j], sh2[j]);
        f[j] = fmaxf(v, 0.f);
      }
      reinterpret_cast<uint4*>(y)[i] = pack8(f);
    }
  }
}

// ------------------------------------------------------------- BN backward
// upstream gradient of row `row`, channels c0..c0+7: full [M,C] (streamed) or
// pooled [N,C] / pool_hw (POOLED; read through L1, rows of one image share it)
template <bool POOLED>
__device__ __forceinline__ uint4 load_up(const bf16* up, int pool_hw, int64_t row, int c0, int C) {
  if (POOLED) return *reinterpret_cast<const uint4*>(up + (row / pool_hw) * C + c0);
  return ld_stream(up + row * C + c0);
}
template <bool POOLED>
__device__ __forceinline__ void unpack_up(uint4 u, float inv_hw, float (&g)[8]) {
  unpack8(u, g);
  if (POOLED) {
#pragma unroll
    for (int j = 0; j < 8; ++j) g[j] *= inv_hw;
  }
}

// Per chunk: sum g and sum g*x (x-hat folded in at the end: sum g*xhat =
// invstd*(sum g*x - mean*sum g)), so no per-channel parameters stay live in
// the loop and occupancy is not register-limited.
template <bool MASKED, bool POOLED>
__device__ __forceinline__ void bn_bwd_chunk(const bf16* __restrict__ up, int pool_hw,
                                             const bf16* __restrict__ mask,
                                             const bf16* __restrict__ x, int64_t M, int C,
                                             int64_t chunk, const float* mean,
                                             const float* invstd, float2* __restrict__ ws) {
  const int tpr = C >> 3, rpi = 256 / tpr;
  const int tx = threadIdx.x % tpr, ty = threadIdx.x / tpr;
  const int c0 = tx * 8;
  const int64_t r0 = int64_t(blockIdx.x) * chunk;
  const int64_t r1 = min(M, r0 + chunk);
  const float inv_hw = POOLED ? 1.f / float(pool_hw) : 1.f;
  float sg[8] = {0}, sgx[8] = {0};
  for (int64_t rb = r0 + ty; rb < r1; rb += UNROLL * rpi) {
    uint4 uv[UNROLL], mv[UNROLL], xv[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t r = rb + u * rpi;
      if (r < r1) {
        uv[u] = load_up<POOLED>(up, pool_hw, r, c0, C);
        if (MASKED) mv[u] = ld_stream(mask + r * C + c0);
        xv[u] = ld_stream(x + r * C + c0);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if (rb + u * rpi >= r1) break;
      float g[8], xf[8];
      unpack_up<POOLED>(uv[u], inv_hw, g);
      if (MASKED) {
        float m[8];
        unpack8(mv[u], m);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = m[j] > 0.f ? g[j] : 0.f;
      }
      unpack8(xv[u], xf);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        sg[j] += g[j];
        sgx[j] = fmaf(g[j], xf[j], sgx[j]);
      }
    }
  }
  __shared__ float a[2048], b[2048];  // [rpi][C]
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[ty * C + c0 + j] = sg[j];
    b[ty * C + c0 + j] = sgx[j];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += 256) {
    float A = 0.f, B = 0.f;
    for (int j = 0; j < rpi; ++j) {
      A += a[j * C + c];
      B += b[j * C + c];
    }
    // sum g*xhat over the chunk = invstd * (sum g*x - mean * sum g)
    ws[int64_t(blockIdx.x) * C + c] = make_float2(A, invstd[c] * (B - mean[c] * A));
  }
}

template <bool MASKED, bool POOLED>
__global__ void __launch_bounds__(256)
    k_bn_bwd_partial(const bf16* __restrict__ up, int pool_hw, const bf16* __restrict__ mask,
                     const bf16* __restrict__ x, int64_t M, int C, int64_t chunk,
                     const float* mean, const float* invstd, float2* __restrict__ ws) {
  pdl_wait();
  pdl_trigger();
  bn_bwd_chunk<MASKED, POOLED>(up, pool_hw, mask, x, M, C, chunk, mean, invstd, ws);
}

// Grid-wide barrier for a grid whose CTAs are all co-resident (a cooperative
// launch guarantees it).  The state is two words at the head of the launch's
// own BN workspace (never a device global, so concurrent launches with their
// own workspaces cannot interleave): bar[0] arrival count, bar[1] generation.
// The last CTA to arrive resets the count and then releases the others, so
// the words return to (0, gen+1): reusable across launches without a memset
// once the workspace was zeroed at allocation.
__device__ __forceinline__ void grid_barrier(unsigned int* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int gen;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      unsigned int g;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
      } while (g == gen);
    }
    __threadfence();
  }
  __syncthreads();
}

// The whole BN backward in one persistent launch (all CTAs resident):
//   1. per-CTA (sum g, sum g*xhat) over a contiguous chunk of rows (bn_bwd_chunk)
//   2. grid barrier; channel c's sums over the CTA rows by one warp, in a fixed
//      order (lane-strided, xor butterfly) -> dbeta, dgamma
//   3. grid barrier; dx over the SAME chunk, last rows first, so the tail of
//      what phase 1 streamed is still in L2.
// Saves the merge launch and, per CTA, up to an L2's share of the second read.
template <bool MASKED, bool POOLED>
__global__ void __launch_bounds__(256)
    k_bn_bwd_grid(const bf16* __restrict__ up, int pool_hw, const bf16* __restrict__ mask,
                  const bf16* __restrict__ x, bf16* __restrict__ dx, int64_t M, int C,
                  int64_t chunk, const float* __restrict__ mean,
                  const float* __restrict__ invstd, const float* __restrict__ gamma,
                  float* dgamma, float* dbeta, float2* ws, unsigned int* bar) {
  pdl_wait();
  bn_bwd_chunk<MASKED, POOLED>(up, pool_hw, mask, x, M, C, chunk, mean, invstd, ws);
  grid_barrier(bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = blockIdx.x * 8 + warp; c < C; c += gridDim.x * 8) {
    float A = 0.f, B = 0.f;
    for (int k = lane; k < int(gridDim.x); k += 32) {
      const float2 p = __ldcg(ws + int64_t(k) * C + c);
      A += p.x;
      B += p.y;
    }
    A = warp_sum(A);
    B = warp_sum(B);
    if (lane == 0) {
      dbeta[c] = A;
      dgamma[c] = B;
    }
  }
  grid_barrier(bar);
  pdl_trigger();
  const int tpr = C >> 3, rpi = 256 / tpr;
  const int tx = threadIdx.x % tpr, ty = threadIdx.x / tpr;
  const int c0 = tx * 8;
  const float invM = 1.f / float(M);
  // the per-channel coefficients once per block, coalesced, through shared
  // memory (as k_bn_bwd_apply)
  __shared__ __align__(16) float s_k1[2048], s_k2[2048], s_k3[2048];
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float is = invstd[c];
    const float a = gamma[c] * is;
    const float kd = __ldcg(dgamma + c) * invM * is;
    s_k1[c] = a;
    s_k2[c] = -a * kd;
    s_k3[c] = a * (kd * mean[c] - __ldcg(dbeta + c) * invM);
  }
  __syncthreads();
  float k1[8], k2[8], k3[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    k1[j] = s_k1[c0 + j];
    k2[j] = s_k2[c0 + j];
    k3[j] = s_k3[c0 + j];
  }
  const float inv_hw = POOLED ? 1.f / float(pool_hw) : 1.f;
  const int64_t r0 = int64_t(blockIdx.x) * chunk;
  const int64_t r1 = min(M, r0 + chunk);
  for (int64_t rb = r1 - 1 - ty; rb >= r0; rb -= UNROLL * rpi) {
    uint4 uv[UNROLL], mv[UNROLL], xv[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t r = rb - u * rpi;
      if (r >= r0) {
        uv[u] = load_up<POOLED>(up, pool_hw, r, c0, C);
        if (MASKED) mv[u] = ld_stream(mask + r * C + c0);
        xv[u] = ld_stream(x + r * C + c0);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t r = rb - u * rpi;
      if (r < r0) break;
      float g[8], xf[8];
      unpack_up<POOLED>(uv[u], inv_hw, g);
      if (MASKED) {
        float m[8];
        unpack8(mv[u], m);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = m[j] > 0.f ? g[j] : 0.f;
      }
      unpack8(xv[u], xf);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = fmaf(k1[j], g[j], fmaf(k2[j], xf[j], k3[j]));
      *reinterpret_cast<uint4*>(dx + r * C + c0) = pack8(g);
    }
  }
}

// warp per channel, lane-strided sums then a fixed xor butterfly
__global__ void __launch_bounds__(256) k_bn_bwd_final(const float2* __restrict__ ws, int chunks,
                                                      int C, float* dgamma, float* dbeta) {
  pdl_wait();
  pdl_trigger();
  const int c0 = blockIdx.x * 8;
  const float2 AB = rows_sum8(ws, chunks, C, c0, [](float2 p) { return p; });
  const int c = c0 + threadIdx.x;
  if (threadIdx.x < 8 && c < C) {
    dbeta[c] = AB.x;
    dgamma[c] = AB.y;
  }
}

// Parameter gradients from the conv epilogue's raw per-tile (sum g, sum g*x)
// partials: pass 1 (when there are many) sums groups of GROUP partials into
// the scratch after them; pass 2 = warp per channel, fixed order; then
// dbeta = sum g, dgamma = invstd * (sum g*x - mean * sum g).
__global__ void __launch_bounds__(256)
    k_bn_bwd_group(const float2* __restrict__ ws, int parts, int C, float2* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int k0 = blockIdx.y * GROUP;
  float2 p[GROUP];
#pragma unroll
  for (int j = 0; j < GROUP; ++j)
    p[j] = k0 + j < parts ? ws[int64_t(k0 + j) * C + c] : make_float2(0.f, 0.f);
  float A = 0.f, B = 0.f;
#pragma unroll
  for (int j = 0; j < GROUP; ++j) {
    A += p[j].x;
    B += p[j].y;
  }
  out[int64_t(blockIdx.y) * C + c] = make_float2(A, B);
}

__global__ void __launch_bounds__(256)
    k_bn_bwd_final_raw(const float2* __restrict__ ws, int parts, int C, const float* mean,
                       const float* invstd, float* dgamma, float* dbeta) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (c >= C) return;
  float A = 0.f, B = 0.f;
  for (int k = lane; k < parts; k += 32) {
    const float2 p = ws[int64_t(k) * C + c];
    A += p.x;
    B += p.y;
  }
  A = warp_sum(A);
  B = warp_sum(B);
  if (lane == 0) {
    dbeta[c] = A;
    dgamma[c] = invstd[c] * (B - mean[c] * A);
  }
}

// dx = gamma*invstd*(g - dbeta/M - xhat*dgamma/M), xhat = (x-mean)*invstd,
// folded per channel into dx = k1*g + k2*x + k3 (3 live coefficients).
// INPLACE: dx == up (the conv-fused BN backward writes its masked gradient g
// in the node's own output slot): `up` is read with coherent loads, not the
// read-only path, since this kernel writes it.
template <bool MASKED, bool POOLED, bool INPLACE = false>
__global__ void __launch_bounds__(256)
    k_bn_bwd_apply(const bf16* up, int pool_hw, const bf16* __restrict__ mask,
                   const bf16* __restrict__ x, bf16* dx, int64_t vecs, int cmask,
                   int logC, int64_t M, const float* __restrict__ mean,
                   const float* __restrict__ invstd, const float* __restrict__ gamma,
                   const float* __restrict__ dgamma, const float* __restrict__ dbeta) {
  // per-channel coefficients of all C (<= 2048) channels, once per block with
  // coalesced loads, read back from shared memory (as k_bn_apply)
  __shared__ __align__(16) float s_k1[2048], s_k2[2048], s_k3[2048];
  pdl_wait();
  pdl_trigger();
  const float invM = 1.f / float(M);
  for (int c = threadIdx.x; c <= cmask; c += blockDim.x) {
    const float is = invstd[c];
    const float a = gamma[c] * is;
    const float kd = dgamma[c] * invM * is;  // coefficient of (x - mean)
    s_k1[c] = a;
    s_k2[c] = -a * kd;
    s_k3[c] = a * (kd * mean[c] - dbeta[c] * invM);
  }
  __syncthreads();
  const int64_t first = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int c0 = int(first * 8) & cmask;
  const int C = cmask + 1;
  float k1[8], k2[8], k3[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    k1[j] = s_k1[c0 + j];
    k2[j] = s_k2[c0 + j];
    k3[j] = s_k3[c0 + j];
  }
  const float inv_hw = POOLED ? 1.f / float(pool_hw) : 1.f;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i0 = first; i0 < vecs; i0 += UNROLL * stride) {
    uint4 uv[UNROLL], mv[UNROLL], xv[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < vecs) {
        uv[u] = POOLED    ? load_up<true>(up, pool_hw, (i * 8) >> logC, c0, C)
                : INPLACE ? ld_coherent(up + i * 8)
                          : ld_stream(up + i * 8);
        if (MASKED) mv[u] = ld_stream(mask + i * 8);
        xv[u] = ld_stream(x + i * 8);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= vecs) break;
      float g[8], xf[8];
      unpack_up<POOLED>(uv[u], inv_hw, g);
      if (MASKED) {
        float m[8];
        unpack8(mv[u], m);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = m[j] > 0.f ? g[j] : 0.f;
      }
      unpack8(xv[u], xf);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = fmaf(k1[j], g[j], fmaf(k2[j], xf[j], k3[j]));
      reinterpret_cast<uint4*>(dx)[i] = pack8(g);
    }
  }
}

// out = (a + g) [* (out_mask > 0)], g = up [* (up_mask > 0)], up full or pooled
template <bool POOLED>
__global__ void __launch_bounds__(256)
    k_add_grad(const bf16* __restrict__ a, const bf16* __restrict__ up, int pool_hw,
               const bf16* __restrict__ up_mask, const bf16* __restrict__ out_mask,
               bf16* __restrict__ out, int64_t vecs, int cmask, int logC, int C) {
  pdl_wait();
  pdl_trigger();
  const float inv_hw = POOLED ? 1.f / float(pool_hw) : 1.f;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < vecs; i += stride) {
    const int c0 = int(i * 8) & cmask;
    const int64_t row = (i * 8) >> logC;
    float fa[8], g[8];
    unpack8(ld_stream(a + i * 8), fa);
    unpack_up<POOLED>(load_up<POOLED>(up, pool_hw, row, c0, C), inv_hw, g);
    if (up_mask) {
      float m[8];
      unpack8(ld_stream(up_mask + i * 8), m);
#pragma unroll
      for (int j = 0; j < 8; ++j) g[j] = m[j] > 0.f ? g[j] : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) fa[j] += g[j];
    if (out_mask) {
      float m[8];
      unpack8(ld_stream(out_mask + i * 8), m);
#pragma unroll
      for (int j = 0; j < 8; ++j) fa[j] = m[j] > 0.f ? fa[j] : 0.f;
    }
    reinterpret_cast<uint4*>(out)[i] = pack8(fa);
  }
}

// ----------------------------------------------------------------- pooling
// Grids: blockIdx.x = one image row (n, row), blockIdx.y x 256 threads span
// (column, 8-channel group) of that row; C/8 is a power of two, so the only
// divisions left are one 32-bit div/mod per thread.
// RPB output rows per block: the input rows shared by neighbouring windows
// are read once (2 RPB + 1 input rows instead of 3 RPB)
template <int RPB>
__global__ void __launch_bounds__(256) k_maxpool_fwd(const bf16* __restrict__ x,
                                                     bf16* __restrict__ y, int N, int H, int W,
                                                     int C, int P, int Q, int lcg) {
  pdl_wait();
  pdl_trigger();
  const int cg = 1 << lcg;
  const int item = blockIdx.y * 256 + threadIdx.x;
  if (item >= Q * cg) return;
  const int q = item >> lcg, c0 = (item & (cg - 1)) * 8;
  const int pb = P / RPB;
  const int n = blockIdx.x / pb, p = (blockIdx.x - n * pb) * RPB;
  float b[RPB][8];
#pragma unroll
  for (int r = 0; r < RPB; ++r)
#pragma unroll
    for (int j = 0; j < 8; ++j) b[r][j] = -INFINITY;
  // input row 2p-1+dh feeds output rows p+r with 2r <= dh <= 2r+2
#pragma unroll
  for (int dh = 0; dh < 2 * RPB + 1; ++dh) {
    const int h = 2 * p - 1 + dh;
    if (h < 0 || h >= H) continue;
#pragma unroll
    for (int dw = 0; dw < 3; ++dw) {
      const int w = 2 * q - 1 + dw;
      if (w < 0 || w >= W) continue;
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(x + ((int64_t(n) * H + h) * W + w) * C + c0), f);
#pragma unroll
      for (int r = 0; r < RPB; ++r) {
        if (dh >= 2 * r && dh <= 2 * r + 2) {
#pragma unroll
          for (int j = 0; j < 8; ++j) b[r][j] = f[j] > b[r][j] ? f[j] : b[r][j];
        }
      }
    }
  }
  const int64_t o = (int64_t(n) * P + p) * Q + q;
#pragma unroll
  for (int r = 0; r < RPB; ++r) reinterpret_cast<uint4*>(y)[(o + r * Q) * cg + (c0 >> 3)] = pack8(b[r]);
}

// Backward in two deterministic passes (no atomics):
//   1. per output window, the first-in-scan-order argmax (0..8) of each
//      channel -> one byte per output element (transient workspace);
//   2. per input pixel, sum the gradient of the <= 4 windows whose argmax it is.
// two output rows per block (P even), as k_maxpool_fwd<2>: scan order and
// the first-maximum rule per window are unchanged
__global__ void __launch_bounds__(256)
    k_maxpool_argmax(const bf16* __restrict__ x, uint8_t* __restrict__ idx, int N, int H, int W,
                     int C, int P, int Q, int lcg) {
  pdl_wait();
  pdl_trigger();
  const int cg = 1 << lcg;
  const int item = blockIdx.y * 256 + threadIdx.x;
  if (item >= Q * cg) return;
  const int q = item >> lcg, c0 = (item & (cg - 1)) * 8;
  const int pp = P >> 1;
  const int n = blockIdx.x / pp, p = (blockIdx.x - n * pp) * 2;
  const uint4 ninf = make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
  uint4 v[15];  // input rows 2p-1 .. 2p+3 x columns 2q-1 .. 2q+1
#pragma unroll
  for (int k = 0; k < 15; ++k) {
    const int h = 2 * p - 1 + k / 3, w = 2 * q - 1 + k % 3;
    const bool ok = (unsigned)h < (unsigned)H && (unsigned)w < (unsigned)W;
    v[k] = ok ? *reinterpret_cast<const uint4*>(x + ((int64_t(n) * H + h) * W + w) * C + c0)
              : ninf;
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    float best[8];
    uint32_t arg[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      best[j] = -INFINITY;
      arg[j] = 0;
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      float f[8];
      unpack8(v[r * 6 + k], f);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (f[j] > best[j]) {
          best[j] = f[j];
          arg[j] = k;
        }
    }
    uint2 packed;
    packed.x = arg[0] | (arg[1] << 8) | (arg[2] << 16) | (arg[3] << 24);
    packed.y = arg[4] | (arg[5] << 8) | (arg[6] << 16) | (arg[7] << 24);
    reinterpret_cast<uint2*>(idx)[((int64_t(n) * P + p + r) * Q + q) * cg + (c0 >> 3)] = packed;
  }
}

// Thread per (output window (p, q), 8 channels): writes the 2x2 input block
// rows {2p, 2p+1} x cols {2q, 2q+1} (H = 2P, W = 2Q: a partition of the
// input).  Even rows/cols lie in one window, odd ones in two: the block sums
// windows (p..p+1, q..q+1), in a fixed order, where their argmax lands.
__global__ void __launch_bounds__(256)
    k_maxpool_bwd_gather(const bf16* __restrict__ dy, const uint8_t* __restrict__ idx,
                         bf16* __restrict__ dx, int N, int H, int W, int C, int P, int Q,
                         int lcg) {
  pdl_wait();
  pdl_trigger();
  const int cg = 1 << lcg;
  const int item = blockIdx.y * 256 + threadIdx.x;
  if (item >= Q * cg) return;
  const int q = item >> lcg, c0 = (item & (cg - 1)) * 8;
  const int n = blockIdx.x / P, p = blockIdx.x - n * P;
  float acc[4][8];
#pragma unroll
  for (int b = 0; b < 4; ++b)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[b][j] = 0.f;
  // the (up to) 4 windows' argmax bytes and gradients, loaded up front
  uint2 av[4];
  uint4 gv[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int pp = p + (t >> 1), qq = q + (t & 1);
    const bool ok = pp < P && qq < Q;
    const int64_t o = ((int64_t(n) * P + pp) * Q + qq) * C + c0;
    av[t] = ok ? *reinterpret_cast<const uint2*>(idx + o) : make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);
    gv[t] = ok ? *reinterpret_cast<const uint4*>(dy + o) : make_uint4(0u, 0u, 0u, 0u);
  }
#pragma unroll
  for (int dp = 0; dp < 2; ++dp)
#pragma unroll
    for (int dq = 0; dq < 2; ++dq) {
      const int pp = p + dp, qq = q + dq;
      const uint2 a = av[dp * 2 + dq];  // 0xFF never matches a tap (0..8)
      float g[8];
      unpack8(gv[dp * 2 + dq], g);
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        // input pixel (2p + (b>>1), 2q + (b&1)) inside window (pp, qq) at tap k
        const int h = 2 * p + (b >> 1), w = 2 * q + (b & 1);
        const int kh = h - (2 * pp - 1), kw = w - (2 * qq - 1);
        if (kh < 0 || kh > 2 || kw < 0 || kw > 2) continue;
        const uint32_t k = uint32_t(kh * 3 + kw);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t aj = ((j < 4 ? a.x : a.y) >> (8 * (j & 3))) & 0xFF;
          if (aj == k) acc[b][j] += g[j];
        }
      }
    }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int h = 2 * p + (b >> 1), w = 2 * q + (b & 1);
    if (h < H && w < W)
      reinterpret_cast<uint4*>(dx)[((int64_t(n) * H + h) * W + w) * cg + (c0 >> 3)] =
          pack8(acc[b]);
  }
}

__global__ void __launch_bounds__(256) k_avgpool_fwd(const bf16* __restrict__ x,
                                                     bf16* __restrict__ y, int N, int HW, int C) {
  pdl_wait();
  pdl_trigger();
  const int cg = C / 8;
  const int64_t total = int64_t(N) * cg;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int c0 = int(i % cg) * 8;
    const int n = int(i / cg);
    float s[8] = {0};
    for (int k = 0; k < HW; ++k) {
      float f[8];
      unpack8(*reinterpret_cast<const uint4*>(x + (int64_t(n) * HW + k) * C + c0), f);
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j] += f[j];
    }
    const float inv = 1.f / float(HW);
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] *= inv;
    reinterpret_cast<uint4*>(y)[i] = pack8(s);
  }
}

// ------------------------------------------------------- softmax x-entropy
__global__ void __launch_bounds__(256) k_softmax_xent(const float* __restrict__ logits,
                                                      const int64_t* __restrict__ labels,
                                                      float* __restrict__ dlogits,
                                                      float* __restrict__ row_loss, int N, int K) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.x;
  const float* l = logits + int64_t(n) * K;
  __shared__ float red[256];
  float mx = -INFINITY;
  for (int k = threadIdx.x; k < K; k += blockDim.x) mx = fmaxf(mx, l[k]);
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  mx = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int k = threadIdx.x; k < K; k += blockDim.x) sum += __expf(l[k] - mx);
  red[threadIdx.x] = sum;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  sum = red[0];
  const int lab = int(labels[n]);
  const float invN = 1.f / float(N);
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const float p = __expf(l[k] - mx) / sum;
    dlogits[int64_t(n) * K + k] = (p - (k == lab ? 1.f : 0.f)) * invN;
  }
  if (threadIdx.x == 0) row_loss[n] = logf(sum) + mx - l[lab];
}

// The classifier head on the tensor-core GEMM's bf16 logits ([N][ld], the
// class dimension padded to ld): logits + bias in fp32, softmax cross-entropy
// per row -> row loss, dlogits (fp32 [N][K]) and its bf16 copy [N][ld] with
// zero pad columns (the A operand of the head's input- and weight-gradient
// GEMMs).
__global__ void __launch_bounds__(256) k_softmax_xent_head(
    const bf16* __restrict__ logits, int ld, const float* __restrict__ bias,
    const int64_t* __restrict__ labels, float* __restrict__ dlogits, bf16* __restrict__ dl_bf16,
    float* __restrict__ row_loss, int N, int K) {
  pdl_wait();
  pdl_trigger();
  const int n = blockIdx.x;
  const bf16* l = logits + int64_t(n) * ld;
  __shared__ float red[256];
  __shared__ float z[1024];
  float mx = -INFINITY;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    const float v = __bfloat162float(l[k]) + bias[k];
    if (k < 1024) z[k] = v;
    mx = fmaxf(mx, v);
  }
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  mx = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int k = threadIdx.x; k < K; k += blockDim.x) sum += __expf(z[k] - mx);
  red[threadIdx.x] = sum;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  sum = red[0];
  const int lab = int(labels[n]);
  const float invN = 1.f / float(N);
  for (int k = threadIdx.x; k < ld; k += blockDim.x) {
    float d = 0.f;
    if (k < K) {
      d = (__expf(z[k] - mx) / sum - (k == lab ? 1.f : 0.f)) * invN;
      dlogits[int64_t(n) * K + k] = d;
    }
    dl_bf16[int64_t(n) * ld + k] = __float2bfloat16_rn(d);
  }
  if (threadIdx.x == 0) row_loss[n] = logf(sum) + mx - z[lab];
}

// column sums of an fp32 [N][K] matrix in a fixed (row) order: the bias gradient
__global__ void __launch_bounds__(256) k_col_sums(const float* __restrict__ a, int N, int K,
                                                  float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  float s = 0.f;
  for (int n = 0; n < N; ++n) s += a[int64_t(n) * K + k];
  out[k] = s;
}

__global__ void k_mean_rows(const float* row_loss, int N, float* loss) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    float s = 0.f;
    for (int i = 0; i < N; ++i) s += row_loss[i];
    *loss = s / float(N);
  }
}

}  // namespace

// The BN workspace: kBarFloats words of grid-barrier state (zeroed once at
// allocation, left zero-count by every launch), then the partial rows.
constexpr int64_t kBarFloats = 64;
int64_t bn_workspace_floats(int64_t M, int C) {
  const int64_t chunk = chunk_rows(M, C);
  const int64_t chunks = (M + chunk - 1) / chunk;
  return kBarFloats + 2 * (chunks + (chunks + GROUP - 1) / GROUP) * C;
}

namespace {
// Merge `parts` (mean, M2) partials of `rows_per` rows (the last shorter) at
// ws[0 .. parts*C) into the channel statistics.  Above 2*GROUP partials a
// grouping pass first writes ceil(parts/GROUP) partials after them (the
// caller's buffer holds both), so each merge warp walks at most a few dozen.
cudaError_t merge_partials(const float2* ws, int parts, int64_t rows_per, int64_t M, int C,
                           float* mean, float* invstd, float eps, float* rm, float* rv, float mom,
                           cudaStream_t st) {
  if (parts > group_above()) {
    const int groups = (parts + GROUP - 1) / GROUP;
    float2* out = const_cast<float2*>(ws) + int64_t(parts) * C;
    const int bx = C < 256 ? C : 256;
    if (cudaError_t e_ = launch_k(k_bn_stats_group, dim3(dim3((C + bx - 1) / bx, groups)), dim3(bx), 0, st, ws, parts, rows_per, M, C, out)) return e_;
    ws = out;
    parts = groups;
    rows_per *= GROUP;
  }
  return launch_k(k_bn_stats_merge, dim3((C + 7) / 8), dim3(256), 0, st, ws, parts, rows_per, M, C,
                  mean, invstd, eps, rm, rv, mom);
}
}  // namespace

cudaError_t bn_stats(const void* x, int64_t M, int C, float* ws, float* mean, float* invstd,
                     float eps, float* rm, float* rv, float mom, cudaStream_t st) {
  if (C % SLICE || (C & (C - 1)) || C > 2048) return cudaErrorInvalidValue;
  ws += kBarFloats;
  const int64_t chunk = chunk_rows(M, C);
  const int chunks = int((M + chunk - 1) / chunk);
  if (cudaError_t e_ = launch_k(k_bn_stats_partial, dim3(chunks), dim3(256), 0, st, static_cast<const bf16*>(x), M, C, chunk, reinterpret_cast<float2*>(ws))) return e_;
  return merge_partials(reinterpret_cast<const float2*>(ws), chunks, chunk, M, C, mean, invstd, eps,
                        rm, rv, mom, st);
}

int stats_parts() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int64_t stats_partials_floats(int C) { return int64_t(stats_parts()) * C * 4; }

cudaError_t bn_stats_from_partials(const float* partials, int C, float* mean, float* invstd,
                                   float eps, float* rm, float* rv, float mom, cudaStream_t st) {
  return launch_k(k_bn_stats_merge_cta, dim3((C + 7) / 8), dim3(256), 0, st,
                  reinterpret_cast<const float4*>(partials), stats_parts(), C, mean, invstd, eps,
                  rm, rv, mom);
}

cudaError_t bn_apply(int mode, const void* x, const void* res, void* y, int64_t M, int C,
                     const float* mean, const float* invstd, const float* gamma, const float* beta,
                     const float* mean2, const float* invstd2, const float* gamma2,
                     const float* beta2, cudaStream_t st) {
  if ((C & (C - 1)) || C < 8 || C > 2048) return cudaErrorInvalidValue;
  const int64_t vecs = M * C / 8;
  const int grid = grid_for(vecs, 256);
  auto X = static_cast<const bf16*>(x);
  auto R = static_cast<const bf16*>(res);
  auto Y = static_cast<bf16*>(y);
  switch (mode) {
    case 0:
      if (cudaError_t e_ = launch_k(k_bn_apply<0>, dim3(grid), dim3(256), 0, st, X, R, Y, vecs, C - 1, mean, invstd, gamma, beta, nullptr, nullptr, nullptr, nullptr)) return e_;
      break;
    case 1:
      if (cudaError_t e_ = launch_k(k_bn_apply<1>, dim3(grid), dim3(256), 0, st, X, R, Y, vecs, C - 1, mean, invstd, gamma, beta, nullptr, nullptr, nullptr, nullptr)) return e_;
      break;
    default:
      if (cudaError_t e_ = launch_k(k_bn_apply<2>, dim3(grid), dim3(256), 0, st, X, R, Y, vecs, C - 1, mean, invstd, gamma, beta, mean2, invstd2, gamma2, beta2)) return e_;
  }
  return cudaGetLastError();
}

// DELTA_BN_BWD_GRID=0: the three-launch BN backward (partial, merge, apply)
bool bn_bwd_one_launch() {
  static const bool on = [] {
    const char* e = std::getenv("DELTA_BN_BWD_GRID");
    return !(e && e[0] == '0');
  }();
  return on;
}

// CTAs of `kernel` (block threads, no dynamic smem) resident at once on the
// current device, capped by the workspace's partial rows (bn_workspace_floats)
template <typename K>
int resident_ctas(K kernel, int threads) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
  const int cap = sms * (per_sm > 0 ? per_sm : 1);
  return cap < 148 * 8 ? cap : 148 * 8;
}

cudaError_t bn_backward(const void* up, int pool_hw, const void* mask, const void* x, void* dx,
                        int64_t M, int C, const float* mean, const float* invstd,
                        const float* gamma, float* dgamma, float* dbeta, float* ws,
                        cudaStream_t st) {
  if (C % SLICE || (C & (C - 1)) || C > 2048) return cudaErrorInvalidValue;
  auto U = static_cast<const bf16*>(up);
  auto Mk = static_cast<const bf16*>(mask);
  auto X = static_cast<const bf16*>(x);
  auto* bar = reinterpret_cast<unsigned int*>(ws);
  ws += kBarFloats;
  if (bn_bwd_one_launch()) {
    const auto k = Mk ? (pool_hw ? k_bn_bwd_grid<true, true> : k_bn_bwd_grid<true, false>)
                      : (pool_hw ? k_bn_bwd_grid<false, true> : k_bn_bwd_grid<false, false>);
    const int cap = resident_ctas(k, 256);
    int64_t chunk = (M + cap - 1) / cap;
    chunk = (chunk + 15) / 16 * 16;
    const int grid = int((M + chunk - 1) / chunk);
    // cooperative: the runtime guarantees every CTA co-resident (even beside
    // kernels on other streams) or refuses the launch; a refusal falls back
    // to the three-launch path below
    const cudaError_t e_ = launch_coop(k, dim3(grid), dim3(256), 0, st, U, pool_hw, Mk, X,
                                       static_cast<bf16*>(dx), M, C, chunk, mean, invstd, gamma,
                                       dgamma, dbeta, reinterpret_cast<float2*>(ws), bar);
    if (e_ == cudaSuccess) return cudaGetLastError();
    if (e_ != cudaErrorCooperativeLaunchTooLarge) return e_;
    cudaGetLastError();  // clear the refusal
  }
  const int64_t chunk = chunk_rows(M, C);
  const int chunks = int((M + chunk - 1) / chunk);
  const auto part = Mk ? (pool_hw ? k_bn_bwd_partial<true, true> : k_bn_bwd_partial<true, false>)
                      : (pool_hw ? k_bn_bwd_partial<false, true> : k_bn_bwd_partial<false, false>);
  if (cudaError_t e_ = launch_k(part, dim3(chunks), dim3(256), 0, st, U, pool_hw, Mk, X, M, C, chunk, mean, invstd, reinterpret_cast<float2*>(ws))) return e_;
  const float2* w2 = reinterpret_cast<const float2*>(ws);
  int parts = chunks;
  if (parts > group_above()) {  // two-level fixed-order sum (scratch after the partials)
    const int groups = (parts + GROUP - 1) / GROUP;
    float2* out = reinterpret_cast<float2*>(ws) + int64_t(parts) * C;
    const int bx = C < 256 ? C : 256;
    if (cudaError_t e_ = launch_k(k_bn_bwd_group, dim3(dim3((C + bx - 1) / bx, groups)), dim3(bx), 0, st, w2, parts, C, out)) return e_;
    w2 = out;
    parts = groups;
  }
  if (cudaError_t e_ = launch_k(k_bn_bwd_final, dim3((C + 7) / 8), dim3(256), 0, st, w2, parts, C, dgamma, dbeta)) return e_;
  const int64_t vecs = M * C / 8;
  const auto app = Mk ? (pool_hw ? k_bn_bwd_apply<true, true> : k_bn_bwd_apply<true, false>)
                     : (pool_hw ? k_bn_bwd_apply<false, true> : k_bn_bwd_apply<false, false>);
  if (cudaError_t e_ = launch_k(app, dim3(grid_for(vecs, 256)), dim3(256), 0, st, U, pool_hw, Mk, X, static_cast<bf16*>(dx), vecs, C - 1, __builtin_ctz(C), M, mean, invstd, gamma, dgamma, dbeta)) return e_;
  return cudaGetLastError();
}

cudaError_t bn_backward_from_partials(const float* partials, const void* g, const void* x,
                                      void* dx, int64_t M, int C, const float* mean,
                                      const float* invstd, const float* gamma, float* dgamma,
                                      float* dbeta, cudaStream_t st) {
  if (C % SLICE || (C & (C - 1)) || C > 2048) return cudaErrorInvalidValue;
  if (cudaError_t e_ = launch_k(k_bn_bwd_final_cta, dim3((C + 7) / 8), dim3(256), 0, st,
                                reinterpret_cast<const float4*>(partials), stats_parts(), C, mean,
                                invstd, dgamma, dbeta))
    return e_;
  const int64_t vecs = M * C / 8;
  const auto app = g == dx ? k_bn_bwd_apply<false, false, true> : k_bn_bwd_apply<false, false>;
  return launch_k(app, dim3(grid_for(vecs, 256)), dim3(256), 0, st,
                  static_cast<const bf16*>(g), 0, nullptr, static_cast<const bf16*>(x),
                  static_cast<bf16*>(dx), vecs, C - 1, __builtin_ctz(C), M, mean, invstd, gamma,
                  dgamma, dbeta);
}

cudaError_t stats_col_sum(const float* partials, int C, float* out, int accumulate,
                          cudaStream_t st) {
  return launch_k(k_stats_col_sum, dim3((C + 7) / 8), dim3(256), 0, st,
                  reinterpret_cast<const float4*>(partials), stats_parts(), C, out, accumulate);
}

cudaError_t add_grad(const void* a, const void* up, int pool_hw, const void* up_mask,
                     const void* out_mask, void* out, int64_t M, int C, cudaStream_t st) {
  if (C & (C - 1)) return cudaErrorInvalidValue;
  const int64_t vecs = M * C / 8;
  if (cudaError_t e_ = launch_k((pool_hw ? k_add_grad<true> : k_add_grad<false>), dim3(grid_for(vecs, 256)), dim3(256), 0, st, static_cast<const bf16*>(a), static_cast<const bf16*>(up), pool_hw, static_cast<const bf16*>(up_mask), static_cast<const bf16*>(out_mask), static_cast<bf16*>(out), vecs, C - 1, __builtin_ctz(C), C)) return e_;
  return cudaGetLastError();
}

cudaError_t maxpool3x3s2_fwd(const void* x, void* y, int N, int H, int W, int C, cudaStream_t st) {
  const int P = (H + 2 - 3) / 2 + 1, Q = (W + 2 - 3) / 2 + 1;
  if (C % 8 || ((C / 8) & (C / 8 - 1))) return cudaErrorInvalidValue;
  const int lcg = __builtin_ctz(C / 8);
  static const int rpb_env = [] {
    const char* e = std::getenv("DELTA_MAXPOOL_RPB");
    return e ? std::atoi(e) : 2;
  }();
  const int rpb = P % rpb_env == 0 ? rpb_env : (P % 2 == 0 ? 2 : 1);
  const auto k = rpb == 4 ? k_maxpool_fwd<4> : (rpb == 2 ? k_maxpool_fwd<2> : k_maxpool_fwd<1>);
  if (cudaError_t e_ = launch_k(k, dim3(dim3(unsigned(N) * (P / rpb), (Q * (C / 8) + 255) / 256)), dim3(256), 0, st, static_cast<const bf16*>(x), static_cast<bf16*>(y), N, H, W, C, P, Q, lcg)) return e_;
  return cudaGetLastError();
}

int64_t maxpool_workspace_bytes(int N, int H, int W, int C) {
  const int P = (H + 2 - 3) / 2 + 1, Q = (W + 2 - 3) / 2 + 1;
  return int64_t(N) * P * Q * C;
}

cudaError_t maxpool3x3s2_bwd(const void* dy, const void* x, void* dx, int N, int H, int W, int C,
                             void* ws, cudaStream_t st) {
  const int P = (H + 2 - 3) / 2 + 1, Q = (W + 2 - 3) / 2 + 1;
  if (C % 8 || ((C / 8) & (C / 8 - 1))) return cudaErrorInvalidValue;
  const int lcg = __builtin_ctz(C / 8);
  if (P & 1) return cudaErrorInvalidValue;  // argmax: two output rows per block
  if (cudaError_t e_ = launch_k(k_maxpool_argmax, dim3(dim3(unsigned(N) * (P / 2), (Q * (C / 8) + 255) / 256)), dim3(256), 0, st, static_cast<const bf16*>(x), static_cast<uint8_t*>(ws), N, H, W, C, P, Q, lcg)) return e_;
  if (H != 2 * P || W != 2 * Q) return cudaErrorInvalidValue;  // even input sizes
  if (cudaError_t e_ = launch_k(k_maxpool_bwd_gather, dim3(dim3(unsigned(N) * P, (Q * (C / 8) + 255) / 256)), dim3(256), 0, st, static_cast<const bf16*>(dy), static_cast<const uint8_t*>(ws), static_cast<bf16*>(dx), N, H, W, C, P, Q, lcg)) return e_;
  return cudaGetLastError();
}

cudaError_t avgpool_fwd(const void* x, void* y, int N, int HW, int C, cudaStream_t st) {
  const int64_t total = int64_t(N) * (C / 8);
  if (cudaError_t e_ = launch_k(k_avgpool_fwd, dim3(grid_for(total, 128)), dim3(128), 0, st, static_cast<const bf16*>(x), static_cast<bf16*>(y), N, HW, C)) return e_;
  return cudaGetLastError();
}

cudaError_t softmax_xent_head(const void* logits, int ld, const float* bias,
                              const int64_t* labels, float* loss, float* dlogits, void* dl_bf16,
                              float* dbias, float* row_loss_ws, int N, int K, cudaStream_t st) {
  if (K > 1024 || ld < K || (ld & 7)) return cudaErrorInvalidValue;
  if (cudaError_t e_ = launch_k(k_softmax_xent_head, dim3(N), dim3(256), 0, st,
                                static_cast<const bf16*>(logits), ld, bias, labels, dlogits,
                                static_cast<bf16*>(dl_bf16), row_loss_ws, N, K))
    return e_;
  if (cudaError_t e_ = launch_k(k_col_sums, dim3((K + 255) / 256), dim3(256), 0, st,
                                static_cast<const float*>(dlogits), N, K, dbias))
    return e_;
  if (cudaError_t e_ = launch_k(k_mean_rows, dim3(1), dim3(32), 0, st, row_loss_ws, N, loss))
    return e_;
  return cudaGetLastError();
}

cudaError_t softmax_xent(const float* logits, const int64_t* labels, float* loss, float* dlogits,
                         float* row_loss_ws, int N, int K, cudaStream_t st) {
  if (cudaError_t e_ = launch_k(k_softmax_xent, dim3(N), dim3(256), 0, st, logits, labels, dlogits, row_loss_ws, N, K)) return e_;
  if (cudaError_t e_ = launch_k(k_mean_rows, dim3(1), dim3(32), 0, st, row_loss_ws, N, loss)) return e_;
  return cudaGetLastError();
}

}  // namespace delta_k
