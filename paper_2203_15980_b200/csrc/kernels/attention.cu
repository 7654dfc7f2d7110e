// Multi-head attention for sm_100a (tcgen05 + TMEM + TMA): the Attention node
// of the reference's transformer trace (ref src/trace.cpp:452) and its
// backward, with attention-probability dropout whose mask is replayed
// (philox.cuh), so a recomputed Attention output is bit-identical.
//
// BERT shapes: head dim 64, sequence S <= 512 (a multiple of 128).  One CTA
// owns one 128-row tile of one (sequence, head) and keeps the WHOLE key range
// on chip — no online-softmax rescaling:
//
// forward (grid S/128 x heads x B): S = Q K^T for all S keys in TMEM (S <= 512
//   fp32 columns = the SM's whole TMEM); 8 softmax warps (two per TMEM lane
//   quarter, each half of the keys) take the row max, then write
//   P = exp2(s*c - m*c) * keep (bf16, unnormalised) to shared memory in the
//   K-major SW128 layout the tensor core reads; K's buffer is refilled with V
//   meanwhile; O = P V (B operand V MN-major) lands in TMEM columns 0-63 and is
//   scaled by dropout_scale / rowsum on the way out.  lse (log2 units) saved.
// backward: two roles of one kernel, both recomputing S and dP = dO V^T per
//   128 x 128 block (thread = one query row, the saved lse and D = rowsum(dO*O)
//   in registers): dS = P (dP*keep*scale - D);
//   ROLE_DQ  (tile = 128 queries, loop over key blocks):  dQ += dS K
//   ROLE_DKV (tile = 128 keys, loop over query blocks):   dV += (P*keep*scale)^T dO,
//                                                          dK += dS^T Q
//   (the transposed products read the same [query][key] smem tiles through
//   MN-major descriptors).  No atomics: every output element is written once,
//   so gradients are deterministic.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels/launch.hpp"
#include "kernels/philox.cuh"
#include "kernels/sm100_common.cuh"
#include "kernels/tma_host.hpp"
#include "kernels/xformer.hpp"

namespace delta_k {

using namespace dsm100;

namespace {

using bf16 = __nv_bfloat16;
constexpr int HD = 64;            // head dim
constexpr int TILE = 128;         // rows per tile
constexpr uint32_t TILE_BYTES = TILE * 128;  // a [128][64] bf16 SW128 tile
constexpr int kThreads = 9 * 32;  // 8 math warps + 1 control warp
constexpr int CTRL = 8;
constexpr float kScale = 0.125f;                              // 1/sqrt(64)
constexpr float kCl2 = 0.125f * 1.4426950408889634f;          // scale * log2(e)

// MN-major operand, 128-byte swizzle (see wgrad.cu): rows of 128 B along MN,
// 8-row K groups 1 KB apart, MN atoms `lbo` bytes apart
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= uint64_t((addr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

__device__ __forceinline__ void bar_math() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// 32 consecutive bf16 of row r at key column `col` (multiple of 32) of a
// [128][ncols] K-major SW128 tile set (64-column atoms of 16 KB)
__device__ __forceinline__ void st_row32(uint32_t base, int r, int col, const uint32_t* w) {
  const uint32_t atom = base + uint32_t(col >> 6) * TILE_BYTES + uint32_t(r) * 128;
  const int u0 = (col & 63) >> 3;
#pragma unroll
  for (int u = 0; u < 4; ++u)
    st_shared_v4(atom + ((uint32_t((u0 + u) ^ (r & 7))) << 4),
                 make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]));
}

struct AttnArgs {
  int B, S, heads;
  int Hd;        // heads * 64
  bf16* out;     // fwd: [T][Hd]; bwd: dqkv [T][3 Hd]
  float* lse;    // [B*heads][S]
  const float* D;
  uint32_t thr;
  float dscale;
  const uint64_t* rng;
  uint32_t tag;
};

// ======================================================================= fwd
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_fwd(const __grid_constant__ CUtensorMap qkv_map, const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = a.S;
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sKV = sQ + TILE_BYTES;
  const uint32_t sP = sKV + uint32_t(S) * 128;
  float* red = reinterpret_cast<float*>(smem + TILE_BYTES + size_t(S) * 128 + size_t(S) * 256);
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 4 * TILE);
  uint64_t* bar_qk = bars;
  uint64_t* bar_v = bars + 1;
  uint64_t* bar_s = bars + 2;
  uint64_t* bar_p = bars + 3;
  uint64_t* bar_o = bars + 4;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 5);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const uint32_t tcols = S <= 128 ? 128 : (S <= 256 ? 256 : 512);

  if (threadIdx.x == 0) {
    mbar_init(bar_qk, 1);
    mbar_init(bar_v, 1);
    mbar_init(bar_s, 1);
    mbar_init(bar_p, 8);
    mbar_init(bar_o, 1);
    fence_mbar_init();
    tma_prefetch_desc(&qkv_map);
  }
  if (warp == CTRL) tmem_alloc(tslot, tcols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  pdl_trigger();
  const int row0 = b * S;  // first token of the sequence

  if (warp == CTRL) {
    if (lane == 0) {
      mbar_arrive_expect_tx(bar_qk, TILE_BYTES + uint32_t(S) * 128);
      tma_load_2d(sQ, &qkv_map, bar_qk, h * HD, row0 + qt * TILE);
      for (int i = 0; i < S / TILE; ++i)
        tma_load_2d(sKV + i * TILE_BYTES, &qkv_map, bar_qk, a.Hd + h * HD, row0 + i * TILE);
    }
    mbar_wait(bar_qk, 0);
    tc_fence_after();
    constexpr uint32_t idS = umma_idesc_bf16(128, 128);
    if (elect_one()) {
      const uint64_t dq = umma_desc_sw128(sQ);
      for (int nb = 0; nb < S / TILE; ++nb) {
        const uint64_t dk = umma_desc_sw128(sKV + nb * TILE_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + nb * TILE, dq + uint64_t(k * 2), dk + uint64_t(k * 2), idS, k > 0);
      }
      umma_commit(bar_s);
    }
    __syncwarp();
    // K consumed: refill the buffer with V while the softmax runs
    mbar_wait(bar_s, 0);
    if (lane == 0) {
      mbar_arrive_expect_tx(bar_v, uint32_t(S) * 128);
      for (int i = 0; i < S / TILE; ++i)
        tma_load_2d(sKV + i * TILE_BYTES, &qkv_map, bar_v, 2 * a.Hd + h * HD, row0 + i * TILE);
    }
    mbar_wait(bar_v, 0);
    mbar_wait(bar_p, 0);
    tc_fence_after();
    constexpr uint32_t idO = umma_idesc_bf16(128, HD) | (1u << 16);  // B (V) MN-major
    if (elect_one()) {
      for (int j = 0; j < S / 64; ++j) {
        const uint64_t dp = umma_desc_sw128(sP + j * TILE_BYTES);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16(tmem, dp + uint64_t(k * 2), desc_mn(sKV + uint32_t(j * 64 + k * 16) * 128, 0),
                    idO, (j | k) != 0);
      }
      umma_commit(bar_o);
    }
    __syncwarp();
  } else {
    // ---- softmax warps: row r of the tile, keys [half*S/2, (half+1)*S/2) ----
    const int quarter = warp & 3, half = warp >> 2;
    const int r = quarter * 32 + lane;
    const int q = qt * TILE + r;
    const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16);
    const int hs = S / 2, nch = hs / 32;
    mbar_wait(bar_s, 0);
    tc_fence_after();
    float m = -INFINITY;
    for (int c = 0; c < nch; ++c) {
      float v[32];
      tmem_ld_32x32b_x32(trow + half * hs + c * 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) m = fmaxf(m, v[i]);
    }
    red[half * TILE + r] = m;
    bar_math();
    m = fmaxf(red[r], red[TILE + r]);
    const float mc = m * kCl2;
    const uint64_t seed = a.rng[0], step = a.rng[1];
    const uint64_t erow = (uint64_t(b * a.heads + h) * S + q) * uint64_t(S);
    float l = 0.f;
    for (int c = 0; c < nch; ++c) {
      float v[32];
      const int col = half * hs + c * 32;
      tmem_ld_32x32b_x32(trow + col, v);
      uint32_t keep = 0xFFFFFFFFu;
      if (a.thr) {
        const uint64_t g = (erow + col) >> 4;
        keep = keep16(drop_block(seed, step, a.tag, g), a.thr) |
               (keep16(drop_block(seed, step, a.tag, g + 1), a.thr) << 16);
      }
      uint32_t w[16];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float p0 = ex2(fmaf(v[i], kCl2, -mc));
        const float p1 = ex2(fmaf(v[i + 1], kCl2, -mc));
        l += p0 + p1;
        w[i >> 1] = pack_bf16x2((keep >> i) & 1u ? p0 : 0.f, (keep >> (i + 1)) & 1u ? p1 : 0.f);
      }
      st_row32(sP, r, col, w);
    }
    red[2 * TILE + half * TILE + r] = l;
    fence_proxy_async_smem();
    tc_fence_before();
    bar_math();
    l = red[2 * TILE + r] + red[3 * TILE + r];
    if (half == 0) a.lse[uint64_t(b * a.heads + h) * S + q] = mc + __log2f(l);
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_p);
    const float inv = a.dscale / l;
    // ---- epilogue: O columns [half*32, half*32+32) of row r ----
    mbar_wait(bar_o, 0);
    tc_fence_after();
    float v[32];
    tmem_ld_32x32b_x32(trow + half * 32, v);
    uint4* dst = reinterpret_cast<uint4*>(a.out + (int64_t(row0) + q) * a.Hd + h * HD + half * 32);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      dst[u] = make_uint4(pack_bf16x2(v[8 * u] * inv, v[8 * u + 1] * inv),
                          pack_bf16x2(v[8 * u + 2] * inv, v[8 * u + 3] * inv),
                          pack_bf16x2(v[8 * u + 4] * inv, v[8 * u + 5] * inv),
                          pack_bf16x2(v[8 * u + 6] * inv, v[8 * u + 7] * inv));
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == CTRL) tmem_dealloc(tmem, tcols);
}

// ======================================================================= bwd
constexpr int ROLE_DQ = 0, ROLE_DKV = 1;

template <int ROLE>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_bwd(const __grid_constant__ CUtensorMap qkv_map, const __grid_constant__ CUtensorMap do_map,
               const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = a.S;
  const int nt = S / TILE;
  // ROLE_DQ : sA0 = Q_i, sA1 = dO_i, sB0 = K (all), sB1 = V (all)
  // ROLE_DKV: sA0 = K_j, sA1 = V_j,  sB0 = Q (all), sB1 = dO (all)
  const uint32_t sA0 = smem_u32(smem);
  const uint32_t sA1 = sA0 + TILE_BYTES;
  const uint32_t sB0 = sA1 + TILE_BYTES;
  const uint32_t sB1 = sB0 + uint32_t(S) * 128;
  const uint32_t sDS = sB1 + uint32_t(S) * 128;  // dS [128 q][128 keys]
  const uint32_t sPD = sDS + 2 * TILE_BYTES;     // ROLE_DKV: P*keep*scale, same layout
  const uint32_t used = 2 * TILE_BYTES + 2 * uint32_t(S) * 128 + (ROLE == ROLE_DKV ? 4 : 2) * TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + used);
  uint64_t* bar_ld = bars;
  uint64_t* bar_sp = bars + 1;
  uint64_t* bar_ds = bars + 2;
  uint64_t* bar_acc = bars + 3;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int row0 = b * S;

  if (threadIdx.x == 0) {
    mbar_init(bar_ld, 1);
    mbar_init(bar_sp, 1);
    mbar_init(bar_ds, 8);
    mbar_init(bar_acc, 1);
    fence_mbar_init();
    tma_prefetch_desc(&qkv_map);
    tma_prefetch_desc(&do_map);
  }
  if (warp == CTRL) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  pdl_trigger();
  // TMEM: S [0,128), dP [128,256), acc0 (dQ | dV) [256,320), acc1 (dK) [320,384)
  if (warp == CTRL) {
    if (lane == 0) {
      mbar_arrive_expect_tx(bar_ld, 2 * TILE_BYTES + 2 * uint32_t(S) * 128);
      if (ROLE == ROLE_DQ) {
        tma_load_2d(sA0, &qkv_map, bar_ld, h * HD, row0 + tile * TILE);
        tma_load_2d(sA1, &do_map, bar_ld, h * HD, row0 + tile * TILE);
        for (int i = 0; i < nt; ++i) {
          tma_load_2d(sB0 + i * TILE_BYTES, &qkv_map, bar_ld, a.Hd + h * HD, row0 + i * TILE);
          tma_load_2d(sB1 + i * TILE_BYTES, &qkv_map, bar_ld, 2 * a.Hd + h * HD, row0 + i * TILE);
        }
      } else {
        tma_load_2d(sA0, &qkv_map, bar_ld, a.Hd + h * HD, row0 + tile * TILE);
        tma_load_2d(sA1, &qkv_map, bar_ld, 2 * a.Hd + h * HD, row0 + tile * TILE);
        for (int i = 0; i < nt; ++i) {
          tma_load_2d(sB0 + i * TILE_BYTES, &qkv_map, bar_ld, h * HD, row0 + i * TILE);
          tma_load_2d(sB1 + i * TILE_BYTES, &do_map, bar_ld, h * HD, row0 + i * TILE);
        }
      }
    }
    mbar_wait(bar_ld, 0);
    tc_fence_after();
    constexpr uint32_t idS = umma_idesc_bf16(128, 128);
    // S = Q K^T and dP = dO V^T of block `it` (rows = queries, cols = keys)
    auto issue_sp = [&](int it) {
      uint32_t q_, k_, do_, v_;
      if (ROLE == ROLE_DQ) {
        q_ = sA0; do_ = sA1; k_ = sB0 + it * TILE_BYTES; v_ = sB1 + it * TILE_BYTES;
      } else {
        q_ = sB0 + it * TILE_BYTES; do_ = sB1 + it * TILE_BYTES; k_ = sA0; v_ = sA1;
      }
      if (elect_one()) {
        const uint64_t dq = umma_desc_sw128(q_), dk = umma_desc_sw128(k_);
        const uint64_t dd = umma_desc_sw128(do_), dv = umma_desc_sw128(v_);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem, dq + uint64_t(k * 2), dk + uint64_t(k * 2), idS, k > 0);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + 128, dd + uint64_t(k * 2), dv + uint64_t(k * 2), idS, k > 0);
        umma_commit(bar_sp);
      }
      __syncwarp();
    };
    issue_sp(0);
    for (int it = 0; it < nt; ++it) {
      mbar_wait(bar_ds, it & 1);
      tc_fence_after();
      if (it + 1 < nt) issue_sp(it + 1);
      if (elect_one()) {
        if (ROLE == ROLE_DQ) {
          // dQ += dS K_it : A = dS (K-major over keys), B = K rows MN-major
          constexpr uint32_t id = umma_idesc_bf16(128, HD) | (1u << 16);
          for (int at = 0; at < 2; ++at) {
            const uint64_t da = umma_desc_sw128(sDS + at * TILE_BYTES);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(tmem + 256, da + uint64_t(k * 2),
                        desc_mn(sB0 + it * TILE_BYTES + uint32_t(at * 64 + k * 16) * 128, 0), id,
                        (it | at | k) != 0);
          }
        } else {
          // dV += Pd^T dO_it, dK += dS^T Q_it : A MN-major over keys (two
          // 64-key atoms 16 KB apart), B MN-major (query rows = K)
          constexpr uint32_t id = umma_idesc_bf16(128, HD) | (1u << 15) | (1u << 16);
#pragma unroll
          for (int k = 0; k < TILE / 16; ++k) {
            umma_bf16(tmem + 256, desc_mn(sPD + k * 2048, TILE_BYTES),
                      desc_mn(sB1 + it * TILE_BYTES + k * 2048, 0), id, (it | k) != 0);
            umma_bf16(tmem + 320, desc_mn(sDS + k * 2048, TILE_BYTES),
                      desc_mn(sB0 + it * TILE_BYTES + k * 2048, 0), id, (it | k) != 0);
          }
        }
        umma_commit(bar_acc);
      }
      __syncwarp();
    }
  } else {
    const int quarter = warp & 3, half = warp >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16);
    const uint64_t seed = a.rng[0], step = a.rng[1];
    const uint64_t bh = uint64_t(b * a.heads + h);
    for (int it = 0; it < nt; ++it) {
      const int qtile = ROLE == ROLE_DQ ? tile : it;
      const int ktile = ROLE == ROLE_DQ ? it : tile;
      const int q = qtile * TILE + r;
      const float lse2 = __ldg(a.lse + bh * S + q);
      const float Dv = __ldg(a.D + bh * S + q);
      const uint64_t erow = (bh * S + q) * uint64_t(S);
      mbar_wait(bar_sp, it & 1);
      tc_fence_after();
      uint32_t wds[2][16], wpd[2][16];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int lc = half * 64 + c * 32;  // column within the 128-key block
        float sv[32], dp[32];
        tmem_ld_32x32b_x32(trow + lc, sv);
        tmem_ld_32x32b_x32(trow + 128 + lc, dp);
        uint32_t keep = 0xFFFFFFFFu;
        if (a.thr) {
          const uint64_t g = (erow + uint64_t(ktile * TILE + lc)) >> 4;
          keep = keep16(drop_block(seed, step, a.tag, g), a.thr) |
                 (keep16(drop_block(seed, step, a.tag, g + 1), a.thr) << 16);
        }
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float p0 = ex2(fmaf(sv[i], kCl2, -lse2));
          const float p1 = ex2(fmaf(sv[i + 1], kCl2, -lse2));
          const float k0 = (keep >> i) & 1u ? a.dscale : 0.f;
          const float k1 = (keep >> (i + 1)) & 1u ? a.dscale : 0.f;
          wds[c][i >> 1] = pack_bf16x2(p0 * fmaf(dp[i], k0, -Dv), p1 * fmaf(dp[i + 1], k1, -Dv));
          if (ROLE == ROLE_DKV) wpd[c][i >> 1] = pack_bf16x2(p0 * k0, p1 * k1);
        }
      }
      // the previous block's accumulate MMAs have read sDS / sPD
      if (it > 0) mbar_wait(bar_acc, (it - 1) & 1);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        st_row32(sDS, r, half * 64 + c * 32, wds[c]);
        if (ROLE == ROLE_DKV) st_row32(sPD, r, half * 64 + c * 32, wpd[c]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_ds);
    }
    // ---- epilogue ----
    mbar_wait(bar_acc, (nt - 1) & 1);
    tc_fence_after();
    const int row = tile * TILE + r;  // DQ: query row; DKV: key row (acc lanes)
    bf16* base = a.out + (int64_t(row0) + row) * (3 * a.Hd) + h * HD + half * 32;
    auto store = [&](uint32_t col, bf16* dst, float s) {
      float v[32];
      tmem_ld_32x32b_x32(trow + col, v);
      uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        d[u] = make_uint4(pack_bf16x2(v[8 * u] * s, v[8 * u + 1] * s),
                          pack_bf16x2(v[8 * u + 2] * s, v[8 * u + 3] * s),
                          pack_bf16x2(v[8 * u + 4] * s, v[8 * u + 5] * s),
                          pack_bf16x2(v[8 * u + 6] * s, v[8 * u + 7] * s));
    };
    if (ROLE == ROLE_DQ) {
      store(256 + half * 32, base, kScale);
    } else {
      store(256 + half * 32, base + 2 * a.Hd, 1.f);   // dV
      store(320 + half * 32, base + a.Hd, kScale);    // dK
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == CTRL) tmem_dealloc(tmem, 512);
}

size_t fwd_smem(int S) {
  return 1024 + TILE_BYTES + size_t(S) * 128 + size_t(S) * 256 + 4 * TILE * 4 + 64;
}
size_t bwd_smem(int S, int role) {
  return 1024 + 2 * TILE_BYTES + 2 * size_t(S) * 128 + (role == ROLE_DKV ? 4 : 2) * TILE_BYTES + 64;
}

bool shape_ok(int S, int heads) { return S > 0 && S % TILE == 0 && S <= 512 && heads > 0; }

}  // namespace

cudaError_t attention_fwd(const void* qkv, void* out, float* lse, int B, int S, int heads,
                          float p, const uint64_t* rng, uint32_t tag, cudaStream_t st) {
  if (!shape_ok(S, heads)) return cudaErrorInvalidValue;
  const int Hd = heads * HD;
  alignas(64) CUtensorMap qm;
  if (!tma_2d_bf16(&qm, qkv, uint64_t(3 * Hd), uint64_t(B) * S, uint64_t(3 * Hd), 64, TILE,
                   CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const DropParams dp = drop_params(p);
  AttnArgs a{B, S, heads, Hd, static_cast<bf16*>(out), lse, nullptr, dp.thr, dp.scale, rng, tag};
  const size_t smem = fwd_smem(S);
  static bool attr = false;
  if (!attr) {
    if (cudaError_t e = cudaFuncSetAttribute(k_attn_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(fwd_smem(512))))
      return e;
    attr = true;
  }
  if (cudaError_t e = launch_k(k_attn_fwd, dim3(S / TILE, heads, B), dim3(kThreads), smem, st, qm, a))
    return e;
  return cudaGetLastError();
}

cudaError_t attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                          float* D, void* dqkv, int B, int S, int heads, float p,
                          const uint64_t* rng, uint32_t tag, cudaStream_t st) {
  if (!shape_ok(S, heads)) return cudaErrorInvalidValue;
  const int Hd = heads * HD;
  const int64_t T = int64_t(B) * S;
  if (cudaError_t e = attn_dvec(out, dout, T, S, heads, D, st)) return e;
  alignas(64) CUtensorMap qm, dm;
  if (!tma_2d_bf16(&qm, qkv, uint64_t(3 * Hd), uint64_t(T), uint64_t(3 * Hd), 64, TILE,
                   CU_TENSOR_MAP_SWIZZLE_128B) ||
      !tma_2d_bf16(&dm, dout, uint64_t(Hd), uint64_t(T), uint64_t(Hd), 64, TILE,
                   CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const DropParams dp = drop_params(p);
  AttnArgs a{B, S, heads, Hd, static_cast<bf16*>(dqkv), const_cast<float*>(lse), D, dp.thr,
             dp.scale, rng, tag};
  static bool attr = false;
  if (!attr) {
    if (cudaError_t e = cudaFuncSetAttribute(k_attn_bwd<ROLE_DQ>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(bwd_smem(512, ROLE_DQ))))
      return e;
    if (cudaError_t e = cudaFuncSetAttribute(k_attn_bwd<ROLE_DKV>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(bwd_smem(512, ROLE_DKV))))
      return e;
    attr = true;
  }
  const dim3 grid(S / TILE, heads, B);
  if (cudaError_t e = launch_k(k_attn_bwd<ROLE_DKV>, grid, dim3(kThreads), bwd_smem(S, ROLE_DKV),
                               st, qm, dm, a))
    return e;
  if (cudaError_t e = launch_k(k_attn_bwd<ROLE_DQ>, grid, dim3(kThreads), bwd_smem(S, ROLE_DQ), st,
                               qm, dm, a))
    return e;
  return cudaGetLastError();
}

}  // namespace delta_k
