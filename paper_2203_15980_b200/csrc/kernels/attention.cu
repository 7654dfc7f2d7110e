// Multi-head attention for sm_100a (tcgen05 + TMEM + TMA): the Attention node
// of the reference's transformer trace (ref src/trace.cpp:452) and its
// backward, with attention-probability dropout whose mask is replayed
// (philox.cuh), so a recomputed Attention output is bit-identical.
//
// BERT shapes: head dim 64, sequence S <= 512 (a multiple of 128); all keys
// of a (sequence, head) stay on chip; no atomics anywhere (deterministic
// gradients).
//
// forward (persistent, one CTA per SM walking (query-tile pair, head,
//   sequence) items, the next item's loads under the current one's tail; two
//   128-row query tiles per CTA, K and V of the sequence resident): per tile
//   and 128-key chunk j, S_j = Q K_j^T in TMEM (128 columns per tile); 8
//   softmax warps per tile, two per TMEM lane quarter, each owning one 64-key
//   half of every chunk with its own running max, row sum and accumulator
//   O_h += P_h V_h (single-pass online softmax; the max is raised, and O_h
//   rescaled in TMEM, only past 2^8 of headroom).  P = exp2(s*c - m*c) * keep
//   (bf16, unnormalised) goes to shared memory in the K-major SW128 layout, V
//   is an MN-major B operand; at the end the halves combine,
//   O = (O_0 2^(m_0-m) + O_1 2^(m_1-m)) * dropout_scale / rowsum, and lse (log2
//   units) is saved.  One MMA warp alternates between the tiles, so each
//   tile's MMAs run under the other's softmax.
// backward (grid heads x B, one CTA per (sequence, head)): for every key
//   block j (128 keys, K_j / V_j loaded by TMA) and query block i
//   (Q, dO of the whole sequence resident): S_ij = Q_i K_j^T and
//   dPd_ij = dO_i V_j^T in two 64-key halves (TMEM 384-511), the softmax
//   warps form P = exp2(s*c - lse), Pd = P*keep*scale and
//   dS = P (dPd*keep*scale - D) into shared memory, then
//     dV_j += Pd^T dO_i,  dK_j += dS^T Q_i   (TMEM 320 / 256, drained per j)
//     dQ_i += dS K_j                         (TMEM 64*i, drained at the end)
//   the transposed products read the [query][key] tiles through MN-major
//   descriptors.  Every softmax term is computed once.
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
constexpr int MATH_W = 16;        // softmax warps: 4 per TMEM lane quarter
constexpr int CTRL = MATH_W;      // TMA / MMA / TMEM warp
constexpr int kThreads = (MATH_W + 1) * 32;
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

__device__ __forceinline__ void bar_math() {
  asm volatile("bar.sync 1, %0;" ::"n"(MATH_W * 32) : "memory");
}

// tcgen05.ld of 16 consecutive fp32 columns of this warp's 32 lanes, without
// the wait (issue several, then tmem_wait once)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// tcgen05.st of 16 consecutive fp32 columns of this warp's 32 lanes
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// keep masks of one Philox block (16 elements): byte i of v[w] = 0xFF iff
// element 4w + i is kept (all kept when thr == 0)
__device__ __forceinline__ uint4 keep_bytes(uint64_t seed, uint64_t step, uint32_t tag, uint64_t g,
                                            uint32_t thr) {
  if (!thr) return make_uint4(~0u, ~0u, ~0u, ~0u);
  return keep_mask_bytes(drop_block(seed, step, tag, g), thr);
}
// 16-bit lane masks of elements (2j, 2j+1) of a 4-byte keep word
__device__ __forceinline__ uint32_t pair_mask(uint32_t kb, int j) {
  return __byte_perm(kb, 0, j ? 0x3322 : 0x1100);
}
// fp32 all-ones / zero mask of element i of a 4-byte keep word
__device__ __forceinline__ uint32_t elem_mask(uint32_t kb, int i) {
  return __byte_perm(kb, 0, 0x1111u * uint32_t(i));
}

// 16 bf16 (two 16-byte chunks) of row r at key column `col` (a multiple of
// 16) of a [128][ncols] K-major SW128 tile set (64-column atoms of 16 KB)
__device__ __forceinline__ void st_row16(uint32_t base, int r, int col, const uint32_t* w) {
  const uint32_t atom = base + uint32_t(col >> 6) * TILE_BYTES + uint32_t(r) * 128;
  const int u0 = (col & 63) >> 3;
#pragma unroll
  for (int u = 0; u < 2; ++u)
    st_shared_v4(atom + ((uint32_t((u0 + u) ^ (r & 7))) << 4),
                 make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]));
}

// 16 fp32 values * s -> 8 packed bf16x2 words
__device__ __forceinline__ void pack16(const uint32_t (&v)[16], float s, uint32_t* w) {
#pragma unroll
  for (int e = 0; e < 8; ++e)
    w[e] = pack_bf16x2(__uint_as_float(v[2 * e]) * s, __uint_as_float(v[2 * e + 1]) * s);
}
__device__ __forceinline__ void store16w(bf16* dst, const uint32_t* w) {
  uint4* d = reinterpret_cast<uint4*>(dst);
  d[0] = make_uint4(w[0], w[1], w[2], w[3]);
  d[1] = make_uint4(w[4], w[5], w[6], w[7]);
}
__device__ __forceinline__ void store16(bf16* dst, const uint32_t (&v)[16], float s) {
  uint32_t w[8];
  pack16(v, s, w);
  store16w(dst, w);
}
// 32 columns of a row scaled, stored as bf16, and (sum) the warp's column sums
// of the stored values: lane c returns column c's sum over the warp's 32 rows
__device__ __forceinline__ float store32_colsum(bf16* dst, const uint32_t (&a)[16],
                                                const uint32_t (&b)[16], float s, bool sum,
                                                int lane) {
  uint32_t w[16];
  pack16(a, s, w);
  pack16(b, s, w + 8);
  store16w(dst, w);
  store16w(dst + 16, w + 8);
  return sum ? warp_colsum32_bf16(w, lane) : 0.f;
}

// debug (builds with -DDELTA_ATTN_DEBUG): progress words in mapped host
// memory (null = off), set by attention_debug(); the host can read them while
// a kernel is stuck.  Compiled out otherwise (they cost issue slots).
__device__ uint32_t* g_attn_dbg = nullptr;
__device__ __forceinline__ void dbg_mark(int slot, uint32_t v) {
#ifdef DELTA_ATTN_DEBUG
  uint32_t* d = g_attn_dbg;
  if (d) {
    *reinterpret_cast<volatile uint32_t*>(d + (blockIdx.y * gridDim.x + blockIdx.x) * 32 + slot) = v;
  }
#endif
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
  float* colpart;  // bwd, optional: [B][3 Hd] per-sequence column sums of dqkv (bias gradient)
};

// ======================================================================= fwd
// Persistent (one CTA per SM walking (query-tile pair, head, sequence) items;
// the next item's Q/K load under the current item's last chunk, V under its
// epilogue); two 128-row query tiles per CTA, K and V of the (sequence, head)
// resident.  Per tile and 128-key chunk j: S_j = Q K_j^T in TMEM (128
// columns); 8 softmax warps per tile, two per TMEM lane quarter, each owning
// one 64-key half of every chunk.  Single pass, online softmax per half: a
// warp keeps its own running max m_h and row sum l_h and accumulates its own
// O_h += P_h V_h (two O accumulators per tile, 64 columns each) — no exchange
// between the halves until the end, where O = O_0 2^(m_0-m) + O_1 2^(m_1-m).
// A half's running max is only raised when a chunk exceeds it by more than
// 2^8 (P <= 256 otherwise, harmless in bf16 / fp32), so the O_h rescale
// (TMEM load, scale, store) is rare.  The one MMA warp alternates the tiles.
constexpr int F2_SW = 8;                       // softmax warps per query tile
constexpr int F2_CTRL = 2 * F2_SW;             // TMA + MMA warp
constexpr int kThreadsF2 = (F2_CTRL + 1) * 32;
constexpr float kRescale = 8.f;                // log2 headroom before a rescale

__device__ __forceinline__ void bar_tile(int t) {
  asm volatile("bar.sync %0, %1;" ::"r"(2 + t), "n"(F2_SW * 32) : "memory");
}

__global__ void __launch_bounds__(kThreadsF2, 1)
    k_attn_fwd2(const __grid_constant__ CUtensorMap qkv_map, const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = a.S, nt = S / TILE;
  const uint32_t sQ = smem_u32(smem);               // [2 tiles][128][64]
  const uint32_t sK = sQ + 2 * TILE_BYTES;          // [nt][128 keys][64]
  const uint32_t sV = sK + uint32_t(nt) * TILE_BYTES;
  const uint32_t sP = sV + uint32_t(nt) * TILE_BYTES;  // [2 tiles][2 halves][128][64 keys]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (sP - sQ) + 4 * TILE_BYTES);
  uint64_t* bar_qk = bars;       // Q tiles and K landed
  uint64_t* bar_v = bars + 1;    // V landed
  uint64_t* bar_s = bars + 2;    // [2] S of a tile computed
  uint64_t* bar_t = bars + 4;    // [2] S of a tile read out of TMEM
  uint64_t* bar_p = bars + 6;    // [2] P of a tile written (and O_h rescaled)
  uint64_t* bar_o = bars + 8;    // [2] a tile's PV MMAs done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 10);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // TMEM: S of tile t at columns 128 t; O_h of tile t at 256 + 128 t + 64 h
  const int nqp = (nt + 1) / 2;
  const int items = nqp * a.heads * a.B;
  auto item = [&](int w, int& qp, int& h, int& b) {
    qp = w % nqp;
    h = (w / nqp) % a.heads;
    b = w / (nqp * a.heads);
  };

  if (threadIdx.x == 0) {
    mbar_init(bar_qk, 1);
    mbar_init(bar_v, 1);
    for (int t = 0; t < 2; ++t) {
      mbar_init(bar_s + t, 1);
      mbar_init(bar_t + t, F2_SW);
      mbar_init(bar_p + t, F2_SW);
      mbar_init(bar_o + t, 1);
    }
    fence_mbar_init();
    tma_prefetch_desc(&qkv_map);
  }
  if (warp == F2_CTRL) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  pdl_trigger();

  if (warp == F2_CTRL) {
    constexpr uint32_t idS = umma_idesc_bf16(128, 128);
    constexpr uint32_t idO = umma_idesc_bf16(128, HD) | (1u << 16);  // B (V) MN-major
    auto load_qk = [&](int w) {
      int qp, h, b;
      item(w, qp, h, b);
      const int ntl = min(2, nt - 2 * qp);
      mbar_arrive_expect_tx(bar_qk, uint32_t(ntl + nt) * TILE_BYTES);
      for (int t = 0; t < ntl; ++t)
        tma_load_2d(sQ + t * TILE_BYTES, &qkv_map, bar_qk, h * HD, b * S + (2 * qp + t) * TILE);
      for (int j = 0; j < nt; ++j)
        tma_load_2d(sK + j * TILE_BYTES, &qkv_map, bar_qk, a.Hd + h * HD, b * S + j * TILE);
    };
    auto load_v = [&](int w) {
      int qp, h, b;
      item(w, qp, h, b);
      mbar_arrive_expect_tx(bar_v, uint32_t(nt) * TILE_BYTES);
      for (int j = 0; j < nt; ++j)
        tma_load_2d(sV + j * TILE_BYTES, &qkv_map, bar_v, 2 * a.Hd + h * HD, b * S + j * TILE);
    };
    auto issue_s = [&](int t, int k) {
      if (elect_one()) {
        const uint64_t dq = umma_desc_sw128(sQ + t * TILE_BYTES);
        const uint64_t dk = umma_desc_sw128(sK + k * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          umma_bf16(tmem + t * TILE, dq + uint64_t(kk * 2), dk + uint64_t(kk * 2), idS, kk > 0);
        umma_commit(bar_s + t);
      }
      __syncwarp();
    };
    uint32_t n_qk = 0, n_v = 0, n_t0 = 0, n_t1 = 0, n_p0 = 0, n_p1 = 0, n_o0 = 0, n_o1 = 0;
    if (lane == 0 && blockIdx.x < items) {
      load_qk(blockIdx.x);
      load_v(blockIdx.x);
    }
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
      int qp, h, b;
      item(w, qp, h, b);
      const int ntile = min(2, nt - 2 * qp);
      const int wn = w + gridDim.x;  // the next item of this CTA
      mbar_wait(bar_qk, n_qk++ & 1);
      tc_fence_after();
      for (int t = 0; t < ntile; ++t) issue_s(t, 0);
      for (int k = 0; k < nt; ++k) {
        for (int t = 0; t < ntile; ++t) {
          mbar_wait(bar_t + t, (t ? n_t1++ : n_t0++) & 1);
          tc_fence_after();
          if (k + 1 < nt) issue_s(t, k + 1);
        }
        // every S MMA of this item is done: Q and K may be refilled
        if (k + 1 == nt && lane == 0 && wn < items) load_qk(wn);
        if (k == 0) mbar_wait(bar_v, n_v++ & 1);
        for (int t = 0; t < ntile; ++t) {
          mbar_wait(bar_p + t, (t ? n_p1++ : n_p0++) & 1);
          tc_fence_after();
          if (elect_one()) {
            // O_h += P_h V_h: half h = keys [64 h, 64 h + 64) of chunk k
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const uint64_t dp = umma_desc_sw128(sP + (t * 2 + hf) * TILE_BYTES);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                umma_bf16(tmem + 256 + t * 128 + hf * HD, dp + uint64_t(kk * 2),
                          desc_mn(sV + k * TILE_BYTES + uint32_t(hf * 64 + kk * 16) * 128, 0),
                          idO, (k | kk) != 0);
            }
            umma_commit(bar_o + t);
          }
          __syncwarp();
        }
      }
      // V is free once this item's last PV MMAs are done
      if (wn < items) {
        for (int t = 0; t < ntile; ++t) mbar_wait(bar_o + t, ((t ? n_o1 : n_o0) + nt - 1) & 1);
        if (lane == 0) load_v(wn);
        __syncwarp();
      }
      n_o0 += nt;
      if (ntile > 1) n_o1 += nt;
    }
  } else {
    const int t = warp / F2_SW, w8 = warp % F2_SW;
    const int quarter = w8 & 3, half = w8 >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16);
    const uint32_t tS = trow + t * TILE + half * 64;
    const uint32_t tOh = trow + 256 + t * 128 + half * HD;  // this warp's O_h rows
    const uint64_t seed = a.rng[0], step = a.rng[1];
    float* red = reinterpret_cast<float*>(smem + (sP - sQ) + t * 2 * TILE_BYTES);  // P's buffer
    const uint32_t pT = sP + (t * 2 + half) * TILE_BYTES;  // this half's P atom
    uint32_t n_s = 0, n_o = 0;  // completions of bar_s[t], bar_o[t] seen so far
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
      int qp, h, b;
      item(w, qp, h, b);
      if (t >= min(2, nt - 2 * qp)) continue;  // this item has one query tile
      const int q = (2 * qp + t) * TILE + r;
      const uint64_t bh = uint64_t(b * a.heads + h);
      // Philox block of keys [j*128 + half*64 + c*16, +16) of row q
      const uint64_t g0 = ((bh * S + q) * uint64_t(S) + half * 64) >> 4;
      float mc = 0.f, l = 0.f;  // running max (scaled, log2 units) and row sum of this half
#pragma unroll 1
      for (int j = 0; j < nt; ++j) {
        mbar_wait(bar_s + t, n_s++ & 1);
        tc_fence_after();
        uint32_t v[4][16];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld16(tS + c * 16, v[c]);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_t + t);
        float m = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 16; ++i) m = fmaxf(m, __uint_as_float(v[c][i]));
        const float mj = m * kCl2;
        // raise the running max only past the headroom (rare after chunk 0)
        float f = 1.f;
        if (j == 0) {
          mc = mj;
        } else if (mj > mc + kRescale) {
          f = ex2(mc - mj);
          l *= f;
          mc = mj;
        }
        // P = exp2(s*c - mc) * keep: the first two 16-key blocks before waiting
        // for the previous chunk's PV MMAs (which run meanwhile), the rest after
        auto form = [&](int c, uint32_t* wv) {
          const uint4 kb = keep_bytes(seed, step, a.tag, g0 + j * 8 + c, a.thr);
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float p0 = ex2(fmaf(__uint_as_float(v[c][i]), kCl2, -mc));
            const float p1 = ex2(fmaf(__uint_as_float(v[c][i + 1]), kCl2, -mc));
            l += p0 + p1;
            wv[i >> 1] = pack_bf16x2(p0, p1) & pair_mask((&kb.x)[i >> 2], (i >> 1) & 1);
          }
        };
        uint32_t w0[8], w1[8];
        form(0, w0);
        form(1, w1);
        // the previous chunk's PV MMAs have read P and updated O_h
        if (j > 0) {
          mbar_wait(bar_o + t, n_o++ & 1);
          if (__any_sync(0xFFFFFFFFu, f != 1.f)) {
            // rare: this half's O (accumulated at the old max) scaled down
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
              uint32_t o[16];
              tmem_ld16(tOh + c * 16, o);
              tmem_wait();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * f);
              tmem_st16(tOh + c * 16, o);
            }
            tmem_wait_st();
          }
        }
        st_row16(pT, r, 0, w0);
        st_row16(pT, r, 16, w1);
        form(2, w0);
        st_row16(pT, r, 32, w0);
        form(3, w1);
        st_row16(pT, r, 48, w1);
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_p + t);
      }
      // the last PV MMAs: P's buffer is then free for the halves' exchange
      mbar_wait(bar_o + t, n_o++ & 1);
      tc_fence_after();
      red[half * TILE + r] = mc;
      red[2 * TILE + half * TILE + r] = l;
      bar_tile(t);
      const float m0 = red[r], m1 = red[TILE + r];
      const float l0 = red[2 * TILE + r], l1 = red[3 * TILE + r];
      bar_tile(t);
      const float mrow = fmaxf(m0, m1);
      const float f0 = ex2(m0 - mrow), f1 = ex2(m1 - mrow);
      const float lrow = fmaf(l0, f0, l1 * f1);
      if (half == 0) a.lse[bh * S + q] = mrow + __log2f(lrow);
      const float inv = a.dscale / lrow;
      // ---- epilogue: O columns [half*32, half*32 + 32) of row r from both halves' O
      uint32_t x0[16], x1[16], y0[16], y1[16];
      tmem_ld16(trow + 256 + t * 128 + half * 32, x0);
      tmem_ld16(trow + 256 + t * 128 + half * 32 + 16, x1);
      tmem_ld16(trow + 256 + t * 128 + HD + half * 32, y0);
      tmem_ld16(trow + 256 + t * 128 + HD + half * 32 + 16, y1);
      tmem_wait();
      tc_fence_before();
      const float g0f = f0 * inv, g1f = f1 * inv;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        x0[i] = __float_as_uint(fmaf(__uint_as_float(x0[i]), g0f, __uint_as_float(y0[i]) * g1f));
        x1[i] = __float_as_uint(fmaf(__uint_as_float(x1[i]), g0f, __uint_as_float(y1[i]) * g1f));
      }
      bf16* dst = a.out + (int64_t(b) * S + q) * a.Hd + h * HD + half * 32;
      store16(dst, x0, 1.f);
      store16(dst + 16, x1, 1.f);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == F2_CTRL) tmem_dealloc(tmem, 512);
}

// ======================================================================= bwd
// TMEM columns
constexpr uint32_t T_DK = 256, T_DV = 320, T_S = 384, T_DP = 448;

__global__ void __launch_bounds__(kThreads, 1)
    k_attn_bwd(const __grid_constant__ CUtensorMap qkv_map, const __grid_constant__ CUtensorMap do_map,
               const AttnArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int S = a.S;
  const int nt = S / TILE;
  const uint32_t sQ = smem_u32(smem);                  // [S][64] Q of the sequence
  const uint32_t sDO = sQ + uint32_t(S) * 128;         // [S][64] dO
  const uint32_t sKV = sDO + uint32_t(S) * 128;        // K_j, V_j
  const uint32_t sP = sKV + 2 * TILE_BYTES;            // Pd [128 q][128 keys]
  const uint32_t sDS = sP + 2 * TILE_BYTES;            // dS [128 q][128 keys]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * size_t(S) * 128 + 6 * TILE_BYTES);
  uint64_t* bar_qd = bars;       // Q, dO landed
  uint64_t* bar_kv = bars + 1;   // K_j / V_j landed
  uint64_t* bar_sp = bars + 3;   // S/dP half computed
  uint64_t* bar_h = bars + 4;    // half 0 of a block written to smem (bar_h1: half 1) — one
                                 // barrier per half, so the MMA warp, which waits for both
                                 // after issuing the next half early, is never two phases
                                 // behind (a parity wait cannot tell phase k from k+2)
  uint64_t* bar_acc = bars + 5;  // accumulate MMAs of a block done
  uint64_t* bar_dr = bars + 6;   // dK/dV of a key block drained
  uint64_t* bar_t = bars + 7;    // S/dP half read out of TMEM (the next half may overwrite)
  uint64_t* bar_h1 = bars + 8;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 9);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = blockIdx.x, b = blockIdx.y;
  const int row0 = b * S;

  if (threadIdx.x == 0) {
    mbar_init(bar_qd, 1);
    mbar_init(bar_kv, 1);
    mbar_init(bar_sp, 1);
    mbar_init(bar_h, MATH_W);
    mbar_init(bar_acc, 1);
    mbar_init(bar_dr, MATH_W);
    mbar_init(bar_t, MATH_W);
    mbar_init(bar_h1, MATH_W);
    fence_mbar_init();
    tma_prefetch_desc(&qkv_map);
    tma_prefetch_desc(&do_map);
  }
  if (threadIdx.x == 0) dbg_mark(20, 0xB1);
  if (warp == CTRL) tmem_alloc(tslot, 512);
  if (threadIdx.x == CTRL * 32) dbg_mark(21, 0xB2);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  pdl_trigger();
  const int nblk = nt * nt;  // (j, i) blocks, j outer
  if (warp == CTRL) {
    auto load_kv = [&](int j) {
      mbar_arrive_expect_tx(bar_kv, 2 * TILE_BYTES);
      tma_load_2d(sKV, &qkv_map, bar_kv, a.Hd + h * HD, row0 + j * TILE);
      tma_load_2d(sKV + TILE_BYTES, &qkv_map, bar_kv, 2 * a.Hd + h * HD, row0 + j * TILE);
    };
    if (lane == 0) {
      mbar_arrive_expect_tx(bar_qd, 2 * uint32_t(S) * 128);
      for (int i = 0; i < nt; ++i) {
        tma_load_2d(sQ + i * TILE_BYTES, &qkv_map, bar_qd, h * HD, row0 + i * TILE);
        tma_load_2d(sDO + i * TILE_BYTES, &do_map, bar_qd, h * HD, row0 + i * TILE);
      }
      load_kv(0);
    }
    mbar_wait(bar_qd, 0);
    constexpr uint32_t idH = umma_idesc_bf16(128, 64);                          // S / dP halves
    constexpr uint32_t idQ = umma_idesc_bf16(128, HD) | (1u << 16);             // dQ: B MN-major
    constexpr uint32_t idKV = umma_idesc_bf16(128, HD) | (1u << 15) | (1u << 16);  // dK, dV
    uint32_t nsp = 0;  // S/dP halves issued
    // S_ij, dPd_ij for keys [hh*64, hh*64+64) of block j
    auto issue_half = [&](int blk, int hh) {
      const int i = blk % nt;
      const uint32_t kb = sKV;
      if (elect_one()) {
        const uint64_t dq = umma_desc_sw128(sQ + i * TILE_BYTES);
        const uint64_t dd = umma_desc_sw128(sDO + i * TILE_BYTES);
        const uint64_t dk = umma_desc_sw128(kb + hh * 64 * 128);
        const uint64_t dv = umma_desc_sw128(kb + TILE_BYTES + hh * 64 * 128);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + T_S, dq + uint64_t(k * 2), dk + uint64_t(k * 2), idH, k > 0);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + T_DP, dd + uint64_t(k * 2), dv + uint64_t(k * 2), idH, k > 0);
        umma_commit(bar_sp);
      }
      __syncwarp();
      ++nsp;
    };
    mbar_wait(bar_kv, 0);
    tc_fence_after();
    issue_half(0, 0);
    uint32_t nt_ = 0;  // bar_t completions consumed
    for (int blk = 0; blk < nblk; ++blk) {
      const int j = blk / nt, i = blk % nt;
      const uint32_t kb = sKV;
      // S/dP of a half are issued as soon as the previous half has been read
      // out of TMEM, so they run while the softmax warps still compute
      if (lane == 0) dbg_mark(16, 0x10000 | blk);
      mbar_wait(bar_t, nt_++ & 1);
      tc_fence_after();
      issue_half(blk, 1);
      if (lane == 0) dbg_mark(16, 0x20000 | blk);
      mbar_wait(bar_t, nt_++ & 1);
      tc_fence_after();
      if (lane == 0) dbg_mark(16, 0x30000 | blk);
      const bool next_same_j = blk + 1 < nblk && (blk + 1) / nt == j;
      if (next_same_j) issue_half(blk + 1, 0);
      // both halves' P and dS in shared memory
      mbar_wait(bar_h, blk & 1);
      if (lane == 0) dbg_mark(16, 0x40000 | blk);
      mbar_wait(bar_h1, blk & 1);
      tc_fence_after();
      if (lane == 0) dbg_mark(16, 0x50000 | blk);
      // the previous key block's dK / dV drained before this block zeroes them
      if (i == 0 && j > 0) {
        mbar_wait(bar_dr, (j - 1) & 1);
        tc_fence_after();
      }
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < TILE / 16; ++k) {
          // dV_j += Pd^T dO_i ; dK_j += dS^T Q_i   (A MN-major over the 128 keys)
          umma_bf16(tmem + T_DV, desc_mn(sP + k * 2048, TILE_BYTES),
                    desc_mn(sDO + i * TILE_BYTES + k * 2048, 0), idKV, (i | k) != 0);
          umma_bf16(tmem + T_DK, desc_mn(sDS + k * 2048, TILE_BYTES),
                    desc_mn(sQ + i * TILE_BYTES + k * 2048, 0), idKV, (i | k) != 0);
        }
        // dQ_i += dS K_j  (A K-major over keys, B = K_j rows MN-major)
        for (int at = 0; at < 2; ++at) {
          const uint64_t da = umma_desc_sw128(sDS + at * TILE_BYTES);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            umma_bf16(tmem + 64 * i, da + uint64_t(k * 2),
                      desc_mn(kb + uint32_t(at * 64 + k * 16) * 128, 0), idQ, (j | at | k) != 0);
        }
        umma_commit(bar_acc);
      }
      __syncwarp();
      if (blk + 1 < nblk && !next_same_j) {
        // next key block: once every MMA reading K_j / V_j is done, load
        // K_j+1 / V_j+1 into the buffer (the dK/dV drain overlaps the load)
        const int jn = (blk + 1) / nt;
        mbar_wait(bar_acc, blk & 1);
        if (lane == 0) load_kv(jn);
        __syncwarp();
        mbar_wait(bar_kv, jn & 1);
        tc_fence_after();
        issue_half(blk + 1, 0);
      }
    }
  } else {
    const int quarter = warp & 3, part = warp >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t trow = tmem + (uint32_t(quarter * 32) << 16);
    const uint64_t seed = a.rng[0], step = a.rng[1];
    const uint64_t bh = uint64_t(b * a.heads + h);
    float lse2[4], Dv[4];  // registers: constant indices only
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      lse2[i] = i < nt ? __ldg(a.lse + bh * S + i * TILE + r) : 0.f;
      Dv[i] = i < nt ? __ldg(a.D + bh * S + i * TILE + r) : 0.f;
    }
    uint32_t nsp = 0;
    float csum_kv = 0.f;
    for (int blk = 0; blk < nblk; ++blk) {
      const int j = blk / nt, i = blk % nt;
      const int q = i * TILE + r;
      float ls = 0.f, dv = 0.f;
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
        if (ii == i) ls = lse2[ii], dv = Dv[ii];
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        const int col = hh * 64 + part * 16;  // key column within the block
        // the half's keep bytes while its S/dP MMAs are in flight
        const uint4 kb = keep_bytes(seed, step, a.tag,
                                    ((bh * S + q) * uint64_t(S) + j * TILE + col) >> 4, a.thr);
        if (lane == 0) dbg_mark(warp, 0x10000 | (blk << 1) | hh);
        mbar_wait(bar_sp, nsp & 1);
        ++nsp;
        tc_fence_after();
        if (lane == 0) dbg_mark(warp, 0x20000 | (blk << 1) | hh);
        uint32_t sv[16], dp[16];
        tmem_ld16(trow + T_S + part * 16, sv);
        tmem_ld16(trow + T_DP + part * 16, dp);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_t);  // this half's TMEM may be overwritten
        uint32_t wds[8], wpd[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const float p0 = ex2(fmaf(__uint_as_float(sv[e]), kCl2, -ls));
          const float p1 = ex2(fmaf(__uint_as_float(sv[e + 1]), kCl2, -ls));
          const uint32_t w = (&kb.x)[e >> 2];
          const float k0 = __uint_as_float(__float_as_uint(a.dscale) & elem_mask(w, e & 3));
          const float k1 = __uint_as_float(__float_as_uint(a.dscale) & elem_mask(w, (e & 3) + 1));
          wds[e >> 1] = pack_bf16x2(p0 * fmaf(__uint_as_float(dp[e]), k0, -dv),
                                    p1 * fmaf(__uint_as_float(dp[e + 1]), k1, -dv));
          wpd[e >> 1] = pack_bf16x2(p0 * k0, p1 * k1);
        }
        // the previous block's accumulate MMAs have read sP / sDS
        if (lane == 0) dbg_mark(warp, 0x30000 | (blk << 1) | hh);
        if (hh == 0 && blk > 0) mbar_wait(bar_acc, (blk - 1) & 1);
        if (lane == 0) dbg_mark(warp, 0x40000 | (blk << 1) | hh);
        st_row16(sDS, r, col, wds);
        st_row16(sP, r, col, wpd);
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(hh ? bar_h1 : bar_h);
      }
      if (i == nt - 1) {
        // key block j complete: drain dK_j, dV_j (TMEM lane = key row)
        mbar_wait(bar_acc, blk & 1);
        tc_fence_after();
        uint32_t v0[16], v1[16];
        const int which = part >> 1;            // 0: dK, 1: dV
        const uint32_t col = (which ? T_DV : T_DK) + (part & 1) * 32;
        tmem_ld16(trow + col, v0);
        tmem_ld16(trow + col + 16, v1);
        tmem_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_dr);
        bf16* dst = a.out + (int64_t(row0) + j * TILE + r) * (3 * a.Hd) + (which ? 2 : 1) * a.Hd +
                    h * HD + (part & 1) * 32;
        // bias gradient: this warp's 32 key rows summed per column (of the
        // stored values), lane c keeps column c across the key blocks
        csum_kv += store32_colsum(dst, v0, v1, which ? 1.f : kScale, a.colpart != nullptr, lane);
      }
    }
    // ---- dQ of every query block (TMEM 64 i, lane = query row) ----
    mbar_wait(bar_acc, (nblk - 1) & 1);
    tc_fence_after();
    float csum_q0 = 0.f, csum_q1 = 0.f;
    for (int i = part; i < nt; i += 4) {
      uint32_t v0[16], v1[16], v2[16], v3[16];
      tmem_ld16(trow + 64 * i, v0);
      tmem_ld16(trow + 64 * i + 16, v1);
      tmem_ld16(trow + 64 * i + 32, v2);
      tmem_ld16(trow + 64 * i + 48, v3);
      tmem_wait();
      bf16* dst = a.out + (int64_t(row0) + i * TILE + r) * (3 * a.Hd) + h * HD;
      csum_q0 = store32_colsum(dst, v0, v1, kScale, a.colpart != nullptr, lane);
      csum_q1 = store32_colsum(dst + 32, v2, v3, kScale, a.colpart != nullptr, lane);
    }
    if (a.colpart) {
      // every MMA is done: P's buffer is scratch.  Combine the warps' column
      // sums in a fixed order into this (sequence, head)'s 192 bias columns.
      float* cs = reinterpret_cast<float*>(smem + (sP - sQ));
      cs[(quarter * 4 + part) * 32 + lane] = csum_kv;             // [quarter][part][32]
      cs[512 + (part * 4 + quarter) * 64 + lane] = csum_q0;       // [tile][quarter][64]
      cs[512 + (part * 4 + quarter) * 64 + 32 + lane] = csum_q1;
      bar_math();
      const int t = threadIdx.x;
      if (t < 3 * HD) {
        float s = 0.f;
        int third, c = t % HD;
        if (t < HD) {
          third = 0;
          for (int i = 0; i < nt; ++i)
            for (int qq = 0; qq < 4; ++qq) s += cs[512 + (i * 4 + qq) * 64 + c];
        } else {
          third = t / HD;  // 1: dK (parts 0, 1), 2: dV (parts 2, 3)
          const int pp = (third - 1) * 2 + c / 32;
          for (int qq = 0; qq < 4; ++qq) s += cs[(qq * 4 + pp) * 32 + (c & 31)];
        }
        a.colpart[int64_t(b) * 3 * a.Hd + third * a.Hd + h * HD + c] = s;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == CTRL) tmem_dealloc(tmem, 512);
}

size_t bwd_smem(int S) { return 1024 + 2 * size_t(S) * 128 + 6 * TILE_BYTES + 128; }  // 10 words

bool shape_ok(int S, int heads) { return S > 0 && S % TILE == 0 && S <= 512 && heads > 0; }

}  // namespace

static int attn_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Q (2 tiles) + P (2 tiles x 2 atoms) + K + V + barriers
static size_t fwd2_smem(int S) {
  return 1024 + 6 * size_t(TILE_BYTES) + 2 * size_t(S) * 128 + 128;
}

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
  static bool attr = false;
  if (!attr) {
    if (cudaError_t e = cudaFuncSetAttribute(k_attn_fwd2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(fwd2_smem(512))))
      return e;
    attr = true;
  }
  const int items = (S / TILE + 1) / 2 * heads * B;
  if (cudaError_t e = launch_k(k_attn_fwd2, dim3(items < attn_sms() ? items : attn_sms()), dim3(kThreadsF2),
                               fwd2_smem(S), st, qm, a))
    return e;
  return cudaGetLastError();
}

cudaError_t attention_debug(void* host_words) {
  uint32_t* p = static_cast<uint32_t*>(host_words);
  return cudaMemcpyToSymbol(g_attn_dbg, &p, sizeof(p));
}

cudaError_t attention_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                          float* D, void* dqkv, int B, int S, int heads, float p,
                          const uint64_t* rng, uint32_t tag, float* dbias, float* ws,
                          cudaStream_t st) {
  if (!shape_ok(S, heads) || (dbias && !ws)) return cudaErrorInvalidValue;
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
             dp.scale, rng, tag, dbias ? ws : nullptr};
  static bool attr = false;
  if (!attr) {
    if (cudaError_t e = cudaFuncSetAttribute(k_attn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(bwd_smem(512))))
      return e;
    attr = true;
  }
  if (cudaError_t e = launch_k(k_attn_bwd, dim3(heads, B), dim3(kThreads), bwd_smem(S), st, qm, dm, a))
    return e;
  if (dbias)
    if (cudaError_t e = merge_parts(ws, B, 3 * Hd, dbias, st)) return e;
  return cudaGetLastError();
}

}  // namespace delta_k
