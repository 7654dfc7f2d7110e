// Convolution weight gradient for sm_100a (tcgen05 + TMEM + TMA), replacing
// the library wgrad on the backward path.
//
// GEMM view (NHWC activations, KRSC weights), reduction over output pixels:
//   dW[k, (r,s,c)] = sum_m dY[m, k] * X[n, p*st-pad+r, q*st-pad+s, c],  m = (n,p,q)
// Both operands are MN-major in shared memory: a TMA box of 64 pixels x 64
// channels lands as 64 rows of 128 B (channels contiguous) — dY rows give the
// A tile (M' = 128 output channels = two boxes), X rows (plain 2D for a 1x1
// stride-1 conv, TMA im2col per tap otherwise, pixel-pair im2col for the C=4
// stem) give the B tile (N' = BN input channels of one tap).  The MMA reads
// them through MN-major descriptors (tcgen05 instruction-descriptor transpose
// bits), so no data is transposed anywhere.
//
// The reduction (N*P*Q pixels: up to 800k) is split over CTAs: work item =
// (split, output tile) with a contiguous pixel range; each writes its fp32
// partial tile to a workspace and a second kernel sums the splits in a fixed
// order straight into the fp32 KRSC gradient (deterministic, no atomics).
//
// Persistent, warp-specialised: warp 0 = TMA producer, warp 1 = TMEM owner +
// single-thread MMA issuer, warps 2-5 = epilogue (TMEM lane quarter = warp%4),
// two TMEM accumulators so the epilogue of one item overlaps the next.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "kernels/kernels.hpp"
#include "kernels/launch.hpp"
#include "kernels/sm100_common.cuh"
#include "kernels/tma_host.hpp"

namespace delta_k {

using namespace dsm100;

namespace {

constexpr int WG_THREADS = 192;
constexpr int KPIX = 64;  // pixels per k-block
constexpr int WG_PLAIN = 0, WG_IM2COL = 1, WG_STEM = 2, WG_STEMRAW = 3;
// head of the workspace: per-tile split counters (up to 4096 tiles)
constexpr size_t WG_COUNTER_BYTES = 16384;
constexpr int WG_FUSE_MAX_SPLITS = 1;  // measured: last-CTA sums of 2-4 splits -1 % ResNet, BERT neutral
// WG_STEMRAW: a k-block is one output row (n, p) of the stem; its 7 input
// rows are staged raw (pixel pairs, zero pads around them, conv_fwd.cu
// MODE_STEMRAW) and the B operand is addressed straight into them
constexpr uint32_t RAW_ROW = 2304, RAW_DATA = 128;

struct WgArgs {
  int K, C, taps, S, P, Q, stride, pad;
  int M;             // pixels N*P*Q
  int kblocks;       // ceil(M / KPIX) (WG_STEMRAW: N*P output rows)
  int W2;            // WG_STEMRAW: pixel pairs per input row
  int tiles_m;       // ceil(K / (128 * MT))
  int ntot;          // N' = taps * C (flattened (tap, channel) columns)
  int tiles;         // tiles_m * ceil(ntot / BN) (stem: tiles_m)
  int splits, kb_per_split;
  int items;         // splits * tiles
  float* ws;         // [items][128 * MT][BN] fp32 partials (splits > 1, and the stem)
  float* dw;         // fp32 [K][ntot] gradient (non-stem modes: written by this kernel)
  unsigned* counters;  // [tiles] splits landed per tile (zero at allocation, self-resetting)
  int fused;         // finish the gradient in this kernel (else: partials + the reduce launch)
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// MN-major operand descriptor, 128-byte swizzle: rows of 128 B along MN (64
// bf16), 8-row (K) groups 1 KB apart (SBO), MN atoms `lbo` bytes apart.
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= uint64_t((addr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}
// MN-major, no swizzle: core matrix = 8 K-rows x 16 B (8 MN elements); K
// groups `lbo` bytes apart, MN groups `sbo` bytes apart.
__device__ __forceinline__ uint64_t desc_mn_interleave(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((addr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  return d;
}

// MT = 2: a tile is 256 output channels x BN columns — two accumulators (the
// whole TMEM, so no double buffering) fed by the same B tile, halving the B
// traffic per flop (the operand stream from L2 paces the large-K shapes)
template <int MODE, int BN, int MT, bool PAIR = false>
constexpr int wg_stages() {
  return PAIR ? 6 : (MODE == WG_STEMRAW ? 6 : (MT == 2 ? 3 : (BN >= 192 ? 4 : 6)));
}

// PAIR: a 2-CTA cluster computes 256-channel tiles (cta_group::2 M=256): each
// CTA stages its own 128 output channels of dY and HALF of the BN input
// channels of X; both CTAs' bytes land on the leader's barrier, the leader
// issues the pair MMAs, commits are multicast, each CTA drains its own TMEM.
template <int BN, int MODE, int MT, bool PAIR = false>
__global__ void __launch_bounds__(WG_THREADS, 1)
    k_wgrad(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
            const WgArgs a) {
  static_assert(!PAIR || (MT == 1 && BN == 256 && (MODE == WG_PLAIN || MODE == WG_IM2COL)),
                "pair weight gradient: 256-column plain / im2col tiles");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr int STAGES = wg_stages<MODE, BN, MT, PAIR>();
  constexpr uint32_t A_STAGE = MT * 2 * KPIX * 128;                      // 2 boxes of 64 ch per 128
  constexpr uint32_t B_STAGE = MODE == WG_STEMRAW ? 7 * RAW_ROW
                               : MODE == WG_STEM  ? 32 * KPIX * 16
                                                  : ((PAIR ? BN / 2 : BN) / 64) * KPIX * 128;
  const uint32_t sA = smem_u32(smem);
  const uint32_t sB = sA + STAGES * A_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (A_STAGE + B_STAGE));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int unit = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int units = PAIR ? int(gridDim.x >> 1) : int(gridDim.x);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], PAIR ? 8 : 4);  // pair: both CTAs' epilogue warps
    }
    fence_mbar_init();
    tma_prefetch_desc(&amap);
    tma_prefetch_desc(&bmap);
  }
  if constexpr (MODE == WG_STEMRAW) {
    // zero pads (2 pairs) either side of every staged input row, once
    const uint32_t data_end = RAW_DATA + uint32_t(a.W2) * 16;
    for (int i = threadIdx.x; i < STAGES * 7 * 4; i += blockDim.x) {
      const int row = i >> 2, part = i & 3;
      const uint32_t off = (part < 2 ? RAW_DATA - 32 : data_end) + (part & 1) * 16;
      st_shared_v4(sB + (row / 7) * B_STAGE + (row % 7) * RAW_ROW + off, make_uint4(0, 0, 0, 0));
    }
    fence_proxy_async_smem();
  }
  // MT=1: two accumulators; MT=2: lo/hi halves (allocation: a power of two)
  constexpr uint32_t TMEM_COLS = 2 * BN <= 256 ? 2 * BN : 512;
  constexpr uint32_t NACC = MT == 2 ? 1 : 2;  // accumulator buffers
  if (warp == 1) {
    if constexpr (PAIR)
      tmem_alloc_pair(tslot, TMEM_COLS);
    else
      tmem_alloc(tslot, TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // prologue done (barriers, TMEM, descriptors): now wait for the predecessor
  pdl_wait();
  pdl_trigger();

  // work item -> (split, tile); tile -> (m block, first flattened column n0);
  // a tile's BN columns may span several taps when C < BN
  auto decode = [&](int item, int& m0, int& n0, int& kb0, int& kb1) {
    const int split = item / a.tiles, tile = item % a.tiles;
    m0 = (tile % a.tiles_m) * 128 * (PAIR ? 2 : MT) + int(rank) * 128;
    n0 = (tile / a.tiles_m) * BN;
    kb0 = split * a.kb_per_split;
    kb1 = min(a.kblocks, kb0 + a.kb_per_split);
  };

  if (warp == 0) {
    // ================================ producer ================================
    if (lane == 0) {
      uint32_t it = 0;
      for (int item = unit; item < a.items; item += units) {
        int m0, n0, kb0, kb1;
        decode(item, m0, n0, kb0, kb1);
        if (PAIR) n0 += int(rank) * (BN / 2);  // this CTA's half of the N tile
        constexpr int BNL = PAIR ? BN / 2 : BN;
        // B boxes of this tile: 64 flattened columns each, inside [0, ntot)
        const int nbox = MODE == WG_STEM ? 28 : max(0, min(BNL / 64, (a.ntot - n0) / 64));
        const uint32_t b_bytes = MODE == WG_STEM ? 28 * KPIX * 16 : nbox * KPIX * 128;
        // per item: each B box's (channel, tap column, tap row) — the single
        // producer thread must not spend its k-loop on divisions
        int bc[BN / 64], bs[BN / 64], br[BN / 64];
#pragma unroll
        for (int b = 0; b < BN / 64; ++b) {
          const int col = n0 + 64 * b, tap = col / a.C;
          bc[b] = col - tap * a.C;
          bs[b] = tap % a.S;
          br[b] = tap / a.S;
        }
        if constexpr (MODE == WG_STEMRAW) {
          // k-block = output row kb: dY rows [kb*Q, kb*Q+Q) and input rows 2p-3+r
          const uint32_t tx = uint32_t(a.Q) * 128u + 7u * uint32_t(a.W2) * 16u;
          int n = kb0 / a.P, p = kb0 - (kb0 / a.P) * a.P;
          for (int kb = kb0; kb < kb1; ++kb, ++it) {
            const uint32_t s = it % STAGES;
            if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], tx);
            tma_load_2d(sA + s * A_STAGE, &amap, &full[s], 0, kb * a.Q);
#pragma unroll
            for (int r = 0; r < 7; ++r)
              tma_load_4d(sB + s * B_STAGE + r * RAW_ROW + RAW_DATA, &bmap, &full[s], 0, 0,
                          2 * p - 3 + r, n);
            if (++p == a.P) {
              p = 0;
              ++n;
            }
          }
          continue;
        }
        // output pixel of the k-block -> (n, p, q), advanced incrementally
        int q = 0, p = 0, n = 0;
        if (MODE != WG_PLAIN) {
          const int pix0 = kb0 * KPIX;
          q = pix0 % a.Q;
          const int t = pix0 / a.Q;
          n = t / a.P;
          p = t - n * a.P;
        }
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const uint32_t s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          const int pix = kb * KPIX;
          // the 64-channel boxes of the A tile only where K has them (rows of D
          // past K are never read back); MT=2 implies K % 256 == 0
          if constexpr (PAIR) {
            // both CTAs' full A halves and B halves land on the leader's
            // barrier; boxes past K / ntot are loaded anyway (zero-filled by
            // the TMA unit) so the byte count is the same in both CTAs
            if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (A_STAGE + B_STAGE));
#pragma unroll
            for (int h = 0; h < 2; ++h)
              tma_load_2d_pair(sA + s * A_STAGE + h * KPIX * 128, &amap, &full[s], m0 + 64 * h, pix);
            if constexpr (MODE == WG_PLAIN) {
#pragma unroll
              for (int b = 0; b < BN / 128; ++b)
                tma_load_2d_pair(sB + s * B_STAGE + b * KPIX * 128, &bmap, &full[s], n0 + 64 * b, pix);
            } else {
              const int wb = q * a.stride - a.pad, hb = p * a.stride - a.pad;
#pragma unroll
              for (int b = 0; b < BN / 128; ++b)
                tma_load_im2col_4d_pair(sB + s * B_STAGE + b * KPIX * 128, &bmap, &full[s], bc[b],
                                        wb, hb, n, uint16_t(bs[b]), uint16_t(br[b]));
            }
          } else {
          const bool a2 = m0 + 64 < a.K;
          mbar_arrive_expect_tx(&full[s], (MT == 2 || a2 ? A_STAGE : A_STAGE / 2) + b_bytes);
#pragma unroll
          for (int h = 0; h < 2 * MT; ++h)
            if (MT == 2 || h == 0 || a2)
              tma_load_2d(sA + s * A_STAGE + h * KPIX * 128, &amap, &full[s], m0 + 64 * h, pix);
          if constexpr (MODE == WG_PLAIN) {
#pragma unroll
            for (int b = 0; b < BN / 64; ++b)
              if (b < nbox)
                tma_load_2d(sB + s * B_STAGE + b * KPIX * 128, &bmap, &full[s], n0 + 64 * b, pix);
          } else if constexpr (MODE == WG_IM2COL) {
            const int wb = q * a.stride - a.pad, hb = p * a.stride - a.pad;
#pragma unroll
            for (int b = 0; b < BN / 64; ++b)
              if (b < nbox)
                tma_load_im2col_4d(sB + s * B_STAGE + b * KPIX * 128, &bmap, &full[s], bc[b],
                                   wb, hb, n, uint16_t(bs[b]), uint16_t(br[b]));
          } else {
            // stem over pixel pairs: 28 taps (7 rows x 4 pairs) x 8 channels
            const int wb = q - 2, hb = p * 2 - 3;
            for (int u = 0; u < 28; ++u)
              tma_load_im2col_4d(sB + s * B_STAGE + u * KPIX * 16, &bmap, &full[s], 0, wb, hb, n,
                                 uint16_t(u & 3), uint16_t(u >> 2));
          }
          }  // !PAIR
          if (MODE != WG_PLAIN) {
            q += KPIX;
            while (q >= a.Q) {
              q -= a.Q;
              if (++p == a.P) {
                p = 0;
                ++n;
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================== MMA issuer ===============================
    if constexpr (MODE == WG_STEMRAW) {
      // the whole warp walks the loop (uniform descriptors: one 64-bit add per
      // MMA), one elected lane issues.  Per 16-pixel step, one M=64 (the 64
      // output channels) x N=32 MMA per filter row r into columns [32r, 32r+32):
      // B = the staged row, MN-major no-swizzle, pixel q's window at +16q (K
      // groups of 8 pixels 128 B apart, the 4 pair columns of a window 16 B
      // apart).  M=64 accumulator rows 16h..16h+15 sit in TMEM lanes 32h..+15.
      constexpr uint32_t idesc32 = umma_idesc_bf16(64, 32) | (1u << 15) | (1u << 16);
      uint32_t it = 0, lt = 0;
      for (int item = blockIdx.x; item < a.items; item += gridDim.x, ++lt) {
        int m0, n0, kb0, kb1;
        decode(item, m0, n0, kb0, kb1);
        const uint32_t acc = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const uint32_t s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          const uint64_t ad0 = desc_mn_sw128(sA + s * A_STAGE, 0);
          const uint64_t bd0 = desc_mn_interleave(sB + s * B_STAGE + RAW_DATA - 32, 128, 16);
          for (int k = 0; k < a.Q / 16; ++k) {
            if (elect_one()) {
#pragma unroll
              for (int r = 0; r < 7; ++r)
                umma_bf16(d + r * 32, ad0 + uint64_t(k) * 128,
                          bd0 + uint64_t(r * (RAW_ROW >> 4) + k * 16), idesc32,
                          (kb != kb0 || k) ? 1u : 0u);
            }
            __syncwarp();
          }
          if (elect_one()) umma_commit(&empty[s]);
          __syncwarp();
        }
        if (elect_one()) umma_commit(&tfull[acc]);
        __syncwarp();
      }
    } else {
      constexpr uint32_t idesc = umma_idesc_bf16(PAIR ? 256 : 128, BN) | (1u << 15) | (1u << 16);
      uint32_t it = 0, lt = 0;
      // pair: only the leader issues
      for (int item = unit; item < ((PAIR && rank != 0) ? 0 : a.items); item += units, ++lt) {
        int m0, n0, kb0, kb1;
        decode(item, m0, n0, kb0, kb1);
        const uint32_t acc = lt % NACC;
        if (lt >= NACC) mbar_wait(&tempty[acc], ((lt / NACC) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const uint32_t s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          tc_fence_after();
          // 16-pixel K steps: 2 KB into the MN-major SW128 tiles (256 B of pairs for the stem)
          const uint64_t ad0 = desc_mn_sw128(sA + s * A_STAGE, KPIX * 128);
          const uint64_t bd0 = MODE == WG_STEM ? desc_mn_interleave(sB + s * B_STAGE, 128, KPIX * 16)
                                               : desc_mn_sw128(sB + s * B_STAGE, KPIX * 128);
          if (elect_one()) {
            if constexpr (PAIR) {
#pragma unroll
              for (int k = 0; k < KPIX / 16; ++k)
                umma_bf16_pair(d, ad0 + uint64_t(k * 128), bd0 + uint64_t(k * 128), idesc,
                               (kb != kb0 || k) ? 1u : 0u);
              umma_commit_pair(&empty[s]);
            } else {
#pragma unroll
            for (int k = 0; k < KPIX / 16; ++k)
#pragma unroll
              for (int h = 0; h < MT; ++h)  // MT=2: the hi 128 channels at +16 KB, columns +BN
                umma_bf16(d + h * BN, ad0 + uint64_t(k * 128 + h * 1024),
                          bd0 + uint64_t(MODE == WG_STEM ? k * 16 : k * 128), idesc,
                          (kb != kb0 || k) ? 1u : 0u);
            umma_commit(&empty[s]);
            }
          }
          __syncwarp();
        }
        if (elect_one()) {
          if constexpr (PAIR)
            umma_commit_pair(&tfull[acc]);
          else
            umma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    // =============================== epilogue ================================
    // Non-stem modes finish the gradient here: one split -> straight into the
    // fp32 KRSC gradient; several -> fp32 partial tiles, and the LAST split of
    // a tile to land (device-scope counter) sums the tile's partials in split
    // order into the gradient (deterministic whichever CTA is last; no
    // separate reduce launch).  The stem keeps its layout-permuting reduce.
    constexpr bool STEMLIKE = MODE == WG_STEM || MODE == WG_STEMRAW;
    __shared__ int s_last;
    const int quarter = warp & 3;
    uint32_t lt = 0;
    for (int item = unit; item < a.items; item += units, ++lt) {
      const uint32_t acc = lt % NACC;
      mbar_wait(&tfull[acc], (lt / NACC) & 1);
      tc_fence_after();
      // WG_STEMRAW (M=64 MMAs): this quarter's lanes 0-15 hold rows 16q..16q+15
      const int row = MODE == WG_STEMRAW ? quarter * 16 + lane : quarter * 32 + lane;
      const bool live = MODE != WG_STEMRAW || lane < 16;
      int m0, n0, kb0, kb1;
      decode(item, m0, n0, kb0, kb1);
      const bool direct = !STEMLIKE && a.fused && a.splits == 1;
      for (int h = 0; h < MT; ++h) {
      // partial tiles are 128*MT rows (pair: 256, this CTA's at +128*rank)
      float* out = a.ws + (size_t(item) * 128 * (PAIR ? 2 : MT) + rank * 128 + h * 128 + row) * BN;
      const int k = m0 + h * 128 + row;
#pragma unroll 1
      for (int j = 0; j < BN / 32; ++j) {
        float v[32];
        tmem_ld_32x32b_x32(tmem + (uint32_t(quarter * 32) << 16) + (acc + h) * BN + j * 32, v);
        if (direct) {
          if (k < a.K && n0 + j * 32 < a.ntot) {
            float4* o = reinterpret_cast<float4*>(a.dw + size_t(k) * a.ntot + n0 + j * 32);
#pragma unroll
            for (int u = 0; u < 8; ++u)
              o[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
          }
          continue;
        }
        float4* o = reinterpret_cast<float4*>(out + j * 32);
        if (live) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            o[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
        }
      }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR)
          mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));  // the leader's
        else
          mbar_arrive(&tempty[acc]);
      }
      if (!STEMLIKE && a.fused && !direct && !PAIR) {
        // publish this split's partial, then count it in
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int tile = item % a.tiles;
        if (threadIdx.x == 64) {
          const unsigned prev = atomicAdd(a.counters + tile, 1u);
          s_last = prev == unsigned(a.splits - 1);
          if (s_last) a.counters[tile] = 0u;  // ready for the next launch
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (s_last) {
          __threadfence();
          for (int h = 0; h < MT; ++h) {
            const int k = m0 + h * 128 + row;
            if (k >= a.K) continue;
            const size_t base = (size_t(tile) * 128 * MT + h * 128 + row) * BN;
            const size_t sstride = size_t(a.tiles) * 128 * MT * BN;
#pragma unroll 1
            for (int j = 0; j < BN / 32; ++j) {
              if (n0 + j * 32 >= a.ntot) break;
              float4 acc4[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) acc4[u] = make_float4(0.f, 0.f, 0.f, 0.f);
              // every split's chunk in flight at once, summed in split order
              float4 t[WG_FUSE_MAX_SPLITS][8];
#pragma unroll
              for (int sp = 0; sp < WG_FUSE_MAX_SPLITS; ++sp)
                if (sp < a.splits) {
                  const float4* src =
                      reinterpret_cast<const float4*>(a.ws + sp * sstride + base + j * 32);
#pragma unroll
                  for (int u = 0; u < 8; ++u) t[sp][u] = __ldcg(src + u);
                }
#pragma unroll
              for (int sp = 0; sp < WG_FUSE_MAX_SPLITS; ++sp)
                if (sp < a.splits) {
#pragma unroll
                  for (int u = 0; u < 8; ++u) {
                    acc4[u].x += t[sp][u].x;
                    acc4[u].y += t[sp][u].y;
                    acc4[u].z += t[sp][u].z;
                    acc4[u].w += t[sp][u].w;
                  }
                }
              float4* o = reinterpret_cast<float4*>(a.dw + size_t(k) * a.ntot + n0 + j * 32);
#pragma unroll
              for (int u = 0; u < 8; ++u) o[u] = acc4[u];
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();
  tc_fence_after();
  if (warp == 1) {
    if constexpr (PAIR)
      tmem_dealloc_pair(tmem, TMEM_COLS);
    else
      tmem_dealloc(tmem, TMEM_COLS);
  }
}

// dW[k][n] (KRSC, n = tap*C + c, fp32) = sum over splits of the partial tiles,
// in split order.  Thread per output element; consecutive threads = consecutive n.
template <int BN, int TM>
__global__ void __launch_bounds__(256)
    k_wgrad_reduce(const float* __restrict__ ws, float* __restrict__ dw, int K, int ntot,
                   int tiles_m, int tiles, int splits) {
  pdl_wait();
  pdl_trigger();
  const int64_t total = int64_t(K) * ntot;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int n = int(e % ntot);
    const int k = int(e / ntot);
    const int tile = (n / BN) * tiles_m + k / TM;
    const size_t off = (size_t(tile) * TM + (k % TM)) * BN + (n % BN);
    const size_t stride = size_t(tiles) * TM * BN;
    float s = 0.f;
    int sp = 0;
    for (; sp + 3 < splits; sp += 4) {  // four loads in flight, same summation order
      const float a0 = ws[size_t(sp) * stride + off], a1 = ws[size_t(sp + 1) * stride + off];
      const float a2 = ws[size_t(sp + 2) * stride + off], a3 = ws[size_t(sp + 3) * stride + off];
      s += a0;
      s += a1;
      s += a2;
      s += a3;
    }
    for (; sp < splits; ++sp) s += ws[size_t(sp) * stride + off];
    dw[e] = s;
  }
}

// stem: partial columns n = (r*4 + j)*8 + e*4 + ch -> dW[k][r][2j+e-1][ch]
__global__ void __launch_bounds__(256)
    k_wgrad_reduce_stem(const float* __restrict__ ws, float* __restrict__ dw, int K, int splits,
                        int tiles) {
  pdl_wait();
  pdl_trigger();
  const int total = K * 7 * 7 * 4;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int ch = e & 3;
    const int s = (e >> 2) % 7;
    const int r = (e / 28) % 7;
    const int k = e / 196;
    const int sp1 = s + 1, j = sp1 >> 1, ee = sp1 & 1;
    const int n = (r * 4 + j) * 8 + ee * 4 + ch;
    const size_t off = (size_t(k / 128) * 128 + (k % 128)) * 256 + n;
    float acc = 0.f;
    for (int sp = 0; sp < splits; ++sp) acc += ws[size_t(sp) * tiles * 128 * 256 + off];
    dw[e] = acc;
  }
}

template <int BN, int MODE, int MT, bool PAIR = false>
constexpr size_t wg_smem_bytes() {
  constexpr int STAGES = wg_stages<MODE, BN, MT, PAIR>();
  constexpr size_t A = MT * 2 * KPIX * 128;
  constexpr size_t B = MODE == WG_STEMRAW ? 7 * RAW_ROW
                       : MODE == WG_STEM  ? 32 * KPIX * 16
                                          : ((PAIR ? BN / 2 : BN) / 64) * KPIX * 128;
  return STAGES * (A + B) + 1024 + 256;
}

int num_sms_wg() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

bool fused_reduce_off() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("DELTA_WGRAD_FUSED_REDUCE");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

template <int BN, int MODE, int MT = 1, bool PAIR = false>
cudaError_t wg_launch(const WgradPlan& wp, const void* dy, const void* x, float* dw, float* ws,
                      cudaStream_t st) {
  auto kern = k_wgrad<BN, MODE, MT, PAIR>;
  constexpr size_t smem = wg_smem_bytes<BN, MODE, MT, PAIR>();
  static_assert(smem <= 227 * 1024, "shared memory");
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  WgArgs a{};
  a.K = wp.K; a.C = wp.C; a.taps = wp.taps; a.S = wp.S; a.P = wp.P; a.Q = wp.Q;
  a.stride = wp.stride; a.pad = wp.pad;
  a.M = wp.N * wp.P * wp.Q;
  a.kblocks = MODE == WG_STEMRAW ? wp.N * wp.P : (a.M + KPIX - 1) / KPIX;
  a.W2 = wp.W / 2;
  constexpr int TM = 128 * (PAIR ? 2 : MT);  // output channels per tile
  a.tiles_m = (wp.K + TM - 1) / TM;
  a.ntot = wp.taps * wp.C;
  a.tiles = wp.tiles;
  a.splits = wp.splits;
  a.kb_per_split = wp.kb_per_split;
  a.items = wp.splits * wp.tiles;
  // the split counters sit at a FIXED place at the head of the workspace (every
  // weight gradient sharing the buffer leaves them zero), the partials after it
  a.counters = reinterpret_cast<unsigned*>(ws);
  ws = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + WG_COUNTER_BYTES);
  (void)TM;
  a.ws = ws;
  a.dw = dw;
  // fused finish only for few splits: the last split's CTA sums the tile alone
  // (with many splits the all-SM reduce launch is faster: 28 vs 21 ms/step for
  // ResNet-50, whose 1x1 weight gradients split 100-way over the pixels)
  a.fused = (fused_reduce_off() || wp.tiles > int(WG_COUNTER_BYTES / 4) ||
             wp.splits > WG_FUSE_MAX_SPLITS) ? 0 : 1;
  alignas(64) CUtensorMap amap, bmap;
  if (!tma_2d_bf16(&amap, dy, uint64_t(wp.K), uint64_t(a.M), uint64_t(wp.K), 64,
                   MODE == WG_STEMRAW ? uint32_t(wp.Q) : uint32_t(KPIX), CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  static_assert(!PAIR || MT == 1, "pair tiles: one accumulator per CTA");
  bool ok;
  if (MODE == WG_PLAIN) {
    ok = tma_2d_bf16(&bmap, x, uint64_t(wp.C), uint64_t(a.M), uint64_t(wp.C), 64, KPIX,
                     CU_TENSOR_MAP_SWIZZLE_128B);
  } else if (MODE == WG_IM2COL) {
    ok = tma_im2col_bf16(&bmap, x, wp.C, wp.W, wp.H, wp.N, -wp.pad, -wp.pad,
                         wp.pad - (wp.S - 1), wp.pad - (wp.R - 1), wp.stride, wp.stride, 64, KPIX,
                         CU_TENSOR_MAP_SWIZZLE_128B);
  } else if (MODE == WG_STEMRAW) {
    ok = stem_raw_rows_map(&bmap, x, wp.N, wp.H, wp.W);
  } else {  // stem: [N][H][W/2][8] pixel pairs, stride (w 1, h 2)
    const int W2 = wp.W / 2;
    ok = tma_im2col_bf16(&bmap, x, 8, W2, wp.H, wp.N, -2, -3, wp.Q - W2 - 2, 2 * wp.P - wp.H - 3,
                         1, 2, 8, KPIX, CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  if (!ok) return cudaErrorInvalidValue;
  if constexpr (PAIR) {
    const int pairs = std::min(a.items, num_sms_wg() / 2);
    if (cudaError_t e_ = launch_cluster(kern, dim3(2 * pairs), dim3(WG_THREADS), smem, st, 2u, amap,
                                        bmap, a))
      return e_;
  } else {
    const int grid = std::min(a.items, num_sms_wg());
    if (cudaError_t e_ = launch_k(kern, dim3(grid), dim3(WG_THREADS), smem, st, amap, bmap, a)) return e_;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (MODE == WG_STEM || MODE == WG_STEMRAW) {
    if (cudaError_t e_ = launch_k(k_wgrad_reduce_stem, dim3((wp.K * 196 + 255) / 256), dim3(256), 0, st, ws, dw, wp.K, wp.splits, wp.tiles)) return e_;
  } else if (!a.fused) {  // many splits, or DELTA_WGRAD_FUSED_REDUCE=0: the all-SM reduce
    const int64_t total = int64_t(wp.K) * a.ntot;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
    if (cudaError_t e_ = launch_k(k_wgrad_reduce<BN, 128 * (PAIR ? 2 : MT)>, dim3(int(blocks)), dim3(256), 0, st, ws, dw, wp.K, a.ntot, a.tiles_m, wp.tiles, wp.splits)) return e_;
  }
  return cudaGetLastError();
}

}  // namespace

int wgrad_plan_init(WgradPlan* wp) {
  WgradPlan& p = *wp;
  const bool stem = p.C == 4;
  if (stem) {
    if (p.R != 7 || p.S != 7 || p.stride != 2 || p.pad != 3 || (p.W & 1)) return 1;
  } else if (p.C % 64 != 0) {
    return 1;
  }
  if (p.K % 64 != 0) return 1;
  p.P = (p.H + 2 * p.pad - p.R) / p.stride + 1;
  p.Q = (p.W + 2 * p.pad - p.S) / p.stride + 1;
  const char* sm = std::getenv("DELTA_STEM_MODE");
  p.mode = stem ? (p.Q % 16 == 0 && p.Q <= 124 && p.K <= 64 && !(sm && sm[0]) ? WG_STEMRAW : WG_STEM)
                : (p.R == 1 && p.S == 1 && p.stride == 1 && p.pad == 0 ? WG_PLAIN : WG_IM2COL);
  p.taps = stem ? 1 : p.R * p.S;
  const int ntot = p.taps * p.C;  // flattened (tap, channel) columns
  // N tile: 256, unless 256-wide tiles would leave much padding and 192 none
  // (3x3 over 64 channels: 576 = 3 x 192 instead of 3 x 256 with a quarter-
  // full last tile: 120 -> 108 us; at 1152 = 4.5 x 256 the 256 tiles win)
  p.bn = stem ? 256 : (ntot >= 256 ? 256 : (ntot >= 128 ? 128 : 64));
  if (!stem && ntot % 192 == 0 && ntot > 256 &&
      double(ntot) / (double((ntot + 255) / 256) * 256.0) < 0.85)
    p.bn = 192;
  // 256-channel tiles (two accumulators on one B tile) for the 3x3 convs with
  // K % 256 == 0 (measured: 62.5 -> 57.5 us at 14x14x256, 76 -> 60 us at
  // 7x7x512); the 1x1 shapes' short items lose more to the undoubled
  // accumulator drain than they gain (39 -> 48 us at 14x14 256->1024)
  static const bool mt2_on = [] {
    const char* e = std::getenv("DELTA_WGRAD_MT2");
    return !(e && e[0] == '0');
  }();
  p.mt = (!stem && mt2_on && p.taps > 1 && p.bn == 256 && p.K % 256 == 0) ? 2 : 1;
  // CTA-pair 256-channel tiles (cta_group::2) for the plain 1x1 shapes with
  // whole 256x256 tiles (DELTA_WGRAD_PAIR=0 disables)
  static const bool pair_on = [] {
    const char* e = std::getenv("DELTA_WGRAD_PAIR");
    return !(e && e[0] == '0');
  }();
  p.pair = (pair_on && !stem && p.mt == 1 && p.mode == WG_PLAIN && p.bn == 256 &&
            p.K % 256 == 0 && ntot % 256 == 0) ? 1 : 0;
  const int tm = 128 * (p.pair ? 2 : p.mt);
  const int tiles_m = (p.K + tm - 1) / tm;
  p.tiles = stem ? tiles_m : tiles_m * ((ntot + p.bn - 1) / p.bn);
  const int M = p.N * p.P * p.Q;
  const int kblocks = p.mode == WG_STEMRAW ? p.N * p.P : (M + KPIX - 1) / KPIX;
  // Split count: minimise the modelled makespan — whole waves of work items
  // over the SMs (a partial last wave costs a full one) times the item
  // length, plus the fp32 partials written and re-read by the reduce.
  // (Rounding "two waves" up left 30% of the SMs idle in the last wave.)
  const int sms = p.pair ? 74 : 148;  // scheduling units (CTA pairs)
  const double t_kb = p.mode == WG_STEMRAW ? 1.3e-6                       // one output row
                                           : 2.0 * 128 * p.mt * p.bn * KPIX / (1.0e15 / 148);
  const double t_ramp = 1.5 * t_kb;  // per item: pipeline fill + accumulator drain
  const double part_bytes = 8.0 * p.tiles * tm * p.bn;  // per split: write + reduce read
  const int smax = std::max(1, kblocks / (p.mode == WG_STEMRAW ? 4 : 8));
  int splits = 1;
  double best = 1e30;
  for (int sp = 1; sp <= smax; ++sp) {
    const int kbps = (kblocks + sp - 1) / sp;
    const int s_eff = (kblocks + kbps - 1) / kbps;
    if (s_eff != sp) continue;  // same partition as a smaller count
    const int waves = (s_eff * p.tiles + sms - 1) / sms;
    const double t = waves * (kbps * t_kb + t_ramp) + s_eff * part_bytes / 6e12;
    if (t < best * 0.999) {
      best = t;
      splits = s_eff;
    }
  }
  p.kb_per_split = (kblocks + splits - 1) / splits;
  p.splits = (kblocks + p.kb_per_split - 1) / p.kb_per_split;
  return 0;
}

int wgrad_launches(const WgradPlan& wp) {
  const bool stem = wp.mode == WG_STEM || wp.mode == WG_STEMRAW;
  const bool fused = !fused_reduce_off() && wp.tiles <= int(WG_COUNTER_BYTES / 4) &&
                     wp.splits <= WG_FUSE_MAX_SPLITS;
  return stem || !fused ? 2 : 1;
}

size_t wgrad_workspace_bytes(const WgradPlan& wp) {
  // the per-tile split counters (must be zero at allocation) + partial tiles
  return WG_COUNTER_BYTES +
         size_t(wp.splits) * wp.tiles * 128 * (wp.pair ? 2 : wp.mt) * wp.bn * sizeof(float);
}

cudaError_t wgrad(const WgradPlan& wp, const void* dy, const void* x, float* dw, float* ws,
                  cudaStream_t st) {
  if (wp.mode == WG_STEMRAW) return wg_launch<256, WG_STEMRAW>(wp, dy, x, dw, ws, st);
  if (wp.mode == WG_STEM) return wg_launch<256, WG_STEM>(wp, dy, x, dw, ws, st);
  switch (wp.bn) {
    case 64:
      return wp.mode == WG_PLAIN ? wg_launch<64, WG_PLAIN>(wp, dy, x, dw, ws, st)
                                 : wg_launch<64, WG_IM2COL>(wp, dy, x, dw, ws, st);
    case 128:
      return wp.mode == WG_PLAIN ? wg_launch<128, WG_PLAIN>(wp, dy, x, dw, ws, st)
                                 : wg_launch<128, WG_IM2COL>(wp, dy, x, dw, ws, st);
    case 192:
      return wp.mode == WG_PLAIN ? wg_launch<192, WG_PLAIN>(wp, dy, x, dw, ws, st)
                                 : wg_launch<192, WG_IM2COL>(wp, dy, x, dw, ws, st);
    default:
      if (wp.pair) return wg_launch<256, WG_PLAIN, 1, true>(wp, dy, x, dw, ws, st);
      if (wp.mt == 2)
        return wp.mode == WG_PLAIN ? wg_launch<256, WG_PLAIN, 2>(wp, dy, x, dw, ws, st)
                                   : wg_launch<256, WG_IM2COL, 2>(wp, dy, x, dw, ws, st);
      return wp.mode == WG_PLAIN ? wg_launch<256, WG_PLAIN>(wp, dy, x, dw, ws, st)
                                 : wg_launch<256, WG_IM2COL>(wp, dy, x, dw, ws, st);
  }
}

}  // namespace delta_k
