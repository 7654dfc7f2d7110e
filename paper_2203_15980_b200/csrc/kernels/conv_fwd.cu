// Implicit-GEMM convolution forward for sm_100a (tcgen05 + TMEM + TMA).
//
// The one dense contraction of the recompute engine: every ConvForward node of
// the ResNet trace (stem 7x7/2, 3x3 s1/s2, 1x1, downsample 1x1/2) runs through
// this kernel both when it is first produced and when DELTA re-materialises
// it, so a recompute is bitwise identical to the original (fixed tiling, fixed
// K order, no split-K, no atomics).
//
// GEMM view (NHWC activations, KRSC weights):
//   Y[m = (n,p,q), k] = sum_{kk = (r,s,c)} X[n, p*st-pad+r, q*st-pad+s, c] * W[k, kk]
// Tile 128 x BN x 64, fp32 accumulators in TMEM.
//
// Persistent, warp-specialised (one CTA per SM, static round-robin tiles):
//   warps 0-3 : producers.  MODE_IM2COL (3x3, strided 1x1): A by the TMA
//               im2col unit (out-of-image taps zero-filled = the padding);
//               MODE_STEMRAW (the C=4 stem): raw input rows, one output row
//               per tile, A addressed straight into them (see below);
//               MODE_TMA (1x1, stride 1): A is a plain [M, C] matrix loaded
//               by TMA; MODE_GATHER (opt-in, DELTA_CONV_GATHER=1) and
//               MODE_STEMG: cp.async im2col; MODE_STEM: TMA im2col over pixel
//               pairs (wide stems).  The weight tile B is one TMA load.
//   warps 4-11: epilogue — TMEM -> registers -> bf16 -> HBM; two warps per
//               TMEM lane quarter, alternating 32-column chunks (8 epilogue
//               warps: the per-chunk work — fused operands, ReLU masks, BN
//               partials — was the pacing stage with 4).
//   warp 12   : TMEM allocation + single-thread tcgen05.mma issue.
// Two TMEM accumulators: the epilogue of tile i drains one while the MMAs of
// tile i+1 fill the other.  smem stages ring with full/empty mbarriers;
// tcgen05.commit releases a stage the moment the tensor core has consumed it.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "kernels/gelu.cuh"
#include "kernels/kernels.hpp"
#include "kernels/launch.hpp"
#include "kernels/sm100_common.cuh"
#include "kernels/stats_cta.cuh"
#include "kernels/tma_host.hpp"

namespace delta_k {

using namespace dsm100;
using bf16 = __nv_bfloat16;

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
// warps 0-3 producers, 4 .. 4+EPI_W-1 epilogue (EPI_W/4 warps per TMEM lane
// quarter, splitting a tile's 32-column chunks), then the MMA warp
#ifndef DELTA_CONV_EPI_WARPS
#define DELTA_CONV_EPI_WARPS 8
#endif
constexpr int EPI_W = DELTA_CONV_EPI_WARPS;
constexpr int MMA_WARP = 4 + EPI_W;
constexpr int kThreads = (MMA_WARP + 1) * 32;
constexpr int MODE_GATHER = 0, MODE_STEM = 1, MODE_TMA = 2, MODE_IM2COL = 3, MODE_STEMG = 4,
              MODE_STEMRAW = 5;
// one output row per tile (rows >= Q of the 128-row tile are junk)
constexpr bool row_tiled(int mode) { return mode == MODE_STEMRAW; }
// MODE_STEMRAW: smem bytes per staged input row.  The row's pixel pairs land
// at +RAW_DATA (128 B aligned for the TMA), pairs -2, -1 and W/2, W/2+1 are
// zeros written once; the junk tile rows q < 128 read up to pair q+3.
constexpr uint32_t RAW_ROW = 2304, RAW_DATA = 128;
// A operand written by the producer threads (cp.async) rather than the TMA unit
constexpr bool gathers(int mode) { return mode == MODE_GATHER || mode == MODE_STEMG; }
// fused-epilogue operand ring: 24 KB per epilogue warp, slots of one 2 KB
// block per operand (12 slots with one operand, 6 with two)
// Fused-epilogue operand ring (all epilogue warps): whatever shared memory the
// operand stages, the output staging and the statistics scratch leave, in
// whole 2 KB blocks per warp — the ring depth is what keeps the epilogue's
// operand reads in flight.
constexpr uint32_t SMEM_MAX = 232448;
// fused epilogues: per-warp BN scale/shift of the 32 chunk columns (float2 x 32)
constexpr uint32_t SCSH_BYTES = EPI_W * 256;
template <int BN, int STAGES>
constexpr uint32_t epi_ring_bytes() {
  return (SMEM_MAX - 1024 - 256 - 4 * BN * 8 - 16384 - SCSH_BYTES -
          STAGES * (128 * 128 + BN * 128)) /
         (EPI_W * 2048) * (EPI_W * 2048);
}



struct ConvArgs {
  const bf16* x;
  bf16* y;
  int N, H, W, C, K, R, S, stride, pad, P, Q;
  int M;        // N*P*Q
  int kblocks;  // reduction length / 64
  int taps;     // R*S
  int n_tiles;  // ceil(K / BN)
  int tiles;    // m_tiles * n_tiles
  float4* stats;  // optional per-CTA partials [grid][K] (stats_cta.cuh): EPI_STORE (count,
                  // mean, M2) of the bf16 outputs; EPI_BN_BWD (sum g, sum g*xc)
  ConvEpilogue e;
};

// ---- epilogue helpers (one thread = one output row, 32 columns per chunk) ----
__device__ __forceinline__ uint4 ldg16(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ void unpack8f(uint4 u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// Row `lane` (16 B chunk u) of a 32x32 bf16 block staged in smem with the 64B
// swizzle (the layout of the TMA boxes the epilogue loads and stores).
__device__ __forceinline__ uint4 ld_row16(uint32_t buf, int lane, int u) {
  uint4 r;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(buf + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4)));
  return r;
}

// Compile-time epilogue variants (the runtime ConvEpilogue.mode picks one at
// launch): straight-line code, operand presence known, packed bf16x2 math.
constexpr int EV_STORE = 0;    // y = bf16(acc)                       [+ BN-stats partials]
constexpr int EV_ADD = 1;      // y = bf16(acc) + add
constexpr int EV_ADD_OM = 2;   // y = (bf16(acc) + add) & [out_mask > 0]
constexpr int EV_POOL = 3;     // y = bf16(acc + pooled/hw * [add_mask > 0]) & [out_mask > 0]
constexpr int EV_BN_BWD = 4;   // y = g = bf16(acc) & [relu(bn(xc)) > 0]; partials (sum g, sum g*xc)
constexpr int EV_ADD_OM_ST = 5;  // EV_ADD_OM + partials (sum y, sum y*xc): the next BN's backward sums
constexpr int EV_SCATTER = 6;  // y[n][2p+a][2q+b] = bf16(acc): a stride-2 input gradient's parity class
constexpr int EV_BIAS = 7;     // y = bf16(acc + bias[k])                     (linear layers)
constexpr int EV_GELU_BWD = 8; // y = bf16(acc * gelu'(xc)), xc = the [M][K] pre-activation
constexpr int EV_ADD_S2 = 9;   // y = (bf16(acc) + add at even (p, q)) & [out_mask > 0]: the add is
                               // a stride-2 shortcut gradient on its [N][P/2][Q/2] grid, read
                               // straight by the lanes of even rows; out_mask by TMA
// epilogues that read [M][K] operand tiles (the operand ring / tile buffers)
__host__ __device__ constexpr bool ev_fused(int ev) {
  return ev != EV_STORE && ev != EV_SCATTER && ev != EV_BIAS;
}
__host__ __device__ constexpr int ev_operands(int ev) {
  return ev == EV_ADD || ev == EV_BN_BWD || ev == EV_GELU_BWD || ev == EV_ADD_S2
             ? 1
             : (ev == EV_ADD_OM || ev == EV_POOL ? 2 : (ev == EV_ADD_OM_ST ? 3 : 0));
}
// epilogues whose statistics are (sum y, sum y*xc) rather than (count, mean, M2)
__host__ __device__ constexpr bool ev_cross(int ev) { return ev == EV_BN_BWD || ev == EV_ADD_OM_ST; }
__host__ __device__ constexpr bool ev_adds(int ev) {
  return ev == EV_ADD || ev == EV_ADD_OM || ev == EV_ADD_OM_ST;
}

// bf16x2 lanes positive (> +0) -> 0xFFFF, else 0 (bf16 bit patterns read as
// int16: positive values are exactly the positive int16s)
__device__ __forceinline__ uint32_t pos_mask2(uint32_t w) { return __vcmpgts2(w, 0u); }
__device__ __forceinline__ uint32_t add_bf16x2(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hadd2(*reinterpret_cast<__nv_bfloat162*>(&a),
                             *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// EV != EV_STORE: the epilogue reads one or two [M][K] operand blocks (t0,
// t1) per 32x32 chunk, cp.async-loaded (slots - 1) chunks ahead into a
// per-warp ring (a chunk's math is far shorter than an HBM round trip; 64 B-row
// TMA boxes were issue-bound).
// OPT: the fused epilogue's operands ([M][K] tensors: add, out_mask, xc) are
// TMA-loaded per tile by producer warp 1 into a double-buffered tile slot
// (32-column x 128-row boxes, the same 64B-swizzled layout the cp.async ring
// uses), instead of per-chunk cp.async gathers by the epilogue warps.
constexpr int OPT_NB = 2;

// PAIR: a 2-CTA cluster (cta_group::2) computes 256-row tiles — each CTA
// stages its 128 rows of A and half of the BN weight rows, the leader issues
// M=256 MMAs that read both CTAs' operands, each CTA's TMEM holds its rows —
// halving the per-SM operand traffic of the B tile (MODE_TMA only).
// BMN: the weight tile is MN-major — weights stored [kdim][K], loaded as
// 64 x 64 boxes (64 K-rows of 128 B along N) and read through MN-major
// descriptors (no transposed weight copy for the input-gradient GEMMs).
template <int BN, int STAGES, int MODE, int EV, bool OPT = false, bool PAIR = false,
          bool BMN = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_fwd(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap,
               const __grid_constant__ CUtensorMap ymap, const __grid_constant__ CUtensorMap emap0,
               const __grid_constant__ CUtensorMap emap1, const __grid_constant__ CUtensorMap emap2,
               const ConvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  // producer signalling lag: a thread keeps LAG+1 stages of gathers in flight
  constexpr uint32_t LAG = STAGES - 2;
  static_assert(!PAIR || ((MODE == MODE_TMA || MODE == MODE_IM2COL) && BN >= 128),
                "pair mode: TMA / TMA-im2col operand paths, N tile 128 or 256");
  constexpr uint32_t A_STAGE = BM * 128;
  constexpr uint32_t B_STAGE = (PAIR ? BN / 2 : BN) * 128;  // this CTA's weight rows
  constexpr uint32_t ACC_COLS = BN;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  const uint32_t sA = smem_u32(smem);
  const uint32_t sB = sA + STAGES * A_STAGE;
  // epilogue staging: 4 warps x 2 buffers x (32 rows x 64 B), 64B-swizzled
  const uint32_t sOut = sA + STAGES * (A_STAGE + B_STAGE);
  // fused-epilogue operand ring: EPI_W warps x EPI_RING_WARP
  constexpr bool FUSED = ev_fused(EV);
  constexpr uint32_t EPI_RING_WARP = epi_ring_bytes<BN, STAGES>() / EPI_W;
  constexpr int NOPS_ = ev_operands(EV);
  constexpr uint32_t OPT_TILE = uint32_t(NOPS_) * BN * 256;  // per tile: NOPS x [128][BN] bf16
  static_assert(EV != EV_ADD_OM_ST || OPT, "three-operand epilogue: TMA-loaded operands only");
  static_assert(EV != EV_ADD_S2 || OPT, "stride-2 add epilogue: TMA-loaded mask only");
  constexpr uint32_t IN_BYTES = !FUSED ? 0 : (OPT ? OPT_NB * OPT_TILE : EPI_W * EPI_RING_WARP);
  const uint32_t sIn = sOut + 16384;
  // BN-statistics scratch: per quarter-warp column (sum, sumsq), [4][BN] float2
  float2* red = reinterpret_cast<float2*>(smem + STAGES * (A_STAGE + B_STAGE) + 16384 + IN_BYTES);
  // FUSED: [EPI_W][32] float2 per-warp BN scale/shift scratch after the statistics scratch
  const uint32_t sScSh = sIn + IN_BYTES + 4 * BN * sizeof(float2);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (A_STAGE + B_STAGE) + 16384 +
                                               IN_BYTES + 4 * BN * sizeof(float2) +
                                               (FUSED ? SCSH_BYTES : 0));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* bfull = tempty + 2;      // MODE_STEMRAW: resident weights landed
  uint64_t* ofull = bfull + 1;       // OPT: epilogue operand tile landed [OPT_NB]
  uint64_t* oempty = ofull + OPT_NB; // OPT: ... and consumed [OPT_NB]
  uint64_t* otrans = oempty + OPT_NB; // XFORM: ... and transformed [OPT_NB]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(otrans + OPT_NB);
  // EV_GELU_BWD: producer warps 1-3 (idle in the TMA mode; warp 0 then also
  // loads the operand tiles) turn each landed pre-activation tile into
  // gelu'(pre) in place (fp16), so the epilogue's per-element work is one
  // multiply
  constexpr bool XFORM = EV == EV_GELU_BWD && OPT;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // tile scheduling unit: the CTA, or the CTA pair
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int unit = PAIR ? int(blockIdx.x >> 1) : int(blockIdx.x);
  const int units = PAIR ? int(gridDim.x >> 1) : int(gridDim.x);
  constexpr int TM = PAIR ? 2 * BM : BM;  // rows per tile
  auto tile_m0 = [&](int tile) { return (tile / a.n_tiles) * TM + int(rank) * BM; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], gathers(MODE) ? 4 + 1 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      // pair: the leader's MMA waits for both CTAs' epilogues
      mbar_init(&tempty[i], PAIR ? 2 * EPI_W : EPI_W);
    }
    mbar_init(bfull, 1);
    for (int i = 0; i < OPT_NB; ++i) {
      mbar_init(&ofull[i], 1);
      mbar_init(&oempty[i], EPI_W);
      mbar_init(&otrans[i], 3);
    }
    fence_mbar_init();
    if (OPT) {
      tma_prefetch_desc(&emap0);
      if (NOPS_ >= 2) tma_prefetch_desc(&emap1);
      if (NOPS_ == 3) tma_prefetch_desc(&emap2);
    }
    tma_prefetch_desc(&wmap);
    if (!gathers(MODE)) tma_prefetch_desc(&amap);
    tma_prefetch_desc(&ymap);
  }
  if constexpr (MODE == MODE_STEMRAW) {
    // the padding pairs around every staged input row: zero once (the TMA
    // only ever writes the W/2 data pairs between them)
    const uint32_t data_end = RAW_DATA + uint32_t(a.W >> 1) * 16;
    for (int i = threadIdx.x; i < STAGES * 7 * 4; i += blockDim.x) {
      const int row = i >> 2, part = i & 3;
      const uint32_t off = (part < 2 ? RAW_DATA - 32 : data_end) + (part & 1) * 16;
      st_shared_v4(sA + (row / 7) * A_STAGE + (row % 7) * RAW_ROW + off, make_uint4(0, 0, 0, 0));
    }
    fence_proxy_async_smem();
  }
  if (warp == MMA_WARP) {
    if constexpr (PAIR)
      tmem_alloc_pair(tslot, TMEM_COLS);
    else
      tmem_alloc(tslot, TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // the peer's barriers exist before any remote use
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // prologue done (barriers, TMEM, descriptors): now wait for the predecessor
  pdl_wait();
  pdl_trigger();

  if (warp < 4) {
    // ============================ producers ============================
    const int tid = threadIdx.x;
    if (OPT && !XFORM && warp == 1) {
      if constexpr (OPT) {
        // epilogue operands of every tile of this CTA, two tiles ahead
        if (lane == 0) {
          uint32_t lt = 0;
          for (int tile = unit; tile < a.tiles; tile += units, ++lt) {
            const int m0 = tile_m0(tile);
            const int n0 = (tile % a.n_tiles) * BN;
            const uint32_t b = lt % OPT_NB;
            if (lt >= OPT_NB) mbar_wait(&oempty[b], ((lt / OPT_NB) - 1) & 1);
            mbar_arrive_expect_tx(&ofull[b], OPT_TILE);
            const uint32_t base = sIn + b * OPT_TILE;
#pragma unroll
            for (int j = 0; j < BN / 32; ++j) {
              tma_load_2d(base + j * 8192, &emap0, &ofull[b], n0 + j * 32, m0);
              if (NOPS_ >= 2)
                tma_load_2d(base + BN * 256 + j * 8192, &emap1, &ofull[b], n0 + j * 32, m0);
              if (NOPS_ == 3)
                tma_load_2d(base + 2 * BN * 256 + j * 8192, &emap2, &ofull[b], n0 + j * 32, m0);
            }
          }
        }
      }
    } else if (XFORM && warp >= 1) {
      if constexpr (XFORM) {
        // gelu'(pre) of every operand tile, in place, as fp16 pairs
        const int t2 = threadIdx.x - 32;
        uint32_t lt = 0;
        for (int tile = unit; tile < a.tiles; tile += units, ++lt) {
          const uint32_t b = lt % OPT_NB;
          mbar_wait(&ofull[b], (lt / OPT_NB) & 1);
          uint4* buf = reinterpret_cast<uint4*>(smem + (sIn - sA) + b * OPT_TILE);
#pragma unroll 2
          for (int i = t2; i < int(OPT_TILE / 16); i += 96) {
            float f[8];
            unpack8f(buf[i], f);
            uint32_t o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const __half2 hv = __floats2half2_rn(gelu_grad1(f[2 * k]), gelu_grad1(f[2 * k + 1]));
              o[k] = *reinterpret_cast<const uint32_t*>(&hv);
            }
            buf[i] = make_uint4(o[0], o[1], o[2], o[3]);
          }
          fence_proxy_async_smem();  // before the buffer's next TMA refill
          __syncwarp();
          if (lane == 0) mbar_arrive(&otrans[b]);
        }
      }
    } else {
    uint32_t it = 0;  // global k-iteration counter (stage ring position)
    for (int tile = unit; tile < a.tiles; tile += units) {
      const int m0 = tile_m0(tile);
      const int n0 = (tile % a.n_tiles) * BN;
      if constexpr (MODE == MODE_IM2COL) {
        if (tid == 0) {
          // tile's first output pixel -> base input coordinate of its window
          const int q = m0 % a.Q;
          const int t = m0 / a.Q;
          const int n = t / a.P;
          const int wb = q * a.stride - a.pad;
          const int hb = (t - n * a.P) * a.stride - a.pad;
          int tap = 0, c0 = 0;
          for (int kb = 0; kb < a.kblocks; ++kb, ++it) {
            const uint32_t s = it % STAGES;
            if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
            const int r = tap / a.S, sx = tap - r * a.S;
            if constexpr (PAIR) {
              if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (A_STAGE + B_STAGE));
              tma_load_im2col_4d_pair(sA + s * A_STAGE, &amap, &full[s], c0, wb, hb, n,
                                      uint16_t(sx), uint16_t(r));
              tma_load_2d_pair(sB + s * B_STAGE, &wmap, &full[s], kb * BK,
                               n0 + int(rank) * (BN / 2));
            } else {
              mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
              tma_load_im2col_4d(sA + s * A_STAGE, &amap, &full[s], c0, wb, hb, n, uint16_t(sx),
                                 uint16_t(r));
              tma_load_2d(sB + s * B_STAGE, &wmap, &full[s], kb * BK, n0);
            }
            c0 += 64;
            if (c0 == a.C) {
              c0 = 0;
              ++tap;
            }
          }
        }
      } else if constexpr (MODE == MODE_STEMRAW) {
        // Stem, one output row (n, p) per tile, no im2col at all: the 7 input
        // rows 2p-3+r are staged as they are (pixel pairs, 2 zero pairs of
        // padding each side from the TMA's out-of-bounds fill), and the MMA
        // reads A straight from them: row q, K-chunk j of filter row r is
        // pair q-2+j, i.e. a K-major no-swizzle operand with 16 B between
        // K-adjacent core matrices and 128 B between M-adjacent ones
        // (overlapping core matrices — each staged pair feeds 4 output
        // columns).  The 32 KB of weights stay resident (loaded once).
        const int n = tile / a.P;
        const int p = tile - n * a.P;
        if (tid == 0) {
          if (tile == int(blockIdx.x)) {
            mbar_arrive_expect_tx(bfull, 4 * B_STAGE);
            for (int kb = 0; kb < 4; ++kb) tma_load_2d(sB + kb * B_STAGE, &wmap, bfull, kb * BK, 0);
          }
          const uint32_t s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          mbar_arrive_expect_tx(&full[s], 7u * uint32_t(a.W >> 1) * 16u);
#pragma unroll
          for (int r = 0; r < 7; ++r)
            tma_load_4d(sA + s * A_STAGE + r * RAW_ROW + RAW_DATA, &amap, &full[s], 0, 0,
                        2 * p - 3 + r, n);
        }
        ++it;
      } else if constexpr (MODE == MODE_STEM) {
        // 7x7/2 stem over C=4 viewed as pixel PAIRS (16 B = 8 channels): a
        // 7x4 stride-(2,1) conv, one 128-pixel x 16 B im2col box per tap,
        // 8 taps per k-block written as K-adjacent no-swizzle core-matrix
        // columns 2 KB apart (taps >= 28 repeat tap 27 against zero weights)
        if (tid == 0) {
          const int q = m0 % a.Q;
          const int t = m0 / a.Q;
          const int n = t / a.P;
          const int wb = q - 2;
          const int hb = (t - n * a.P) * 2 - 3;
          for (int kb = 0; kb < a.kblocks; ++kb, ++it) {
            const uint32_t s = it % STAGES;
            if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int tap = min(kb * 8 + u, 27);
              tma_load_im2col_4d(sA + s * A_STAGE + u * 2048, &amap, &full[s], 0, wb, hb, n,
                                 uint16_t(tap & 3), uint16_t(tap >> 2));
            }
            tma_load_2d(sB + s * B_STAGE, &wmap, &full[s], kb * BK, n0);
          }
        }
      } else if constexpr (MODE == MODE_TMA) {
        if (tid == 0) {
          if constexpr (XFORM) {
            // this tile's epilogue operand (two tiles of buffering)
            const uint32_t lt = it / uint32_t(a.kblocks);  // tiles issued so far
            const uint32_t b = lt % OPT_NB;
            if (lt >= OPT_NB) mbar_wait(&oempty[b], ((lt / OPT_NB) - 1) & 1);
            mbar_arrive_expect_tx(&ofull[b], OPT_TILE);
#pragma unroll
            for (int j = 0; j < BN / 32; ++j)
              tma_load_2d(sIn + b * OPT_TILE + j * 8192, &emap0, &ofull[b], n0 + j * 32, m0);
          }
          for (int kb = 0; kb < a.kblocks; ++kb, ++it) {
            const uint32_t s = it % STAGES;
            if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
            if constexpr (PAIR) {
              // both CTAs' bytes complete on the leader's barrier
              if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * (A_STAGE + B_STAGE));
              tma_load_2d_pair(sA + s * A_STAGE, &amap, &full[s], kb * BK, m0);
              if constexpr (BMN) {
#pragma unroll
                for (int b = 0; b < BN / 128; ++b)
                  tma_load_2d_pair(sB + s * B_STAGE + b * 8192, &wmap, &full[s],
                                   n0 + int(rank) * (BN / 2) + 64 * b, kb * BK);
              } else {
                tma_load_2d_pair(sB + s * B_STAGE, &wmap, &full[s], kb * BK,
                                 n0 + int(rank) * (BN / 2));
              }
            } else {
              mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
              tma_load_2d(sA + s * A_STAGE, &amap, &full[s], kb * BK, m0);
              if constexpr (BMN) {
#pragma unroll
                for (int b = 0; b < BN / 64; ++b)
                  tma_load_2d(sB + s * B_STAGE + b * 8192, &wmap, &full[s], n0 + 64 * b, kb * BK);
              } else {
                tma_load_2d(sB + s * B_STAGE, &wmap, &full[s], kb * BK, n0);
              }
            }
          }
        }
      } else {
        constexpr int ROWS = 8;
        constexpr int RSTEP = 16;
        const int part = tid & 7;
        const int row0 = tid >> 3;
        // Per tile, once: each row's input base pointer (top-left tap, may
        // point into the padding) and a validity mask: bits [0,R) say which
        // filter rows land inside the image, bits [8,8+S) which columns.
        // Per k-block the only address math left is one scalar tap offset.
        const bf16* rowp[ROWS];
        uint32_t vm[ROWS];
        {
          // decode (n, p, q) of this thread's first row once, then step by
          // RSTEP rows (a division-free walk: RSTEP < Q for every ResNet conv
          // but the loop handles any Q)
          const int mfirst = m0 + row0;
          int q = mfirst % a.Q;
          const int t = mfirst / a.Q;
          int n = t / a.P;
          int p = t - n * a.P;
          const bool stem = MODE == MODE_STEMG;
          const int R = stem ? 7 : a.R, S = stem ? 4 : a.S;
          const int Wv = stem ? (a.W >> 1) : a.W;          // pixels (pairs for the stem)
          const long long pix = stem ? 8ll : (long long)a.C;  // elements per (pair) pixel
          const int st = stem ? 2 : a.stride, sp = stem ? 3 : a.pad;
#pragma unroll
          for (int i = 0; i < ROWS; ++i) {
            const int m = mfirst + RSTEP * i;
            vm[i] = 0;
            rowp[i] = a.x;
            if (m < a.M) {
              const int hb = p * st - sp;
              const int wb = stem ? q - 2 : q * st - sp;
              rowp[i] = a.x + (((long long)n * a.H + hb) * Wv + wb) * pix;
              // valid filter rows r: 0 <= hb + r < H; columns c: 0 <= wb + c < Wv
              const int rlo = min(max(-hb, 0), R), rhi = min(max(a.H - hb, 0), R);
              const int clo = min(max(-wb, 0), S), chi = min(max(Wv - wb, 0), S);
              const uint32_t rm = ((1u << rhi) - 1u) & ~((1u << rlo) - 1u);
              const uint32_t cm = ((1u << chi) - 1u) & ~((1u << clo) - 1u);
              vm[i] = rm | (cm << 8);
            }
            q += RSTEP;
            while (q >= a.Q) {
              q -= a.Q;
              if (++p == a.P) {
                p = 0;
                ++n;
              }
            }
          }
        }
        // swizzled smem destination of (row, part): the XOR term is constant
        // per thread because every row this thread owns has the same row & 7
        const uint32_t dst_thread = uint32_t(row0 * 128 + ((part ^ (row0 & 7)) << 4));
        const int cpt = a.C >> 6;  // 64-channel slices per tap (gather mode)
        int tap = 0, c0 = 0;        // gather-mode k-block -> (tap, channel slice)
        for (int kb = 0; kb < a.kblocks; ++kb, ++it) {
          const uint32_t s = it % STAGES;
          if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
          if (tid == 0) {
            mbar_arrive_expect_tx(&full[s], B_STAGE);
            tma_load_2d(sB + s * B_STAGE, &wmap, &full[s], kb * BK, n0);
          }
          const uint32_t dstA = sA + s * A_STAGE + dst_thread;
          if constexpr (MODE == MODE_STEMG) {
            // this thread's 16 B column of the k-block is pair-tap kb*8+part
            // (taps >= 28 meet zero weights: zero-filled)
            const int tp = kb * 8 + part;
            const int r = tp >> 2, j = tp & 3;
            const long long off = (long long)(r * (a.W >> 1) + j) * 8;
            const uint32_t need = (1u << r) | (1u << (8 + j));
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
              const bool ok = tp < 28 && (vm[i] & need) == need;
              // L1-allocating: neighbouring rows' windows overlap
              cp_async_16_ca(dstA + i * (RSTEP * 128), ok ? rowp[i] + off : a.x, ok);
            }
          } else {
            const int r = tap / a.S, sx = tap - r * a.S;
            const long long off = (long long)(r * a.W + sx) * a.C + c0 + part * 8;
            const uint32_t need = (1u << r) | (1u << (8 + sx));
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
              const bool ok = (vm[i] & need) == need;
              cp_async_16(dstA + i * (RSTEP * 128), ok ? rowp[i] + off : a.x, ok);
            }
            c0 += 64;
            if (c0 == a.C) {
              c0 = 0;
              ++tap;
            }
          }
          (void)cpt;
          // signal the stage issued LAG iterations ago: its copies have
          // landed for this thread; make them visible to the async proxy
          // (tcgen05 reads smem through it), then one arrive per warp.
          cp_async_commit();
          if (it >= LAG) {
            cp_async_wait<int(LAG)>();
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[(it - LAG) % STAGES]);
          }
        }
      }
    }
    if constexpr (gathers(MODE)) {
      // drain: signal the last LAG stages
      cp_async_wait<0>();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const uint32_t first = it >= LAG ? it - LAG : 0;
        for (uint32_t j = first; j < it; ++j) mbar_arrive(&full[j % STAGES]);
      }
    }
    }
  } else if (warp < MMA_WARP) {
    // ============================ epilogue =============================
    const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32)
    // HALVES warps share a lane quarter: warp `half` takes chunks half,
    // half + HALVES, ... of every tile (CHW of them)
    constexpr int HALVES = EPI_W / 4;
    const int half = (warp - 4) >> 2;
    // fused operands: t0 = add / add_mask (pooled) / xc, t1 = out_mask
    constexpr int NOPS = ev_operands(EV);
    constexpr uint32_t SLOT = NOPS * 2048u;
    constexpr uint32_t NSLOTS = NOPS ? EPI_RING_WARP / SLOT : 1;
    static_assert(OPT || !NOPS || NSLOTS >= 2, "operand ring");
    constexpr uint32_t OP1 = OPT ? BN * 256 : 2048;  // second operand, from the first's slot
    const uint32_t ring = sIn + (warp - 4) * EPI_RING_WARP;
    constexpr int CH = BN / 32;         // chunks per tile
    constexpr int CHW = CH / HALVES;    // chunks per tile of this warp
    static_assert(CHW >= 1 && CH % HALVES == 0, "epilogue split");
    const bf16* src0 = static_cast<const bf16*>(
        EV == EV_BN_BWD || EV == EV_GELU_BWD ? a.e.xc : (EV == EV_POOL ? a.e.add_mask : a.e.add));
    const bf16* src1 = static_cast<const bf16*>(a.e.out_mask);
    // stage this warp's chunk number e (tile = first + (e / CHW) * grid,
    // chunk j = half + (e % CHW) * HALVES)
    // with cp.async: 4 x 16 B per lane per operand, 8 full rows per instruction,
    // rows past M zero-filled; one commit group per chunk (possibly empty)
    auto prefetch = [&](uint32_t e) {
      const int tile_ = unit + int(e / CHW) * units;
      if (tile_ < a.tiles) {
        const uint32_t sb = ring + (e % NSLOTS) * SLOT;
        const int pm = tile_m0(tile_) + quarter * 32;
        const int pc = (tile_ % a.n_tiles) * BN + (half + int(e % CHW) * HALVES) * 32;
        // stride-2 add: (n, p, q) of the block's first row, once per chunk
        int q0 = 0, p0 = 0, n0_ = 0;
        if (ev_adds(EV) && a.e.add_stride2) {
          q0 = pm % a.Q;
          const int t = pm / a.Q;
          p0 = t % a.P;
          n0_ = t / a.P;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = i * 8 + (lane >> 2), u = lane & 3;
          const int m = pm + r;
          const bool ok = m < a.M;
          const int64_t go = int64_t(ok ? m : 0) * a.K + pc + u * 8;
          const uint32_t so = r * 64 + ((u ^ ((r >> 1) & 3)) << 4);
          if (ev_adds(EV) && a.e.add_stride2) {
            // the add is the input gradient of a stride-2 1x1 conv, given at
            // its [N][P/2][Q/2] sampling points: zero at odd rows/columns
            int q = q0 + r, pp = p0, n = n0_;
            while (q >= a.Q) {  // a 32-row block wraps an image row at most 32/Q times
              q -= a.Q;
              if (++pp == a.P) {
                pp = 0;
                ++n;
              }
            }
            const bool on = ok && !((pp | q) & 1);
            const int64_t srow = (int64_t(n) * (a.P >> 1) + (pp >> 1)) * (a.Q >> 1) + (q >> 1);
            cp_async_16(sb + so, src0 + (on ? srow : 0) * a.K + pc + u * 8, on);
          } else {
            cp_async_16(sb + so, src0 + go, ok);
          }
          if (NOPS == 2) cp_async_16(sb + OP1 + so, src1 + go, ok);
        }
      }
      cp_async_commit();
    };
    if constexpr (FUSED && !OPT)
      for (uint32_t e = 0; e + 1 < NSLOTS; ++e) prefetch(e);
    // One N tile (K <= BN = 64): every tile of this CTA covers the same columns, so
    // each lane keeps its chunk columns' statistics in registers across the
    // whole persistent loop (Chan merge / sums per chunk) and the quarters are
    // combined once at the end — no per-tile barrier or global round trip.
    // Several N tiles: per-tile cross-quarter combine folded into the CTA row.
    // (only with one chunk per lane per tile: with more, the per-chunk merges
    // cost more than the per-tile barrier they save — measured at BN=256)
    const bool reg_stats = CHW == 1 && a.stats != nullptr && a.n_tiles == 1;
    float4 racc[CHW];
#pragma unroll
    for (int jj = 0; jj < CHW; ++jj) racc[jj] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.stats != nullptr && !reg_stats)
      stats_row_zero(a.stats, a.K, BN, (warp - 4) * 32 + lane, EPI_W * 32);
    uint32_t ec = 0;  // chunks consumed by this warp
    uint32_t lt = 0;
    for (int tile = unit; tile < a.tiles; tile += units, ++lt) {
      // row-tiled stem: tile = one output row of Q pixels (rows >= Q are junk)
      const int m0 = row_tiled(MODE) ? (tile / a.n_tiles) * a.Q : tile_m0(tile);
      const int n0 = (tile % a.n_tiles) * BN;
      const uint32_t acc = lt & 1;
      // EV_ADD_S2: this lane's row -> its shortcut-gradient row (even p and q only)
      int64_t s2row = -1;
      if constexpr (EV == EV_ADD_S2) {
        const int m = m0 + quarter * 32 + lane;
        if (m < a.M) {
          const int q = m % a.Q, t = m / a.Q;
          const int p = t % a.P, n = t / a.P;
          if (!((p | q) & 1)) s2row = (int64_t(n) * (a.P >> 1) + (p >> 1)) * (a.Q >> 1) + (q >> 1);
        }
      }
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t obuf = sIn + (lt % OPT_NB) * OPT_TILE;
      if constexpr (FUSED && OPT)
        mbar_wait(XFORM ? &otrans[lt % OPT_NB] : &ofull[lt % OPT_NB], (lt / OPT_NB) & 1);
      // TMA-store staging: 16 KB over the epilogue warps, NBUF 2 KB buffers each
      constexpr int NBUF = 16384 / EPI_W / 2048;
      const uint32_t stage_base = sOut + (warp - 4) * (NBUF * 2048);
#pragma unroll 1
      for (int j = half; j < CH; j += HALVES, ++ec) {
        // the slot refilled here was consumed (and __syncwarp'ed) last chunk
        if constexpr (FUSED && !OPT) prefetch(ec + NSLOTS - 1);
        float v[32];
        tmem_ld_32x32b_x32(tmem + (uint32_t(quarter * 32) << 16) + acc * ACC_COLS + j * 32, v);
        const int col = n0 + j * 32;
        const uint32_t sb = OPT ? obuf + j * 8192 + quarter * 2048 : ring + (ec % NSLOTS) * SLOT;
        if constexpr (FUSED && !OPT) {
          cp_async_wait<NSLOTS - 1>();  // this chunk's group is the oldest committed
          __syncwarp();
        }
        if constexpr (EV == EV_POOL) {
          // pooled head gradient (read through L1) masked by add_mask, added in fp32
          const int64_t m = int64_t(m0) + quarter * 32 + lane;
          const bf16* pool = static_cast<const bf16*>(a.e.add);
          const float inv = 1.f / float(a.e.pool_hw);
          const int64_t prow = (m < a.M ? m : 0) / a.e.pool_hw;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float g[8], mk[8];
            unpack8f(ldg16(pool + prow * a.K + col + u * 8), g);
            unpack8f(ld_row16(sb, lane, u), mk);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[u * 8 + i] += mk[i] > 0.f ? g[i] * inv : 0.f;
          }
        }
        if constexpr (EV == EV_BIAS) {
          // lane c holds bias[col + c]; broadcast column by column
          const float bl = col + lane < a.K ? __ldg(a.e.beta + col + lane) : 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += __shfl_sync(0xFFFFFFFFu, bl, i);
        }
        if constexpr (EV == EV_GELU_BWD) {
          // d(pre-activation) = d(gelu output) * gelu'(pre-activation), fp32;
          // gelu' already formed (fp16) by the transform warps
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint4 q = ld_row16(sb, lane, u);
            const __half2* hq = reinterpret_cast<const __half2*>(&q);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 g = __half22float2(hq[k]);
              v[u * 8 + 2 * k] *= g.x;
              v[u * 8 + 2 * k + 1] *= g.y;
            }
          }
        }
        if constexpr (row_tiled(MODE)) {
          // junk rows past the output row: zero (they feed the BN statistics)
          if (quarter * 32 + lane >= a.Q) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
        }
        // pack to bf16 (packed epilogue ops on top), stage for the TMA store
        uint4 pk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          pk[u].x = pack_bf16x2(v[u * 8 + 0], v[u * 8 + 1]);
          pk[u].y = pack_bf16x2(v[u * 8 + 2], v[u * 8 + 3]);
          pk[u].z = pack_bf16x2(v[u * 8 + 4], v[u * 8 + 5]);
          pk[u].w = pack_bf16x2(v[u * 8 + 6], v[u * 8 + 7]);
        }
        if constexpr (ev_adds(EV)) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint4 ad = ld_row16(sb, lane, u);
            pk[u].x = add_bf16x2(pk[u].x, ad.x);
            pk[u].y = add_bf16x2(pk[u].y, ad.y);
            pk[u].z = add_bf16x2(pk[u].z, ad.z);
            pk[u].w = add_bf16x2(pk[u].w, ad.w);
          }
        }
        if constexpr (EV == EV_ADD_S2) {
          if (s2row >= 0) {
            const bf16* addp = static_cast<const bf16*>(a.e.add) + s2row * a.K + col;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const uint4 ad = ldg16(addp + u * 8);
              pk[u].x = add_bf16x2(pk[u].x, ad.x);
              pk[u].y = add_bf16x2(pk[u].y, ad.y);
              pk[u].z = add_bf16x2(pk[u].z, ad.z);
              pk[u].w = add_bf16x2(pk[u].w, ad.w);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint4 om = ld_row16(sb, lane, u);
            pk[u].x &= pos_mask2(om.x);
            pk[u].y &= pos_mask2(om.y);
            pk[u].z &= pos_mask2(om.z);
            pk[u].w &= pos_mask2(om.w);
          }
        }
        if constexpr (EV == EV_ADD_OM || EV == EV_POOL || EV == EV_ADD_OM_ST) {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint4 om = ld_row16(sb + OP1, lane, u);
            pk[u].x &= pos_mask2(om.x);
            pk[u].y &= pos_mask2(om.y);
            pk[u].z &= pos_mask2(om.z);
            pk[u].w &= pos_mask2(om.w);
          }
        }
        if constexpr (EV == EV_BN_BWD) {
          // ReLU mask of the forward output relu(bn(xc)) = bf16(max(xc*sc+sh, 0)):
          // positive iff xc*sc+sh > 2^-134 (the bf16 rounding threshold), with
          // k_bn_apply<0>'s exact scale/shift arithmetic
          // lane c computes column c's (scale, shift) into the warp's scratch;
          // every lane then reads them back two columns per 16 B broadcast load
          const uint32_t scsh = sScSh + (warp - 4) * 256;
          {
            const float my_sc = __ldg(a.e.invstd + col + lane) * __ldg(a.e.gamma + col + lane);
            const float my_sh =
                fmaf(-__ldg(a.e.mean + col + lane), my_sc, __ldg(a.e.beta + col + lane));
            asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(scsh + lane * 8), "f"(my_sc),
                         "f"(my_sh)
                         : "memory");
            __syncwarp();
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            float x[8];
            unpack8f(ld_row16(sb, lane, u), x);
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
              float sc0, sh0, sc1, sh1;
              asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(sc0), "=f"(sh0), "=f"(sc1), "=f"(sh1)
                           : "r"(scsh + (u * 8 + i) * 8));
              const uint32_t bits = (fmaf(x[i], sc0, sh0) > 0x1p-134f ? 0xFFFFu : 0u) |
                                    (fmaf(x[i + 1], sc1, sh1) > 0x1p-134f ? 0xFFFF0000u : 0u);
              (&pk[u].x)[i >> 1] &= bits;
            }
          }
        }
        if constexpr (FUSED) __syncwarp();  // every lane has read the slot before it is refilled
        if constexpr (EV == EV_SCATTER) {
          // one parity class of a stride-2 input gradient: output pixel
          // (n, p, q) lands at (2p + a, 2q + b) of the [N][2P][2Q][K] gradient;
          // each lane stores its row's 64 contiguous bytes
          const int m = m0 + quarter * 32 + lane;
          if (m < a.M && col < a.K) {
            const int q = m % a.Q, t = m / a.Q;
            const int p = t % a.P, n = t / a.P;
            bf16* dst = a.y + ((int64_t(n) * (2 * a.P) + 2 * p + (a.e.scatter >> 1)) * (2 * a.Q) +
                               2 * q + (a.e.scatter & 1)) * a.K + col;
#pragma unroll
            for (int u = 0; u < 4; ++u) reinterpret_cast<uint4*>(dst)[u] = pk[u];
          }
          continue;
        }
        const uint32_t buf = stage_base + (ec % NBUF) * 2048;
        // the TMA store that last read this buffer (NBUF chunks ago) is done
        if (lane == 0) bulk_wait_read<NBUF - 1>();
        __syncwarp();
        // row `lane` = 64 B = 4 chunks of 16 B; 64B swizzle: chunk ^= (row>>1)&3
#pragma unroll
        for (int u = 0; u < 4; ++u)
          st_shared_v4(buf + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4), pk[u]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && col < a.K) {
          if constexpr (row_tiled(MODE))
            tma_store_3d(&ymap, buf, col, quarter * 32, tile / a.n_tiles);  // clipped at Q
          else
            tma_store_2d(&ymap, buf, col, m0 + quarter * 32);
          bulk_commit();
        }
        if (a.stats != nullptr) {
          // column `lane` of this 32x32 block, from the staged bf16 values
          // (exactly what is stored); rows past M are zeros.  BN backward:
          // (sum g, sum g*xc), xc from the operand buffer (same layout)
          const float2 cs = column_sums32<ev_cross(EV)>(
              buf, EV == EV_ADD_OM_ST ? sb + 2 * OP1 : sb, 0xFFFFFFFFu, lane);
          const float sum = cs.x, sq = cs.y;
          if (reg_stats) {
            const int nq = min(max((row_tiled(MODE) ? a.Q : min(BM, a.M - m0)) - quarter * 32, 0), 32);
            const int jj = (j - half) / HALVES;
            if (ev_cross(EV) || nq > 0)
              racc[jj] = stats_merge_tile<ev_cross(EV)>(racc[jj], float(nq), sum, sq);
          } else {
            red[quarter * BN + j * 32 + lane] = make_float2(sum, sq);
          }
        }
        if constexpr (ev_cross(EV)) __syncwarp();  // ring slot read by the stats pass
      }
      if (a.stats != nullptr && !reg_stats) {
        // combine the four row quarters -> this tile's column partials, folded
        // into the CTA's row of the statistics table
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_W * 32) : "memory");
        const int et = (warp - 4) * 32 + lane;
        const int n_rows = row_tiled(MODE) ? a.Q : min(BM, a.M - m0);
        for (int c = et; c < BN; c += EPI_W * 32) {
          float S = 0.f, Q = 0.f;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            S += red[qq * BN + c].x;
            Q += red[qq * BN + c].y;
          }
          if (n0 + c < a.K && n_rows > 0)
            stats_fold_tile<ev_cross(EV)>(a.stats, a.K, n0 + c, float(n_rows), S, Q);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(EPI_W * 32) : "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR)
          mbar_arrive_cluster(mapa_shared(smem_u32(&tempty[acc]), 0));  // the leader's
        else
          mbar_arrive(&tempty[acc]);
        if (FUSED && OPT) mbar_arrive(&oempty[lt % OPT_NB]);  // operand tile read
      }
    }
    if (reg_stats) {
      // the quarters' register statistics through the (now idle) output
      // staging buffer as float4 [4][BN], combined in quarter order
      if (lane == 0) bulk_wait<0>();
      __syncwarp();
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_W * 32) : "memory");
      float4* qs = reinterpret_cast<float4*>(smem + STAGES * (A_STAGE + B_STAGE));
      static_assert(4 * BN * sizeof(float4) <= 16384, "staging buffer");
#pragma unroll
      for (int jj = 0; jj < CHW; ++jj) qs[quarter * BN + (half + jj * HALVES) * 32 + lane] = racc[jj];
      asm volatile("bar.sync 1, %0;" ::"n"(EPI_W * 32) : "memory");
      const int et = (warp - 4) * 32 + lane;
      if (et < BN && et < a.K) {
        float4 r = qs[et];
#pragma unroll
        for (int qq = 1; qq < 4; ++qq) {
          const float4 b = qs[qq * BN + et];
          if (ev_cross(EV)) {
            r.x += b.x;
            r.y += b.y;
          } else {
            r = stats_merge_pair(r, b);
          }
        }
        a.stats[size_t(blockIdx.x) * a.K + et] = r;
      }
    }
  } else {
    // ============================ MMA issuer ===========================
    // The whole warp walks the loop (barrier waits, warp-uniform descriptors
    // built by 64-bit adds), one elected lane issues each k-block's MMAs:
    // issuing from lane 0 alone cost a dozen dependent uniform-datapath
    // instructions per MMA, the pacing stage for the N <= 128 tiles.
    constexpr uint32_t idesc = umma_idesc_bf16(PAIR ? 2 * BM : BM, BN) | (BMN ? (1u << 16) : 0u);
    uint32_t it = 0, lt = 0;
    // pair: only the leader issues (its MMAs read both CTAs' smem, write both TMEMs)
    for (int tile = unit; tile < ((PAIR && rank != 0) ? 0 : a.tiles); tile += units, ++lt) {
      const uint32_t acc = lt & 1;
      if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * ACC_COLS;
      if constexpr (MODE == MODE_STEMRAW) {
        if (lt == 0) mbar_wait(bfull, 0);
        const uint32_t s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        // A: K step k of filter row r = 16 B x (2k) into the staged row
        const uint64_t ad0 = umma_desc_noswz(sA + s * A_STAGE + RAW_DATA - 32, 16, 128);
        const uint64_t bd0 = umma_desc_sw128(sB);
        if (elect_one()) {
#pragma unroll
          for (int r = 0; r < 7; ++r)
#pragma unroll
            for (int k = 0; k < 2; ++k)
              umma_bf16(d, ad0 + uint64_t(r * (RAW_ROW >> 4) + k * 2),
                        bd0 + uint64_t((r >> 1) * (B_STAGE >> 4) + (r & 1) * 4 + k * 2), idesc,
                        (r | k) != 0 ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        __syncwarp();
        ++it;
      }
      for (int kb = 0; kb < (MODE == MODE_STEMRAW ? 0 : a.kblocks); ++kb, ++it) {
        const uint32_t s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        fence_proxy_async_smem();
        tc_fence_after();
        const uint64_t ad0 = MODE == MODE_STEM ? umma_desc_noswz(sA + s * A_STAGE, 2048, 128)
                                               : umma_desc_sw128(sA + s * A_STAGE);
        // BMN: K step of 16 rows = 2 KB into the MN-major boxes (8 KB apart along N)
        const uint64_t bd0 = BMN ? umma_desc_mn_sw128(sB + s * B_STAGE, 8192)
                                 : umma_desc_sw128(sB + s * B_STAGE);
        constexpr int BSTEP = BMN ? 128 : 2;
        if (elect_one()) {
          if constexpr (PAIR) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_pair(d, ad0 + uint64_t(k * 2), bd0 + uint64_t(k * BSTEP), idesc,
                             (kb | k) != 0 ? 1u : 0u);
            umma_commit_pair(&empty[s]);
          } else {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16(d, ad0 + uint64_t(MODE == MODE_STEM ? k * 256 : k * 2),
                        bd0 + uint64_t(k * BSTEP), idesc, (kb | k) != 0 ? 1u : 0u);
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
  if (warp >= 4 && warp < MMA_WARP && lane == 0) bulk_wait<0>();  // output visible before exit
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // both CTAs done with the pair's TMEM
  tc_fence_after();
  if (warp == MMA_WARP) {
    if constexpr (PAIR)
      tmem_dealloc_pair(tmem, TMEM_COLS);
    else
      tmem_dealloc(tmem, TMEM_COLS);
  }
}

template <int BN, int STAGES, int EV, bool OPT, bool PAIR = false>
constexpr size_t conv_smem_bytes() {
  constexpr bool FUSED = ev_fused(EV);
  return size_t(STAGES) * (BM * 128 + (PAIR ? BN / 2 : BN) * 128) + 16384 /*epilogue staging*/ +
         (!FUSED ? 0
          : OPT  ? size_t(OPT_NB) * ev_operands(EV) * BN * 256
                 : epi_ring_bytes<BN, STAGES>()) /*epilogue operands*/ + 4 * BN * 8 /*stats scratch*/ +
         (FUSED ? SCSH_BYTES : 0) /*BN scale/shift*/ +
         1024 /*align*/ + 256 /*barriers*/;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor map, inner dimension `cols` (K-major), 64x`box_rows` box,
// 128-byte swizzle (matches the UMMA SW128 K-major smem layout).
bool encode_2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col_fn() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  });
  return fn;
}

// im2col map over the NHWC input: 128 pixels x 64 channels per load; the
// pixel box [-pad, W+pad-(S-1)) x [-pad, H+pad-(R-1)) stepped by the conv
// stride enumerates exactly the P x Q output positions, zero-filled outside
// the image (the padding).
bool encode_im2col(CUtensorMap* m, const void* x, const ConvPlan& cp) {
  auto fn = encode_im2col_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {cuuint64_t(cp.C), cuuint64_t(cp.W), cuuint64_t(cp.H), cuuint64_t(cp.N)};
  cuuint64_t strides[3] = {cuuint64_t(cp.C) * 2, cuuint64_t(cp.W) * cp.C * 2,
                           cuuint64_t(cp.H) * cp.W * cp.C * 2};
  int lower[2] = {-cp.pad, -cp.pad};
  int upper[2] = {cp.pad_end_w - (cp.S - 1), cp.pad_end_h - (cp.R - 1)};
  cuuint32_t estr[4] = {1, cuuint32_t(cp.stride), cuuint32_t(cp.stride), 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower,
            upper, 64, BM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Stem im2col map over the C=4 input viewed as [N][H][W/2][8] (pixel pairs,
// 16 B): traversal stride (w 1, h 2), box corners give exactly P x Q output
// positions (w from -2, h from -3), one 16 B channel box per pixel, no swizzle.
bool encode_stem_im2col(CUtensorMap* m, const void* x, const ConvPlan& cp) {
  auto fn = encode_im2col_fn();
  if (!fn) return false;
  const int W2 = cp.W / 2;
  cuuint64_t dims[4] = {8, cuuint64_t(W2), cuuint64_t(cp.H), cuuint64_t(cp.N)};
  cuuint64_t strides[3] = {16, cuuint64_t(W2) * 16, cuuint64_t(cp.H) * W2 * 16};
  int lower[2] = {-2, -3};
  int upper[2] = {cp.Q - W2 - 2, 2 * cp.P - cp.H - 3};
  cuuint32_t estr[4] = {1, 1, 2, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower,
            upper, 8, BM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Output map: [M rows][K cols] bf16, 32x32 box, 64-byte swizzle (epilogue
// staging layout), out-of-range rows/cols clipped by the TMA unit.
bool encode_out(CUtensorMap* m, void* y, uint64_t cols, uint64_t rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Output of the row-tiled stem: [N*P rows][Q][K], 32x32 boxes clipped at Q.
bool encode_out_rows(CUtensorMap* m, void* y, const ConvPlan& cp) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {cuuint64_t(cp.K), cuuint64_t(cp.Q), cuuint64_t(cp.N) * cp.P};
  cuuint64_t strides[2] = {cuuint64_t(cp.K) * 2, cuuint64_t(cp.Q) * cp.K * 2};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, y, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// operand stages at BN=128 with TMA-loaded epilogue operands: the two tile
// buffers of a two-operand epilogue leave room for two
template <int EV>
constexpr int opt_stages() {
  return ev_operands(EV) == 1 ? 4 : 2;
}

// DELTA_EPI_TMA=0 keeps the fused epilogue operands on the cp.async ring
bool operands_tma() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("DELTA_EPI_TMA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

bool s2_ring() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("DELTA_S2_RING");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// DELTA_CONV_GATHER=1 selects the cp.async im2col gather instead of the TMA
// im2col unit (kept as the reference path for the A operand).
bool gather_forced() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("DELTA_CONV_GATHER");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// Stems whose output rows do not fit a tile (or DELTA_STEM_MODE=tma|gather):
// 128-pixel tiles with the A operand from the TMA im2col unit (one 128 x 16 B
// box per pair-tap) or gathered by the producer threads (cp.async, 16 B pairs).
bool stem_tma() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("DELTA_STEM_MODE");
    v = (e && e[0] == 't') ? 1 : 0;
  }
  return v == 1;
}

// CTA-pair (cta_group::2) tiles: N tile 128 or 256, a reduction of >= 512
// (measured: +5-13 % on the BERT GEMMs at K = 1024-4096; no gain on the
// short-K ResNet 1x1 convs, slower at K = 64), at least one wave of pairs.
// Outputs are bit-identical to the 1-CTA tiles; BN-statistics rows are per
// CTA either way (a pair CTA folds 128-row half tiles).  DELTA_PAIR=0
// disables; DELTA_PAIR_IM2COL=0 keeps the im2col (3x3, strided) convs on
// 1-CTA tiles.
int num_sms();
bool pair_ok(const ConvPlan& cp, bool tma_a) {
  static int v = -1, vi = -1;
  if (v < 0) {
    const char* e = std::getenv("DELTA_PAIR");
    v = (e && e[0] == '0') ? 0 : 1;
    const char* f = std::getenv("DELTA_PAIR_IM2COL");
    vi = (f && f[0] == '0') ? 0 : 1;
  }
  if (!v || (cp.bn != 256 && cp.bn != 128) || cp.C == 4 || cp.kdim < 512) return false;
  if (!tma_a && (!vi || cp.halo || gather_forced())) return false;
  const int64_t M = int64_t(cp.N) * cp.P * cp.Q;
  const int64_t tiles = (M + 255) / 256 * ((cp.K + cp.bn - 1) / cp.bn);
  return tiles >= num_sms() / 2;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int STAGES, int MODE, int EV, bool OPT = false, bool PAIR = false,
          bool BMN = false>
cudaError_t launch(const ConvPlan& cp, const void* x, void* y, float* stats,
                   const ConvEpilogue& epi, cudaStream_t st) {
  auto kern = k_conv_fwd<BN, STAGES, MODE, EV, OPT, PAIR, BMN>;
  constexpr size_t smem = conv_smem_bytes<BN, STAGES, EV, OPT, PAIR>();
  static_assert(smem <= 227 * 1024, "shared memory");
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  ConvArgs a;
  a.x = static_cast<const bf16*>(x);
  a.y = static_cast<bf16*>(y);
  a.N = cp.N; a.H = cp.H; a.W = cp.W; a.C = cp.C; a.K = cp.K; a.R = cp.R; a.S = cp.S;
  a.stride = cp.stride; a.pad = cp.pad; a.P = cp.P; a.Q = cp.Q;
  a.M = cp.N * cp.P * cp.Q;
  a.kblocks = cp.kdim / BK;
  a.taps = cp.R * cp.S;
  a.n_tiles = (cp.K + BN - 1) / BN;
  constexpr int TM = PAIR ? 2 * BM : BM;
  a.tiles = (row_tiled(MODE) ? cp.N * cp.P : (a.M + TM - 1) / TM) * a.n_tiles;
  a.stats = reinterpret_cast<float4*>(stats);
  a.e = epi;
  alignas(64) CUtensorMap amap;
  alignas(64) CUtensorMap ymap;
  if (MODE == MODE_TMA) {
    if (!encode_2d(&amap, x, uint64_t(cp.C), uint64_t(a.M), BM)) return cudaErrorInvalidValue;
  } else if (MODE == MODE_IM2COL) {
    if (!encode_im2col(&amap, x, cp)) return cudaErrorInvalidValue;
  } else if (MODE == MODE_STEM) {
    if (!encode_stem_im2col(&amap, x, cp)) return cudaErrorInvalidValue;
  } else if (MODE == MODE_STEMRAW) {
    if (!stem_raw_rows_map(&amap, x, cp.N, cp.H, cp.W)) return cudaErrorInvalidValue;
  } else {
    amap = *reinterpret_cast<const CUtensorMap*>(cp.wmap);  // unused
  }
  if (row_tiled(MODE) ? !encode_out_rows(&ymap, y, cp)
                           : !encode_out(&ymap, y, uint64_t(cp.K), uint64_t(a.M)))
    return cudaErrorInvalidValue;
  // OPT: the fused epilogue's [M][K] operands as 32-column x 128-row boxes
  alignas(64) CUtensorMap emap0 = ymap, emap1 = ymap, emap2 = ymap;
  if (OPT) {
    const void* op0 = EV == EV_BN_BWD || EV == EV_GELU_BWD ? epi.xc
                       : EV == EV_ADD_S2                  ? epi.out_mask
                       : (EV == EV_POOL ? epi.add_mask : epi.add);
    if (!tma_2d_bf16(&emap0, op0, uint64_t(cp.K), uint64_t(a.M), uint64_t(cp.K), 32, BM,
                     CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
    if (ev_operands(EV) >= 2 &&
        !tma_2d_bf16(&emap1, epi.out_mask, uint64_t(cp.K), uint64_t(a.M), uint64_t(cp.K), 32, BM,
                     CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
    if (ev_operands(EV) == 3 &&
        !tma_2d_bf16(&emap2, epi.xc, uint64_t(cp.K), uint64_t(a.M), uint64_t(cp.K), 32, BM,
                     CU_TENSOR_MAP_SWIZZLE_64B))
      return cudaErrorInvalidValue;
  }
  // statistics come as one partial row per CTA: always one CTA per SM then
  if constexpr (PAIR) {
    // CTA pairs: the weight map's box is this CTA's half of the N tile (BMN:
    // 64 x 64 boxes either way)
    alignas(64) CUtensorMap wmap = *reinterpret_cast<const CUtensorMap*>(cp.wmap);
    if (!BMN && !encode_2d(&wmap, cp.wptr, uint64_t(cp.kdim), uint64_t(cp.K), uint32_t(BN / 2)))
      return cudaErrorInvalidValue;
    const int sms2 = num_sms() & ~1;
    const int grid = (stats != nullptr || 2 * a.tiles > sms2) ? sms2 : 2 * a.tiles;
    if (cudaError_t e_ = launch_cluster(kern, dim3(grid), dim3(kThreads), smem, st, 2u, wmap, amap,
                                        ymap, emap0, emap1, emap2, a))
      return e_;
    return cudaGetLastError();
  }
  const int grid = (stats != nullptr || a.tiles > num_sms()) ? num_sms() : a.tiles;
  if (cudaError_t e_ = launch_k(kern, dim3(grid), dim3(kThreads), smem, st, *reinterpret_cast<const CUtensorMap*>(cp.wmap), amap, ymap, emap0, emap1, emap2, a)) return e_;
  return cudaGetLastError();
}

}  // namespace

int conv_plan_init(ConvPlan* cp, const void* w) {
  cp->wptr = w;
  if (cp->C % 64 != 0 && cp->C != 4) return 1;
  if (cp->K % 8 != 0) return 1;
  // the C=4 stem path is the 7x7/2 pad-3 ResNet stem over an even width
  if (cp->C == 4 && (cp->R != 7 || cp->S != 7 || cp->stride != 2 || cp->pad != 3 || (cp->W & 1)))
    return 1;
  if (cp->pad_end_h < 0) cp->pad_end_h = cp->pad;
  if (cp->pad_end_w < 0) cp->pad_end_w = cp->pad;
  if ((cp->pad_end_h != cp->pad || cp->pad_end_w != cp->pad) && (cp->C == 4 || cp->stride != 1))
    return 1;  // asymmetric padding: stride-1, im2col / 1x1 paths only
  cp->P = (cp->H + cp->pad + cp->pad_end_h - cp->R) / cp->stride + 1;
  cp->Q = (cp->W + cp->pad + cp->pad_end_w - cp->S) / cp->stride + 1;
  cp->kdim = cp->C == 4 ? 256 : cp->R * cp->S * cp->C;
  cp->bn = cp->K <= 64 ? 64 : (cp->K <= 128 ? 128 : 256);
  // 3x3 stride-1, 64 -> 64 channels: stage the input halo once per tile with
  // the 9 weight tiles resident (conv_halo.cu; 124 -> 88 us at 56x56, bs 256).
  // DELTA_CONV_HALO=0 disables it, =1 also routes the other 3x3 stride-1
  // shapes there (experimental).
  // the stem runs row-tiled over raw input rows (MODE_STEMRAW) when an output
  // row fits a tile; DELTA_STEM_MODE=tma / gather select the 128-pixel-tile
  // im2col paths (also the fallback for wider images)
  const char* sm = std::getenv("DELTA_STEM_MODE");
  cp->stem_rows = cp->C == 4 && cp->K <= 64 && cp->Q >= 4 && cp->Q <= 124 && !(sm && sm[0]);
  const char* he = std::getenv("DELTA_CONV_HALO");
  cp->halo = gather_forced() ? 0
             : he             ? (he[0] == '1' && conv_halo_eligible(*cp))
                              : conv_halo_default(*cp);
  if (cp->halo) {
    conv_halo_shape(cp);
    if (cp->halo_rows == 0) cp->halo = 0;
  }
  if (!encode_fn()) return 2;
  if (cp->bmn) {
    // [kdim][K] weights: 64 (N) x 64 (K) boxes, 128-byte swizzle (MN-major)
    if (cp->R != 1 || cp->S != 1 || cp->stride != 1 || cp->pad != 0 || cp->K % 64) return 1;
    return tma_2d_bf16(reinterpret_cast<CUtensorMap*>(cp->wmap), w, uint64_t(cp->K),
                       uint64_t(cp->kdim), uint64_t(cp->K), 64, 64, CU_TENSOR_MAP_SWIZZLE_128B)
               ? 0
               : 3;
  }
  return encode_2d(reinterpret_cast<CUtensorMap*>(cp->wmap), w, uint64_t(cp->kdim),
                   uint64_t(cp->K), uint32_t(cp->bn))
             ? 0
             : 3;
}

int conv_plan_set_tile_n(ConvPlan* cp, int bn, const void* w) {
  if (bn != 64 && bn != 128 && bn != 256) return 1;
  if (cp->C == 4 || cp->K % bn != 0) return 1;
  cp->bn = bn;
  if (cp->bmn) return 0;  // its 64 x 64 boxes do not depend on the tile
  return encode_2d(reinterpret_cast<CUtensorMap*>(cp->wmap), w, uint64_t(cp->kdim),
                   uint64_t(cp->K), uint32_t(cp->bn))
             ? 0
             : 3;
}

cudaError_t conv_forward(const ConvPlan& cp, const void* x, void* y, float* stats,
                         cudaStream_t st, const ConvEpilogue* epi) {
  ConvEpilogue e{};
  if (epi != nullptr) e = *epi;
  if (e.mode != EPI_STORE && (cp.K % 32 != 0 || cp.C == 4)) return cudaErrorInvalidValue;
  if (e.mode == EPI_BN_BWD && (!e.xc || !e.mean || !e.invstd || !e.gamma || !e.beta))
    return cudaErrorInvalidValue;
  const bool stem = cp.C == 4;
  const bool tma_a = !stem && cp.R == 1 && cp.S == 1 && cp.stride == 1 && cp.pad == 0 &&
                     cp.pad_end_h == 0 && cp.pad_end_w == 0;
  const bool use_gather = gather_forced();
  if (cp.bmn) {
    // [kdim][K] weights (MN-major B): the linear layers' input gradients;
    // `stats` (gelu' epilogue): per-CTA column statistics of the output
    // (its column sums are the up-projection's bias gradient)
    if (!tma_a || (stats && e.mode != EPI_GELU_BWD)) return cudaErrorInvalidValue;
    const bool pr = pair_ok(cp, true);
    if (e.mode == EPI_STORE) {
      switch (cp.bn) {
        case 64: return launch<64, 8, MODE_TMA, EV_STORE, false, false, true>(cp, x, y, nullptr, e, st);
        case 128: return launch<128, 6, MODE_TMA, EV_STORE, false, false, true>(cp, x, y, nullptr, e, st);
        default:
          return pr ? launch<256, 6, MODE_TMA, EV_STORE, false, true, true>(cp, x, y, nullptr, e, st)
                    : launch<256, 4, MODE_TMA, EV_STORE, false, false, true>(cp, x, y, nullptr, e, st);
      }
    }
    if (e.mode == EPI_GELU_BWD && e.xc && operands_tma()) {
      if (cp.bn == 64) return launch<64, 4, MODE_TMA, EV_GELU_BWD, true, false, true>(cp, x, y, stats, e, st);
      if (cp.bn == 128)
        return pr ? launch<128, 5, MODE_TMA, EV_GELU_BWD, true, true, true>(cp, x, y, stats, e, st)
                  : launch<128, 4, MODE_TMA, EV_GELU_BWD, true, false, true>(cp, x, y, stats, e, st);
    }
    return cudaErrorInvalidValue;
  }
  if (e.mode == EPI_SCATTER2) {
    if (stats || (cp.K % 32) || stem || unsigned(e.scatter) > 3u) return cudaErrorInvalidValue;
    switch (cp.bn) {
      case 64:
        return tma_a ? launch<64, 8, MODE_TMA, EV_SCATTER>(cp, x, y, nullptr, e, st)
                     : launch<64, 8, MODE_IM2COL, EV_SCATTER>(cp, x, y, nullptr, e, st);
      case 128:
        return tma_a ? launch<128, 6, MODE_TMA, EV_SCATTER>(cp, x, y, nullptr, e, st)
                     : launch<128, 6, MODE_IM2COL, EV_SCATTER>(cp, x, y, nullptr, e, st);
      default:
        return tma_a ? launch<256, 4, MODE_TMA, EV_SCATTER>(cp, x, y, nullptr, e, st)
                     : launch<256, 4, MODE_IM2COL, EV_SCATTER>(cp, x, y, nullptr, e, st);
    }
  }
  const bool pair = pair_ok(cp, tma_a);
  if (e.mode == EPI_BIAS || e.mode == EPI_GELU_BWD) {
    // linear layers (a 1x1 conv over [tokens][features]): bias epilogue, or
    // the MLP input gradient times gelu' of the saved pre-activation
    if (!tma_a || stats) return cudaErrorInvalidValue;
    if (e.mode == EPI_BIAS) {
      if (!e.beta) return cudaErrorInvalidValue;
      switch (cp.bn) {
        case 64: return launch<64, 8, MODE_TMA, EV_BIAS>(cp, x, y, nullptr, e, st);
        case 128: return launch<128, 6, MODE_TMA, EV_BIAS>(cp, x, y, nullptr, e, st);
        default:
          return pair && tma_a ? launch<256, 6, MODE_TMA, EV_BIAS, false, true>(cp, x, y, nullptr, e, st)
                               : launch<256, 4, MODE_TMA, EV_BIAS>(cp, x, y, nullptr, e, st);
      }
    }
    if (!e.xc || !operands_tma()) return cudaErrorInvalidValue;
    if (cp.bn == 64) return launch<64, 4, MODE_TMA, EV_GELU_BWD, true>(cp, x, y, nullptr, e, st);
    if (cp.bn == 128 && pair)
      return launch<128, 5, MODE_TMA, EV_GELU_BWD, true, true>(cp, x, y, nullptr, e, st);
    if (cp.bn == 128)
      return launch<128, opt_stages<EV_GELU_BWD>(), MODE_TMA, EV_GELU_BWD, true>(cp, x, y, nullptr,
                                                                                 e, st);
    return cudaErrorInvalidValue;
  }
  if (cp.halo && e.mode == EPI_STORE && !use_gather) return conv_halo_forward(cp, x, y, stats, st);
  if (e.mode != EPI_STORE) {
    // fused epilogues (backward dgrad): fewer stages pay for the operand ring;
    // N tiles are capped at 128 (delta_conv_set_tile_n)
    int ev;
    if (e.mode == EPI_BN_BWD) {
      ev = EV_BN_BWD;
    } else if (e.pool_hw) {
      if (!e.add || !e.add_mask || !e.out_mask) return cudaErrorInvalidValue;
      ev = EV_POOL;
    } else {
      if (!e.add) return cudaErrorInvalidValue;
      ev = e.out_mask ? EV_ADD_OM : EV_ADD;
      // + the following BN backward's sums (sum y, sum y*xc): three TMA-loaded
      // operands, 64-column N tiles (the operand tiles of two tiles in flight)
      if (e.out_mask && e.xc && stats) {
        if (!tma_a || e.add_stride2 || cp.bn != 64 || !operands_tma()) return cudaErrorInvalidValue;
        return launch<64, 4, MODE_TMA, EV_ADD_OM_ST, true>(cp, x, y, stats, e, st);
      }
    }
    if (cp.bn == 256 && ev == EV_BN_BWD)
      return tma_a ? launch<256, 3, MODE_TMA, EV_BN_BWD>(cp, x, y, stats, e, st)
                   : launch<256, 3, MODE_IM2COL, EV_BN_BWD>(cp, x, y, stats, e, st);
    if (cp.bn != 64 && cp.bn != 128) return cudaErrorInvalidValue;
    if (e.add_stride2 && (ev == EV_POOL || ev == EV_BN_BWD || (cp.P & 1) || (cp.Q & 1)))
      return cudaErrorInvalidValue;
    // stride-2 shortcut gradient + ReLU mask: the mask by TMA tiles, the
    // quarter-density add read straight by the even rows' lanes (the cp.async
    // operand ring ran at ~0.55 of HBM: 322 us for layer2.0 conv1; DELTA_S2_RING=1
    // keeps it)
    if (ev == EV_ADD_OM && e.add_stride2 && !stats && operands_tma() && !s2_ring()) {
      if (cp.bn == 64)
        return tma_a ? launch<64, 4, MODE_TMA, EV_ADD_S2, true>(cp, x, y, nullptr, e, st)
                     : launch<64, 4, MODE_IM2COL, EV_ADD_S2, true>(cp, x, y, nullptr, e, st);
      return tma_a ? launch<128, opt_stages<EV_ADD_S2>(), MODE_TMA, EV_ADD_S2, true>(cp, x, y, nullptr, e, st)
                   : launch<128, opt_stages<EV_ADD_S2>(), MODE_IM2COL, EV_ADD_S2, true>(cp, x, y, nullptr, e, st);
    }
    // Operands by TMA (per-tile boxes into two tile buffers) unless the add is
    // the stride-2 shortcut gradient (cp.async gather from its sampling grid).
    // One-operand epilogues (BN backward, plain add) keep the usual stage
    // count; two-operand ones need two stages at BN=128, which only pays for
    // a short reduction (measured: 281 -> 218 us at 56x56 64->256, floor 205;
    // a 512-deep one loses more to the 2 stages than it gains).
    const bool one_op = ev == EV_BN_BWD || ev == EV_ADD;
    const bool opt = !e.add_stride2 && operands_tma() && (one_op || cp.bn == 64 || cp.kdim <= 256);
#define DELTA_FUSED(EVV)                                                                      \
  case EVV:                                                                                   \
    if (opt && cp.bn == 64)                                                                   \
      return tma_a ? launch<64, 4, MODE_TMA, EVV, true>(cp, x, y, stats, e, st)                \
                   : launch<64, 4, MODE_IM2COL, EVV, true>(cp, x, y, stats, e, st);            \
    if (opt)                                                                                  \
      return tma_a ? launch<128, opt_stages<EVV>(), MODE_TMA, EVV, true>(cp, x, y, stats, e, st) \
                   : launch<128, opt_stages<EVV>(), MODE_IM2COL, EVV, true>(cp, x, y, stats, e, st); \
    if (cp.bn == 64)                                                                          \
      return tma_a ? launch<64, 4, MODE_TMA, EVV>(cp, x, y, stats, e, st)                      \
                   : launch<64, 4, MODE_IM2COL, EVV>(cp, x, y, stats, e, st);                  \
    return tma_a ? launch<128, 3, MODE_TMA, EVV>(cp, x, y, stats, e, st)                       \
                 : launch<128, 3, MODE_IM2COL, EVV>(cp, x, y, stats, e, st);
    switch (ev) {
      DELTA_FUSED(EV_ADD)
      DELTA_FUSED(EV_ADD_OM)
      DELTA_FUSED(EV_POOL)
      DELTA_FUSED(EV_BN_BWD)
      default:
        return cudaErrorInvalidValue;
    }
#undef DELTA_FUSED
  }
  switch (cp.bn) {
    case 64:
      if (stem && cp.stem_rows) return launch<64, 8, MODE_STEMRAW, EV_STORE>(cp, x, y, stats, e, st);
      if (stem && !stem_tma()) return launch<64, 8, MODE_STEMG, EV_STORE>(cp, x, y, stats, e, st);
      return stem ? launch<64, 8, MODE_STEM, EV_STORE>(cp, x, y, stats, e, st)
             : tma_a ? launch<64, 8, MODE_TMA, EV_STORE>(cp, x, y, stats, e, st)
             : use_gather ? launch<64, 8, MODE_GATHER, EV_STORE>(cp, x, y, stats, e, st)
                          : launch<64, 8, MODE_IM2COL, EV_STORE>(cp, x, y, stats, e, st);
    case 128:
      if (pair)
        return tma_a ? launch<128, 8, MODE_TMA, EV_STORE, false, true>(cp, x, y, stats, e, st)
                     : launch<128, 8, MODE_IM2COL, EV_STORE, false, true>(cp, x, y, stats, e, st);
      return stem ? launch<128, 6, MODE_STEM, EV_STORE>(cp, x, y, stats, e, st)
             : tma_a ? launch<128, 6, MODE_TMA, EV_STORE>(cp, x, y, stats, e, st)
             : use_gather ? launch<128, 6, MODE_GATHER, EV_STORE>(cp, x, y, stats, e, st)
                          : launch<128, 6, MODE_IM2COL, EV_STORE>(cp, x, y, stats, e, st);
    default:
      if (pair)
        return tma_a ? launch<256, 6, MODE_TMA, EV_STORE, false, true>(cp, x, y, stats, e, st)
                     : launch<256, 6, MODE_IM2COL, EV_STORE, false, true>(cp, x, y, stats, e, st);
      return stem ? launch<256, 4, MODE_STEM, EV_STORE>(cp, x, y, stats, e, st)
             : tma_a ? launch<256, 4, MODE_TMA, EV_STORE>(cp, x, y, stats, e, st)
             : use_gather ? launch<256, 4, MODE_GATHER, EV_STORE>(cp, x, y, stats, e, st)
                          : launch<256, 4, MODE_IM2COL, EV_STORE>(cp, x, y, stats, e, st);
  }
}

}  // namespace delta_k
