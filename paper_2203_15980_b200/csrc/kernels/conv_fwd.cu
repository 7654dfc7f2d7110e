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
//   warps 0-3 : producers.  MODE_GATHER / MODE_STEM: im2col gather of A with
//               cp.async (zero-fill implements the padding); MODE_TMA (1x1,
//               stride 1): A is a plain [M, C] matrix loaded by TMA.  Thread 0
//               issues the TMA of the weight tile B.
//   warps 4-7 : epilogue — TMEM -> registers -> bf16 -> HBM, one TMEM lane
//               quarter each.
//   warp 8    : TMEM allocation + single-thread tcgen05.mma issue.
// Two TMEM accumulators: the epilogue of tile i drains one while the MMAs of
// tile i+1 fill the other.  smem stages ring with full/empty mbarriers;
// tcgen05.commit releases a stage the moment the tensor core has consumed it.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "kernels/kernels.hpp"
#include "kernels/sm100_common.cuh"

namespace delta_k {

using namespace dsm100;
using bf16 = __nv_bfloat16;

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kThreads = 288;
constexpr int MODE_GATHER = 0, MODE_STEM = 1, MODE_TMA = 2, MODE_IM2COL = 3;


struct ConvArgs {
  const bf16* x;
  bf16* y;
  int N, H, W, C, K, R, S, stride, pad, P, Q;
  int M;        // N*P*Q
  int kblocks;  // reduction length / 64
  int taps;     // R*S
  int n_tiles;  // ceil(K / BN)
  int tiles;    // m_tiles * n_tiles
  float2* stats;  // optional: per (m_tile, channel) (mean, M2) of the bf16 outputs
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

template <int BN, int STAGES, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_fwd(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap amap,
               const __grid_constant__ CUtensorMap ymap, const ConvArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  // producer signalling lag: a thread keeps LAG+1 stages of gathers in flight
  constexpr uint32_t LAG = STAGES - 2;
  constexpr uint32_t A_STAGE = BM * 128;
  constexpr uint32_t B_STAGE = BN * 128;
  constexpr uint32_t ACC_COLS = BN;
  constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  const uint32_t sA = smem_u32(smem);
  const uint32_t sB = sA + STAGES * A_STAGE;
  // epilogue staging: 4 warps x 2 buffers x (32 rows x 64 B), 64B-swizzled
  const uint32_t sOut = sA + STAGES * (A_STAGE + B_STAGE);
  // BN-statistics scratch: per quarter-warp column (sum, sumsq), [4][BN] float2
  float2* red = reinterpret_cast<float2*>(smem + STAGES * (A_STAGE + B_STAGE) + 16384);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (A_STAGE + B_STAGE) + 16384 +
                                               4 * BN * sizeof(float2));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], (MODE == MODE_TMA || MODE == MODE_IM2COL) ? 1 : 4 + 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
    tma_prefetch_desc(&wmap);
    if (MODE == MODE_TMA || MODE == MODE_IM2COL) tma_prefetch_desc(&amap);
    tma_prefetch_desc(&ymap);
  }
  if (warp == 8) tmem_alloc(tslot, TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp < 4) {
    // ============================ producers ============================
    const int tid = threadIdx.x;
    uint32_t it = 0;  // global k-iteration counter (stage ring position)
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
      const int m0 = (tile / a.n_tiles) * BM;
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
            mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
            tma_load_im2col_4d(sA + s * A_STAGE, &amap, &full[s], c0, wb, hb, n, uint16_t(sx),
                               uint16_t(r));
            tma_load_2d(sB + s * B_STAGE, &wmap, &full[s], kb * BK, n0);
            c0 += 64;
            if (c0 == a.C) {
              c0 = 0;
              ++tap;
            }
          }
        }
      } else if constexpr (MODE == MODE_TMA) {
        if (tid == 0) {
          for (int kb = 0; kb < a.kblocks; ++kb, ++it) {
            const uint32_t s = it % STAGES;
            if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], A_STAGE + B_STAGE);
            tma_load_2d(sA + s * A_STAGE, &amap, &full[s], kb * BK, m0);
            tma_load_2d(sB + s * B_STAGE, &wmap, &full[s], kb * BK, n0);
          }
        }
      } else {
        constexpr int ROWS = MODE == MODE_GATHER ? 8 : 16;
        constexpr int RSTEP = MODE == MODE_GATHER ? 16 : 8;
        const int part = MODE == MODE_GATHER ? (tid & 7) : (tid & 15);
        const int row0 = MODE == MODE_GATHER ? (tid >> 3) : (tid >> 4);
        // Per tile, once: each row's input base pointer (top-left tap, may
        // point into the padding) and a validity mask: bits [0,R) say which
        // filter rows land inside the image, bits [8,8+S) which columns.
        // Per k-block the only address math left is one scalar tap offset.
        const bf16* rowp[ROWS];
        uint32_t vm[ROWS];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
          const int m = m0 + row0 + RSTEP * i;
          vm[i] = 0;
          rowp[i] = a.x;
          if (m < a.M) {
            const int q = m % a.Q;
            const int t = m / a.Q;
            const int n = t / a.P;
            const int hb = (t - n * a.P) * a.stride - a.pad;
            const int wb = q * a.stride - a.pad;
            rowp[i] = a.x + (((long long)n * a.H + hb) * a.W + wb) * (long long)a.C;
            uint32_t rm = 0, cm = 0;
            for (int r = 0; r < a.R; ++r) rm |= uint32_t((unsigned)(hb + r) < (unsigned)a.H) << r;
            for (int c = 0; c < a.S; ++c) cm |= uint32_t((unsigned)(wb + c) < (unsigned)a.W) << c;
            vm[i] = rm | (cm << 8);
          }
        }
        // swizzled smem destination of (row, part): the XOR term is constant
        // per thread because every row this thread owns has the same row & 7
        const uint32_t dst_thread = MODE == MODE_GATHER
                                        ? uint32_t(row0 * 128 + ((part ^ (row0 & 7)) << 4))
                                        : uint32_t(row0 * 128 + (((part >> 1) ^ (row0 & 7)) << 4) +
                                                   (part & 1) * 8);
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
          if constexpr (MODE == MODE_GATHER) {
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
          } else {
            const int t = kb * 16 + part;
            const int r = t / a.S, sx = t - r * a.S;
            const uint32_t need = t < a.taps ? (1u << r) | (1u << (8 + sx)) : 0xFFFFFFFFu;
            const long long off = (long long)(r * a.W + sx) * 4;
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
              const bool ok = (vm[i] & need) == need;
              cp_async_8(dstA + i * (RSTEP * 128), ok ? rowp[i] + off : a.x, ok);
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
    if constexpr (MODE == MODE_GATHER || MODE == MODE_STEM) {
      // drain: signal the last LAG stages
      cp_async_wait<0>();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const uint32_t first = it >= LAG ? it - LAG : 0;
        for (uint32_t j = first; j < it; ++j) mbar_arrive(&full[j % STAGES]);
      }
    }
  } else if (warp < 8) {
    // ============================ epilogue =============================
    const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32)
    uint32_t lt = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++lt) {
      const int m0 = (tile / a.n_tiles) * BM;
      const int n0 = (tile % a.n_tiles) * BN;
      const uint32_t acc = lt & 1;
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t stage_base = sOut + quarter * 4096;
#pragma unroll 1
      for (int j = 0; j < BN / 32; ++j) {
        float v[32];
        tmem_ld_32x32b_x32(tmem + (uint32_t(quarter * 32) << 16) + acc * ACC_COLS + j * 32, v);
        const int col = n0 + j * 32;
        const uint32_t buf = stage_base + (j & 1) * 2048;
        // the TMA store that last read this buffer (two chunks ago) is done
        if (lane == 0) bulk_wait_read<1>();
        __syncwarp();
        // row `lane` = 64 B = 4 chunks of 16 B; 64B swizzle: chunk ^= (row>>1)&3
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint4 pk;
          pk.x = pack_bf16x2(v[u * 8 + 0], v[u * 8 + 1]);
          pk.y = pack_bf16x2(v[u * 8 + 2], v[u * 8 + 3]);
          pk.z = pack_bf16x2(v[u * 8 + 4], v[u * 8 + 5]);
          pk.w = pack_bf16x2(v[u * 8 + 6], v[u * 8 + 7]);
          st_shared_v4(buf + lane * 64 + ((u ^ ((lane >> 1) & 3)) << 4), pk);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && col < a.K) {
          tma_store_2d(&ymap, buf, col, m0 + quarter * 32);
          bulk_commit();
        }
        if (a.stats != nullptr) {
          // column `lane` of this 32x32 block, from the staged bf16 values
          // (exactly what BN will read back); rows past M are zeros.
          const uint32_t cbyte = (uint32_t(lane) & 7u) * 2u;
          const uint32_t c16 = uint32_t(lane) >> 3;
          float sum = 0.f, sq = 0.f;
#pragma unroll 8
          for (int rr = 0; rr < 32; ++rr) {
            uint16_t h;
            asm volatile("ld.shared.u16 %0, [%1];"
                         : "=h"(h)
                         : "r"(buf + rr * 64 + ((c16 ^ ((rr >> 1) & 3)) << 4) + cbyte));
            const float f = __bfloat162float(__ushort_as_bfloat16(h));
            sum += f;
            sq = fmaf(f, f, sq);
          }
          red[quarter * BN + j * 32 + lane] = make_float2(sum, sq);
        }
      }
      if (a.stats != nullptr) {
        // combine the four row quarters -> one (mean, M2) per channel per tile
        asm volatile("bar.sync 1, 128;" ::: "memory");
        const int et = (warp - 4) * 32 + lane;
        const int n_rows = min(BM, a.M - m0);
        for (int c = et; c < BN; c += 128) {
          float S = 0.f, Q = 0.f;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            S += red[qq * BN + c].x;
            Q += red[qq * BN + c].y;
          }
          const float mu = S / float(n_rows);
          if (n0 + c < a.K)
            a.stats[size_t(m0 / BM) * a.K + n0 + c] = make_float2(mu, fmaxf(Q - S * mu, 0.f));
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  } else {
    // ============================ MMA issuer ===========================
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
      uint32_t it = 0, lt = 0;
      for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++lt) {
        const uint32_t acc = lt & 1;
        if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * ACC_COLS;
        for (int kb = 0; kb < a.kblocks; ++kb, ++it) {
          const uint32_t s = it % STAGES;
          mbar_wait(&full[s], (it / STAGES) & 1);
          fence_proxy_async_smem();
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = umma_desc_sw128(sA + s * A_STAGE + k * 32);
            const uint64_t bd = umma_desc_sw128(sB + s * B_STAGE + k * 32);
            umma_bf16(d, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  }
  if (warp >= 4 && warp < 8 && lane == 0) bulk_wait<0>();  // output visible before exit
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 8) tmem_dealloc(tmem, TMEM_COLS);
}

template <int BN, int STAGES>
constexpr size_t conv_smem_bytes() {
  return size_t(STAGES) * (BM * 128 + BN * 128) + 16384 /*epilogue staging*/ +
         4 * BN * 8 /*stats scratch*/ + 1024 /*align*/ + 256 /*barriers*/;
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
  int upper[2] = {cp.pad - (cp.S - 1), cp.pad - (cp.R - 1)};
  cuuint32_t estr[4] = {1, cuuint32_t(cp.stride), cuuint32_t(cp.stride), 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower,
            upper, 64, BM, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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

template <int BN, int STAGES, int MODE>
cudaError_t launch(const ConvPlan& cp, const void* x, void* y, float* stats, cudaStream_t st) {
  auto kern = k_conv_fwd<BN, STAGES, MODE>;
  constexpr size_t smem = conv_smem_bytes<BN, STAGES>();
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
  a.tiles = ((a.M + BM - 1) / BM) * a.n_tiles;
  a.stats = reinterpret_cast<float2*>(stats);
  alignas(64) CUtensorMap amap;
  alignas(64) CUtensorMap ymap;
  if (MODE == MODE_TMA) {
    if (!encode_2d(&amap, x, uint64_t(cp.C), uint64_t(a.M), BM)) return cudaErrorInvalidValue;
  } else if (MODE == MODE_IM2COL) {
    if (!encode_im2col(&amap, x, cp)) return cudaErrorInvalidValue;
  } else {
    amap = *reinterpret_cast<const CUtensorMap*>(cp.wmap);  // unused
  }
  if (!encode_out(&ymap, y, uint64_t(cp.K), uint64_t(a.M))) return cudaErrorInvalidValue;
  const int grid = a.tiles < num_sms() ? a.tiles : num_sms();
  kern<<<grid, kThreads, smem, st>>>(*reinterpret_cast<const CUtensorMap*>(cp.wmap), amap, ymap,
                                     a);
  return cudaGetLastError();
}

}  // namespace

int conv_plan_init(ConvPlan* cp, const void* w) {
  if (cp->C % 64 != 0 && cp->C != 4) return 1;
  if (cp->K % 8 != 0) return 1;
  cp->P = (cp->H + 2 * cp->pad - cp->R) / cp->stride + 1;
  cp->Q = (cp->W + 2 * cp->pad - cp->S) / cp->stride + 1;
  cp->kdim = cp->C == 4 ? ((cp->R * cp->S * 4 + 63) / 64) * 64 : cp->R * cp->S * cp->C;
  cp->bn = cp->K <= 64 ? 64 : (cp->K <= 128 ? 128 : 256);
  if (!encode_fn()) return 2;
  return encode_2d(reinterpret_cast<CUtensorMap*>(cp->wmap), w, uint64_t(cp->kdim),
                   uint64_t(cp->K), uint32_t(cp->bn))
             ? 0
             : 3;
}

cudaError_t conv_forward(const ConvPlan& cp, const void* x, void* y, float* stats,
                         cudaStream_t st) {
  const bool stem = cp.C == 4;
  const bool tma_a = !stem && cp.R == 1 && cp.S == 1 && cp.stride == 1 && cp.pad == 0;
  const bool use_gather = gather_forced();
  switch (cp.bn) {
    case 64:
      return stem ? launch<64, 8, MODE_STEM>(cp, x, y, stats, st)
             : tma_a ? launch<64, 8, MODE_TMA>(cp, x, y, stats, st)
             : use_gather ? launch<64, 8, MODE_GATHER>(cp, x, y, stats, st)
                          : launch<64, 8, MODE_IM2COL>(cp, x, y, stats, st);
    case 128:
      return stem ? launch<128, 6, MODE_STEM>(cp, x, y, stats, st)
             : tma_a ? launch<128, 6, MODE_TMA>(cp, x, y, stats, st)
             : use_gather ? launch<128, 6, MODE_GATHER>(cp, x, y, stats, st)
                          : launch<128, 6, MODE_IM2COL>(cp, x, y, stats, st);
    default:
      return stem ? launch<256, 4, MODE_STEM>(cp, x, y, stats, st)
             : tma_a ? launch<256, 4, MODE_TMA>(cp, x, y, stats, st)
             : use_gather ? launch<256, 4, MODE_GATHER>(cp, x, y, stats, st)
                          : launch<256, 4, MODE_IM2COL>(cp, x, y, stats, st);
  }
}

}  // namespace delta_k
