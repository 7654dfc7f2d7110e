// 3x3 stride-1 convolution with the input HALO staged once per tile (sm_100a).
//
// The im2col TMA path (conv_fwd.cu) re-reads every input pixel 9 times (once
// per tap) from L2; at the narrow ResNet widths (56x56x64) that L2 traffic,
// not the tensor cores, bounds it.  Here an M tile is `rows` whole output rows
// of one image laid out in `slot`-pixel slots (slot = 16/32/64 >= W, rows *
// slot = 128), and its input halo — rows+2 input rows x slot columns starting
// at column -1, zero-filled outside the image by the TMA tiled unit, 64
// channels per load — lands in shared memory as slot-strided 128-byte pixel
// rows (K-major, 128B swizzle).  Tap (r, s) of output pixel i = (i/slot,
// i%slot) reads halo pixel i + r*slot + s: a CONTIGUOUS 128-row window, so
// each tap is an ordinary UMMA on a shifted descriptor (start = window row).
// Input traffic per tile drops from 9 x 128 rows to (rows+2) x slot rows.
//
// Output pixels with i % slot >= W are computed and discarded: the TMA store
// box (4-D [N][P][Q][K]) clips them, and the fused BN-statistics epilogue
// skips them.  Every tile has exactly rows*W valid outputs (rows divides P),
// so the statistics partials have a constant row count.
//
// Warp roles as in conv_fwd.cu: warp 0 thread 0 = TMA producer (A-halo ring +
// weight ring), warps 4-11 = epilogue, warp 12 = TMEM owner + MMA issuer.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels/kernels.hpp"
#include "kernels/launch.hpp"
#include "kernels/sm100_common.cuh"
#include "kernels/stats_cta.cuh"
#include "kernels/tma_host.hpp"

namespace delta_k {

using namespace dsm100;
using bf16 = __nv_bfloat16;

namespace {

// warps 0 producer, 1-3 idle, 4..4+HE-1 epilogue (two per TMEM lane quarter,
// alternating 32-column chunks, as in conv_fwd.cu), then the MMA warp
constexpr int HE = 8;
constexpr int HMMA = 4 + HE;
constexpr int HT = (HMMA + 1) * 32;  // threads
constexpr int BM = 128;

struct HaloArgs {
  int N, P, Q, C, K;
  int slot, rows;     // M tile = rows x slot pixel slots
  int tiles_per_img;  // P / rows
  int m_tiles;        // N * tiles_per_img
  int n_tiles, tiles;
  int kc;             // C / 64 channel blocks
  float4* stats;      // optional: per-CTA (count, mean, M2) rows [grid][K] (stats_cta.cuh)
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// K-major SW128 descriptor at an arbitrary 128-byte row.  The swizzle is a
// function of the ABSOLUTE shared-memory address bits (as the TMA unit wrote
// it), so a window starting mid-atom needs no base offset (measured: setting
// the base-offset field to the start's row phase corrupts the operand).
__device__ __forceinline__ uint64_t desc_sw128_at(uint32_t addr) {
  uint64_t d = 0;
  d |= uint64_t((addr & 0x3FFFF) >> 4);
  d |= uint64_t(1) << 16;          // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;  // SBO: 8-row groups
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// RES: all 9 taps' weights (C = 64, one channel block) stay resident in
// shared memory for the whole persistent loop — the weight tiles are the same
// for every M tile, so re-streaming them per tile was most of the traffic.
template <int BN, int A_STAGES, int B_STAGES, bool RES>
__global__ void __launch_bounds__(HT, 1)
    k_conv_halo(const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap xmap,
                const __grid_constant__ CUtensorMap ymap, const HaloArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr uint32_t A_MAX = 10 * 16 * 128 > 4 * 64 * 128 ? 10 * 16 * 128 : 4 * 64 * 128;  // 32 KB
  constexpr uint32_t B_STAGE = BN * 128;
  const uint32_t sA = smem_u32(smem);
  const uint32_t sB = sA + A_STAGES * A_MAX;
  const uint32_t sOut = sB + B_STAGES * B_STAGE;
  float2* red = reinterpret_cast<float2*>(smem + A_STAGES * A_MAX + B_STAGES * B_STAGE + 16384);
  uint64_t* afull = reinterpret_cast<uint64_t*>(red + 4 * BN);
  uint64_t* aempty = afull + A_STAGES;
  uint64_t* bfull = aempty + A_STAGES;
  uint64_t* bempty = bfull + B_STAGES;
  uint64_t* tfull = bempty + B_STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* bres = tempty + 2;  // resident weights landed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bres + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t a_bytes = uint32_t(a.rows + 2) * a.slot * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < A_STAGES; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int s = 0; s < B_STAGES; ++s) {
      mbar_init(&bfull[s], 1);
      mbar_init(&bempty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], HE);
    }
    mbar_init(bres, 1);
    fence_mbar_init();
    tma_prefetch_desc(&wmap);
    tma_prefetch_desc(&xmap);
    tma_prefetch_desc(&ymap);
  }
  if (warp == HMMA) tmem_alloc(tslot, 2 * BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // prologue done (barriers, TMEM, descriptors): now wait for the predecessor
  pdl_wait();
  pdl_trigger();

  if (warp == 0) {
    // ================================ producer ================================
    if (lane == 0) {
      uint32_t ia = 0, ib = 0;
      if constexpr (RES) {  // one n tile, one channel block: 9 weight tiles, once
        mbar_arrive_expect_tx(bres, 9 * B_STAGE);
        for (int tap = 0; tap < 9; ++tap)
          tma_load_2d(sB + tap * B_STAGE, &wmap, bres, tap * a.C, 0);
      }
      for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x) {
        const int mt = tile / a.n_tiles, n0 = (tile % a.n_tiles) * BN;
        const int n = mt / a.tiles_per_img, p0 = (mt % a.tiles_per_img) * a.rows;
        for (int kc = 0; kc < a.kc; ++kc, ++ia) {
          const uint32_t s = ia % A_STAGES;
          if (ia >= A_STAGES) mbar_wait(&aempty[s], ((ia / A_STAGES) - 1) & 1);
          mbar_arrive_expect_tx(&afull[s], a_bytes);
          tma_load_4d(sA + s * A_MAX, &xmap, &afull[s], kc * 64, -1, p0 - 1, n);
          if constexpr (RES) continue;
          for (int tap = 0; tap < 9; ++tap, ++ib) {
            const uint32_t sb = ib % B_STAGES;
            if (ib >= B_STAGES) mbar_wait(&bempty[sb], ((ib / B_STAGES) - 1) & 1);
            mbar_arrive_expect_tx(&bfull[sb], B_STAGE);
            tma_load_2d(sB + sb * B_STAGE, &wmap, &bfull[sb], tap * a.C + kc * 64, n0);
          }
        }
      }
    }
  } else if (warp < 4) {
    // idle
  } else if (warp < HMMA) {
    // ================================ epilogue ================================
    const int quarter = warp & 3;
    constexpr int HALVES = HE / 4;
    const int half = (warp - 4) >> 2;
    constexpr int NBUF = 16384 / HE / 2048;  // 2 KB TMA-store staging buffers per warp
    uint32_t ec = 0;
    const int qpx = a.slot < 32 ? a.slot : 32;  // pixels per store row
    const int qrows = 32 / qpx;                 // image rows per 32-row chunk
    // one N tile: each lane keeps its columns' statistics in registers across
    // the persistent loop, the quarters are combined once at the end
    const bool reg_stats = a.stats != nullptr && a.n_tiles == 1;
    float4 racc[BN / 32];
#pragma unroll
    for (int j = 0; j < BN / 32; ++j) racc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.stats != nullptr && !reg_stats)
      stats_row_zero(a.stats, a.K, BN, (warp - 4) * 32 + lane, HE * 32);
    uint32_t lt = 0;
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++lt) {
      const int mt = tile / a.n_tiles, n0 = (tile % a.n_tiles) * BN;
      const int n = mt / a.tiles_per_img, p0 = (mt % a.tiles_per_img) * a.rows;
      const int i0 = quarter * 32;  // first tile row of this warp
      const int prow = p0 + i0 / a.slot, pcol = i0 % a.slot;
      const uint32_t acc = lt & 1;
      // this warp's valid rows (pixel column < Q, inside the tile's rows),
      // as a bit mask, once per tile
      uint32_t vmask = 0;
      if (a.stats != nullptr) {
        const bool ok = ((i0 + lane) % a.slot) < a.Q && (i0 + lane) < a.rows * a.slot;
        vmask = __ballot_sync(0xffffffffu, ok);
      }
      mbar_wait(&tfull[acc], (lt >> 1) & 1);
      tc_fence_after();
      const uint32_t stage_base = sOut + (warp - 4) * (NBUF * 2048);
#pragma unroll 1
      for (int j = half; j < BN / 32; j += HALVES, ++ec) {
        float v[32];
        tmem_ld_32x32b_x32(tmem + (uint32_t(quarter * 32) << 16) + acc * BN + j * 32, v);
        const int col = n0 + j * 32;
        const uint32_t buf = stage_base + (ec % NBUF) * 2048;
        if (lane == 0) bulk_wait_read<NBUF - 1>();
        __syncwarp();
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
          // box {32 ch, qpx px, qrows rows, 1}: columns >= Q are clipped
          tma_store_4d(&ymap, buf, col, pcol, prow, n);
          bulk_commit();
        }
        if (a.stats != nullptr) {
          // column `lane`, over this warp's valid rows (pixel column < Q;
          // garbage rows may hold anything)
          const float2 cs = column_sums32<false>(buf, buf, vmask, lane);
          const float sum = cs.x, sq = cs.y;
          if (reg_stats) {
            const float nq = float(__popc(vmask));
            if (nq > 0.f) racc[j] = stats_merge_tile<false>(racc[j], nq, sum, sq);
          } else {
            red[quarter * BN + j * 32 + lane] = make_float2(sum, sq);
          }
        }
      }
      (void)qrows;
      if (a.stats != nullptr && !reg_stats) {
        asm volatile("bar.sync 1, %0;" ::"n"(HE * 32) : "memory");
        const int et = (warp - 4) * 32 + lane;
        const float n_rows = float(a.rows * a.Q);
        for (int c = et; c < BN; c += HE * 32) {
          float S = 0.f, Qs = 0.f;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            S += red[qq * BN + c].x;
            Qs += red[qq * BN + c].y;
          }
          if (n0 + c < a.K) stats_fold_tile<false>(a.stats, a.K, n0 + c, n_rows, S, Qs);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(HE * 32) : "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
    if (reg_stats) {
      // quarters combined through the idle output staging buffer, in order
      if (lane == 0) bulk_wait<0>();
      __syncwarp();
      asm volatile("bar.sync 1, %0;" ::"n"(HE * 32) : "memory");
      float4* qs = reinterpret_cast<float4*>(smem + (sOut - smem_u32(smem)));
      static_assert(4 * BN * sizeof(float4) <= 16384, "staging buffer");
#pragma unroll
      for (int j = half; j < BN / 32; j += HALVES) qs[quarter * BN + j * 32 + lane] = racc[j];
      asm volatile("bar.sync 1, %0;" ::"n"(HE * 32) : "memory");
      for (int c = (warp - 4) * 32 + lane; c < BN && c < a.K; c += HE * 32) {
        float4 r = qs[c];
#pragma unroll
        for (int qq = 1; qq < 4; ++qq) r = stats_merge_pair(r, qs[qq * BN + c]);
        a.stats[size_t(blockIdx.x) * a.K + c] = r;
      }
    }
  } else {
    // ============================== MMA issuer ===============================
    // whole warp walks the loop (uniform 64-bit descriptor adds), one elected
    // lane issues: single-lane issue cost ~12 dependent instructions per MMA
    constexpr uint32_t idesc = umma_idesc_bf16(BM, BN);
    uint32_t ia = 0, ib = 0, lt = 0;
    if constexpr (RES) mbar_wait(bres, 0);
    for (int tile = blockIdx.x; tile < a.tiles; tile += gridDim.x, ++lt) {
      const uint32_t acc = lt & 1;
      if (lt >= 2) mbar_wait(&tempty[acc], ((lt >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * BN;
      for (int kc = 0; kc < a.kc; ++kc, ++ia) {
        const uint32_t s = ia % A_STAGES;
        mbar_wait(&afull[s], (ia / A_STAGES) & 1);
        tc_fence_after();
        const uint64_t ad0 = desc_sw128_at(sA + s * A_MAX);
        for (int tap = 0; tap < 9; ++tap) {
          uint32_t bst;
          if constexpr (RES) {
            bst = sB + tap * B_STAGE;
          } else {
            const uint32_t sb = ib % B_STAGES;
            mbar_wait(&bfull[sb], (ib / B_STAGES) & 1);
            tc_fence_after();
            bst = sB + sb * B_STAGE;
          }
          const int r = tap / 3, sx = tap - r * 3;
          // window of this tap: (r * slot + sx) rows of 128 B into the halo
          const uint64_t aw = ad0 + uint64_t((r * a.slot + sx) * 8);
          const uint64_t bw = umma_desc_sw128(bst);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_bf16(d, aw + uint64_t(k * 2), bw + uint64_t(k * 2), idesc,
                        (kc | tap | k) != 0 ? 1u : 0u);
            if constexpr (!RES) umma_commit(&bempty[ib % B_STAGES]);
          }
          __syncwarp();
          if constexpr (!RES) ++ib;
        }
        if (elect_one()) umma_commit(&aempty[s]);
        __syncwarp();
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
    }
  }
  if (warp >= 4 && warp < HMMA && lane == 0) bulk_wait<0>();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == HMMA) tmem_dealloc(tmem, 2 * BN);
}

template <int BN, int A_STAGES, int B_STAGES, bool RES>
constexpr size_t halo_smem() {
  return size_t(A_STAGES) * 32768 + size_t(B_STAGES) * BN * 128 + 16384 + 4 * BN * 8 + 1024 + 512;
}

template <int BN, int A_STAGES, int B_STAGES, bool RES = false>
cudaError_t halo_launch(const ConvPlan& cp, const void* x, void* y, float* stats,
                        cudaStream_t st) {
  auto kern = k_conv_halo<BN, A_STAGES, B_STAGES, RES>;
  constexpr size_t smem = halo_smem<BN, A_STAGES, B_STAGES, RES>();
  static_assert(smem <= 227 * 1024, "shared memory");
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    attr = true;
  }
  HaloArgs a{};
  a.N = cp.N; a.P = cp.P; a.Q = cp.Q; a.C = cp.C; a.K = cp.K;
  a.slot = cp.halo_slot;
  a.rows = cp.halo_rows;
  a.tiles_per_img = cp.P / cp.halo_rows;
  a.m_tiles = cp.N * a.tiles_per_img;
  a.n_tiles = (cp.K + BN - 1) / BN;
  a.tiles = a.m_tiles * a.n_tiles;
  a.kc = cp.C / 64;
  a.stats = reinterpret_cast<float4*>(stats);
  // input: 4-D [N][H][W][C], box {64 ch, slot px, rows+2 rows, 1}, 128B swizzle
  alignas(64) CUtensorMap xmap, ymap;
  {
    auto fn = tma_tiled_fn();
    if (!fn) return cudaErrorInvalidValue;
    cuuint64_t dims[4] = {cuuint64_t(cp.C), cuuint64_t(cp.W), cuuint64_t(cp.H), cuuint64_t(cp.N)};
    cuuint64_t strides[3] = {cuuint64_t(cp.C) * 2, cuuint64_t(cp.W) * cp.C * 2,
                             cuuint64_t(cp.H) * cp.W * cp.C * 2};
    cuuint32_t box[4] = {64, cuuint32_t(a.slot), cuuint32_t(a.rows + 2), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    if (fn(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box,
           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
    // output: 4-D [N][P][Q][K], box {32 ch, qpx px, qrows rows, 1}, 64B swizzle
    const int qpx = a.slot < 32 ? a.slot : 32;
    cuuint64_t odims[4] = {cuuint64_t(cp.K), cuuint64_t(cp.Q), cuuint64_t(cp.P), cuuint64_t(cp.N)};
    cuuint64_t ostr[3] = {cuuint64_t(cp.K) * 2, cuuint64_t(cp.Q) * cp.K * 2,
                          cuuint64_t(cp.P) * cp.Q * cp.K * 2};
    cuuint32_t obox[4] = {32, cuuint32_t(qpx), cuuint32_t(32 / qpx), 1};
    if (fn(&ymap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, y, odims, ostr, obox, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (stats != nullptr || a.tiles > sms) ? sms : a.tiles;
  if (cudaError_t e_ = launch_k(kern, dim3(grid), dim3(HT), smem, st, *reinterpret_cast<const CUtensorMap*>(cp.wmap), xmap, ymap, a)) return e_;
  return cudaGetLastError();
}

}  // namespace

// Dispatched only with resident weights (C = K = 64: the ResNet layer-1 3x3,
// 124 -> 88 us at bs 256).  The streamed-weight variant (wider layers) is kept
// for experiments behind DELTA_CONV_HALO=1 only: it is slower than the im2col
// path there and fails the W=14, K=256 parity case.
bool conv_halo_eligible(const ConvPlan& cp) {
  if (!(cp.R == 3 && cp.S == 3 && cp.stride == 1 && cp.pad == 1 && cp.C % 64 == 0)) return false;
  if (cp.W > 64 || cp.P != cp.H || cp.Q != cp.W) return false;
  return true;
}

bool conv_halo_default(const ConvPlan& cp) {
  return conv_halo_eligible(cp) && cp.C == 64 && cp.K == 64;
}

// slot = smallest of 16/32/64 holding a padded row; rows = the largest divisor
// of P with rows * slot <= 128 and (rows + 2) * slot * 128 B <= 32 KB
void conv_halo_shape(ConvPlan* cp) {
  int slot = cp->W + 2 <= 16 ? 16 : (cp->W + 2 <= 32 ? 32 : 64);
  // the window of tap s reads halo columns q + s (q < W, s <= 2): slot >= W + 2
  int rows = 0;
  for (int r = 128 / slot; r >= 1; --r)
    if (cp->P % r == 0 && (r + 2) * slot * 128 <= 32768) {
      rows = r;
      break;
    }
  cp->halo_slot = slot;
  cp->halo_rows = rows;
}

cudaError_t conv_halo_forward(const ConvPlan& cp, const void* x, void* y, float* stats,
                              cudaStream_t st) {
  if (cp.C == 64 && cp.K == 64) return halo_launch<64, 4, 9, true>(cp, x, y, stats, st);
  switch (cp.bn) {
    case 64:
      return halo_launch<64, 2, 8>(cp, x, y, stats, st);
    case 128:
      return halo_launch<128, 2, 6>(cp, x, y, stats, st);
    default:
      return halo_launch<256, 2, 4>(cp, x, y, stats, st);
  }
}

}  // namespace delta_k
