// Host-side TMA tensor-map encoders (driver entry points resolved once).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <mutex>

namespace delta_k {

inline PFN_cuTensorMapEncodeTiled_v12000 tma_tiled_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

inline PFN_cuTensorMapEncodeIm2col_v12000 tma_im2col_fn() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(p);
  });
  return fn;
}

// bf16 [rows][cols] row-major, box {box_cols, box_rows}
inline bool tma_2d_bf16(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows,
                        uint64_t row_stride_elems, uint32_t box_cols, uint32_t box_rows,
                        CUtensorMapSwizzle sw) {
  auto fn = tma_tiled_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC bf16 im2col: `pixels` output positions x `channels` per load, pixel
// box corners (lower/upper, w then h) and traversal strides (w, h).
inline bool tma_im2col_bf16(CUtensorMap* m, const void* x, int C, int W, int H, int N, int lo_w,
                            int lo_h, int up_w, int up_h, int st_w, int st_h, uint32_t channels,
                            uint32_t pixels, CUtensorMapSwizzle sw) {
  auto fn = tma_im2col_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {cuuint64_t(C), cuuint64_t(W), cuuint64_t(H), cuuint64_t(N)};
  cuuint64_t strides[3] = {cuuint64_t(C) * 2, cuuint64_t(W) * C * 2, cuuint64_t(H) * W * C * 2};
  int lower[2] = {lo_w, lo_h};
  int upper[2] = {up_w, up_h};
  cuuint32_t estr[4] = {1, cuuint32_t(st_w), cuuint32_t(st_h), 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, lower,
            upper, channels, pixels, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The C=4 stem input [N][H][W/2 pixel pairs][8] as whole input rows: runs of
// c = 8 x 2^k elements (the longest run of <= 8 pairs dividing W/2), one box =
// one row (W/2*8/c runs), rows outside the image zero-filled, no swizzle.
// Used by the raw-row stem forward and weight-gradient kernels.
inline bool stem_raw_rows_map(CUtensorMap* m, const void* x, int N, int H, int W) {
  auto fn = tma_tiled_fn();
  if (!fn) return false;
  const uint64_t W2 = uint64_t(W / 2);
  uint64_t c = 8;
  while (c < 64 && (W2 * 8) % (2 * c) == 0) c *= 2;
  const uint64_t runs = W2 * 8 / c;
  if (runs > 256) return false;
  cuuint64_t dims[4] = {c, runs, cuuint64_t(H), cuuint64_t(N)};
  cuuint64_t strides[3] = {c * 2, W2 * 16, uint64_t(H) * W2 * 16};
  cuuint32_t box[4] = {cuuint32_t(c), cuuint32_t(runs), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace delta_k
