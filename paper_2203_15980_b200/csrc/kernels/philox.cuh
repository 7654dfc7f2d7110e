// Counter-based dropout masks (Philox4x32-10, Salmon et al. SC'11) so that a
// RECOMPUTED tensor sees exactly the mask its first production drew: the mask
// of element e of dropout site `tag` in training step `step` is a pure
// function of (seed, step, tag, e) — no generator state is consumed, so the
// recompute engine (and the backward pass) replays it bit for bit.
//
// One Philox block (128 bits) serves 16 consecutive elements: byte j of the
// block decides element 16*g + j (keep iff byte >= thr, thr = round(p * 256),
// i.e. the drop probability is quantised to 1/256; scale = 256 / (256 - thr)).
#pragma once
#include <cstdint>

namespace delta_k {

struct DropParams {
  uint32_t thr;   // drop iff byte < thr (0 = no dropout)
  float scale;    // 1 / keep probability
};

inline DropParams drop_params(float p) {
  int thr = int(p * 256.f + 0.5f);
  if (thr < 0) thr = 0;
  if (thr > 255) thr = 255;
  return DropParams{uint32_t(thr), 256.f / float(256 - thr)};
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// The 16 keep-bytes of block g (elements 16g .. 16g+15) of site `tag`:
// rng = {seed, step} on the device (read per launch, so a captured CUDA graph
// draws a fresh mask each step once the optimizer advances `step`).
__device__ __forceinline__ uint4 drop_block(uint64_t seed, uint64_t step, uint32_t tag,
                                            uint64_t g) {
  return philox4x32_10(make_uint4(uint32_t(g), uint32_t(g >> 32), tag, uint32_t(step)),
                       uint32_t(seed), uint32_t(seed >> 32) ^ uint32_t(step >> 32));
}

// keep bits of 4 elements (byte lanes of word w) -> 4-bit mask
__device__ __forceinline__ uint32_t keep4(uint32_t w, uint32_t thr) {
  return uint32_t((w & 0xFFu) >= thr) | (uint32_t(((w >> 8) & 0xFFu) >= thr) << 1) |
         (uint32_t(((w >> 16) & 0xFFu) >= thr) << 2) | (uint32_t((w >> 24) >= thr) << 3);
}
// 16 keep bits of block g
__device__ __forceinline__ uint32_t keep16(uint4 b, uint32_t thr) {
  return keep4(b.x, thr) | (keep4(b.y, thr) << 4) | (keep4(b.z, thr) << 8) |
         (keep4(b.w, thr) << 12);
}

// the same decisions as 16 byte masks (byte i of word w = 0xFF iff element
// 4w + i is kept): SIMD byte compares, no per-element bit extraction
__device__ __forceinline__ uint4 keep_mask_bytes(uint4 b, uint32_t thr) {
  const uint32_t t4 = thr * 0x01010101u;
  return make_uint4(__vcmpgeu4(b.x, t4), __vcmpgeu4(b.y, t4), __vcmpgeu4(b.z, t4),
                    __vcmpgeu4(b.w, t4));
}
// fp32 all-ones / zero mask of byte i of a keep-mask word
__device__ __forceinline__ uint32_t keep_mask_elem(uint32_t kb, int i) {
  return __byte_perm(kb, 0, 0x1111u * uint32_t(i));
}

}  // namespace delta_k
