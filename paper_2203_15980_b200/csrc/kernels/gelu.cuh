// erf GELU and its derivative with one exp and one reciprocal per element
// (Abramowitz & Stegun 7.1.26: |erf error| <= 1.5e-7, below the bf16 output
// rounding by four orders of magnitude), shared by the Gelu node's kernel
// (xformer.cu) and the MLP input-gradient epilogue (conv_fwd.cu EV_GELU_BWD),
// so forward and backward use the same Phi.  Deterministic (MUFU.EX2/RCP are
// fixed functions).
#pragma once

namespace delta_k {

// Phi(x) = 0.5 (1 + erf(x / sqrt 2)) and E = exp(-x^2 / 2)
__device__ __forceinline__ float gelu_cdf(float x, float& E) {
  const float z = fabsf(x) * 0.70710678118654752f;
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.f)));
  float p = fmaf(1.061405429f, t, -1.453152027f);
  p = fmaf(p, t, 1.421413741f);
  p = fmaf(p, t, -0.284496736f);
  p = fmaf(p, t, 0.254829592f);
  p *= t;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(E) : "f"(-z * z * 1.4426950408889634f));
  const float erf_abs = fmaf(-p, E, 1.f);
  const float erf = x < 0.f ? -erf_abs : erf_abs;
  return fmaf(0.5f, erf, 0.5f);
}

__device__ __forceinline__ float gelu_fwd1(float x) {
  float E;
  return x * gelu_cdf(x, E);
}

// d gelu / dx = Phi(x) + x phi(x)
__device__ __forceinline__ float gelu_grad1(float x) {
  float E;
  const float cdf = gelu_cdf(x, E);
  return fmaf(x * 0.3989422804014327f, E, cdf);
}

}  // namespace delta_k
