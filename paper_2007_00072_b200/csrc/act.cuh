// Activation functions of BAD (paper `brd` / `bdrb`; R6),
// shared by the element-wise BAD kernels (ops_ffn.cu) and the fused GEMM epilogues
// (wgemm.cu).
#pragma once
#include <math.h>

namespace enc {

enum { kActGeluErf = 0, kActGeluTanh = 1, kActRelu = 2 };

// GELU-erf without erff: Abramowitz & Stegun 7.1.26, erf(x) = 1 - poly(t) e^{-x^2},
// t = 1/(1 + p x), |error| <= 1.5e-7 (below fp32 resolution of 1 + erf).  With
// x = |h|/sqrt(2), e^{-x^2} = e^{-h^2/2} is also the Gaussian density's exponential, so
// GELU and GELU' share one MUFU.EX2 and one MUFU.RCP.
__device__ __forceinline__ float ex2_approx(float x) {   // MUFU.EX2, flush-to-zero
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// ea = erf(|h| / sqrt 2) and e = exp(-h^2 / 2) (one MUFU.RCP, one MUFU.EX2, 4 FFMA for the
// polynomial).  Then GELU(h) = h Phi(h) = (h + |h| ea) / 2 and
// GELU'(h) = Phi(h) + h phi(h) = (1 + sign(h) ea) / 2 + h e / sqrt(2 pi).
struct GeluErfParts {
  float ea;
  float e;
};
__device__ __forceinline__ GeluErfParts gelu_erf_parts(float h) {
  const float x = fabsf(h) * 0.70710678118654752f;
  const float t = __fdividef(1.f, fmaf(0.3275911f, x, 1.f));  // MUFU.RCP
  float q = fmaf(1.061405429f, t, -1.453152027f);
  q = fmaf(q, t, 1.421413741f);
  q = fmaf(q, t, -0.284496736f);
  q = fmaf(q, t, 0.254829592f);
  // e^{-h^2/2} = 2^{-h^2 log2(e) / 2} (argument <= 0: result in [0, 1])
  const float e = ex2_approx((-0.72134752044448170f * h) * h);
  GeluErfParts r;
  r.ea = fmaf(-q, t * e, 1.f);   // 1 - t q(t) e^{-x^2}
  r.e = e;
  return r;
}

// GELU scaled by 2 for the erf form (the caller folds the 1/2 into its multiplier)
template <int ACT>
__device__ __forceinline__ float act_f2(float h) {
  if (ACT == kActGeluErf) return fmaf(fabsf(h), gelu_erf_parts(h).ea, h);
  if (ACT == kActGeluTanh) {
    const float u = 0.7978845608028654f * fmaf(0.044715f * h, h * h, h);
    return h * (1.f + tanhf(u));
  }
  return h > 0.f ? 2.f * h : 0.f;
}

template <int ACT>
__device__ __forceinline__ float act_df(float h) {
  if (ACT == kActGeluErf) {
    const GeluErfParts g = gelu_erf_parts(h);
    // Phi(h) + h phi(h)
    return fmaf(h * 0.3989422804014327f, g.e, fmaf(0.5f, copysignf(g.ea, h), 0.5f));
  }
  if (ACT == kActGeluTanh) {
    const float c = 0.7978845608028654f;
    const float t = tanhf(c * fmaf(0.044715f * h, h * h, h));
    return 0.5f * (1.f + t) + 0.5f * h * (1.f - t * t) * c * (1.f + 3.f * 0.044715f * h * h);
  }
  return h > 0.f ? 1.f : 0.f;
}

#define ENC_ACT_DISPATCH(act, ...)                                                \
  do {                                                                            \
    if ((act) == kActGeluErf) { constexpr int ACT = kActGeluErf; __VA_ARGS__; }   \
    else if ((act) == kActGeluTanh) { constexpr int ACT = kActGeluTanh; __VA_ARGS__; } \
    else { constexpr int ACT = kActRelu; __VA_ARGS__; }                           \
  } while (0)

}  // namespace enc
