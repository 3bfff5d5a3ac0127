// swiglu_math.cuh -- the one SwiGLU arithmetic every kernel uses (the gate/up GEMM epilogue,
// swiglu_fwd / swiglu_bwd, the fused SwiGLU-backward + dA kernel), so the activation the
// forward feeds the down projection and the one the backward re-forms are bit-identical.
//   s = sigmoid(g) = 1 / (1 + exp(-g)) (fast reciprocal: MUFU, no IEEE division),  act = (g s) u,
//   du = da g s,  dg = da u s (1 + g (1 - s))
#pragma once

namespace plora {

__device__ __forceinline__ float swiglu_sig(float g) { return __fdividef(1.f, 1.f + __expf(-g)); }

__device__ __forceinline__ float swiglu_act(float g, float u) { return g * swiglu_sig(g) * u; }

__device__ __forceinline__ void swiglu_bwd_elem(float da, float g, float u, float& dg, float& du, float& act) {
  const float s = swiglu_sig(g);
  act = g * s * u;
  du = da * g * s;
  dg = da * u * s * (1.f + g * (1.f - s));
}

}  // namespace plora
