// adamw.cu -- K7: fused per-adapter AdamW with bf16 shadow write-back.
//
// The reference has no optimizer implementation; it only models the state
// (GRAD_COPIES=1, OPT_COPIES=2, pkg/src/lorasweep/costmodel.py:56-58) and carries
// a per-config learning rate (workload.py:135-136,144).  Semantics follow
// torch.optim.AdamW (decoupled weight decay, bias-corrected moments), applied with
// each adapter's own hyper-parameters.
//
// HBM-bound: per parameter it reads p,g,m,v (16 B) and writes p,m,v (12 B) plus
// the bf16 compute shadow (2 B) = 30 B.  Work is described by a chunk table so a
// single launch covers every (layer, target, A|B) region of every adapter; each
// chunk is a run of whole rows of one adapter's [rows][rpad16] block, so the
// shadow address of a 4-element vector is a simple row/column remap into the
// rank-64-padded shadow layout.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/plora.h"
#include "pdl.cuh"

namespace plora {
int set_error(const std::string& msg);
}

namespace {

__global__ void __launch_bounds__(256) adamw_kernel(int64_t n_chunks, const longlong4* __restrict__ chunks,
                                                    float* __restrict__ param,
                                                    const float* __restrict__ grad,
                                                    float* __restrict__ exp_avg,
                                                    float* __restrict__ exp_avg_sq,
                                                    __nv_bfloat16* __restrict__ shadow,
                                                    const float4* __restrict__ hp, float beta1,
                                                    float beta2, float eps, float bc1_all, float bc2_sqrt_all) {
  plora::pdl_wait();
  plora::pdl_trigger();
  for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const longlong4 ch = chunks[c];
    const int64_t p_off = ch.x;
    const int64_t sh_off = ch.y;
    const int32_t n_rows = static_cast<int32_t>(ch.z & 0xffffffffLL);
    const int32_t rpad = static_cast<int32_t>(ch.z >> 32);
    const int32_t adapter = static_cast<int32_t>(ch.w & 0xffffffffLL);
    const int32_t sh_ld = static_cast<int32_t>(ch.w >> 32);
    const float4 h = hp[adapter];
    const float lr = h.x, wd = h.y;
    // bias corrections: one step count for the launch, or the adapter's own (hp.z, on device)
    // (double, as the host path: 1 - beta2^t cancels catastrophically in fp32 at small t)
    const float bc1 = bc1_all > 0.f ? bc1_all : static_cast<float>(1.0 - pow(static_cast<double>(beta1), h.z));
    const float bc2_sqrt = bc1_all > 0.f ? bc2_sqrt_all
                                         : static_cast<float>(sqrt(1.0 - pow(static_cast<double>(beta2), h.z)));
    const float decay = 1.0f - lr * wd;
    const float step_size = lr / bc1;
    const float inv_bc2 = 1.0f / bc2_sqrt;
    const int32_t n4 = n_rows * rpad / 4;
    float4* p4 = reinterpret_cast<float4*>(param + p_off);
    const float4* g4 = reinterpret_cast<const float4*>(grad + p_off);
    float4* m4 = reinterpret_cast<float4*>(exp_avg + p_off);
    float4* v4 = reinterpret_cast<float4*>(exp_avg_sq + p_off);
    const int32_t q_per_row = rpad / 4;
#pragma unroll 2
    for (int32_t i = threadIdx.x; i < n4; i += blockDim.x) {
      float4 p = p4[i];
      const float4 g = g4[i];
      float4 m = m4[i];
      float4 v = v4[i];
      float* pp = &p.x;
      const float* gg = &g.x;
      float* mm = &m.x;
      float* vv = &v.x;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        pp[j] *= decay;
        mm[j] = mm[j] + (1.0f - beta1) * (gg[j] - mm[j]);  // exp_avg.lerp_(grad, 1-beta1)
        vv[j] = vv[j] * beta2 + (1.0f - beta2) * gg[j] * gg[j];
        // fast reciprocal-based divisions (<= 2 ulp): the kernel is HBM-bound only if the
        // per-element math stays short (IEEE divisions cost ~0.2 of the memory time)
        const float denom = sqrtf(vv[j]) * inv_bc2 + eps;
        pp[j] = pp[j] - step_size * __fdividef(mm[j], denom);
      }
      p4[i] = p;
      m4[i] = m;
      v4[i] = v;
      const int32_t row = i / q_per_row;
      const int32_t col = (i - row * q_per_row) * 4;
      __nv_bfloat162 lo = __floats2bfloat162_rn(p.x, p.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(p.z, p.w);
      uint2 packed;
      packed.x = *reinterpret_cast<uint32_t*>(&lo);
      packed.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(shadow + sh_off + static_cast<int64_t>(row) * sh_ld + col) = packed;
    }
  }
}

}  // namespace

extern "C" int plora_adamw(void* stream, int64_t n_chunks, const int64_t* chunks, float* param,
                           const float* grad, float* exp_avg, float* exp_avg_sq, void* shadow,
                           const float* hp, float beta1, float beta2, float eps, int64_t step) {
  if (n_chunks <= 0) return 0;
  if (step < 0) return plora::set_error("adamw: step must be >= 1 (or 0: per-adapter counts in hp[i].z)");
  if (!chunks || !param || !grad || !exp_avg || !exp_avg_sq || !shadow || !hp)
    return plora::set_error("adamw: NULL argument");
  const double bc1 = step > 0 ? 1.0 - pow(static_cast<double>(beta1), static_cast<double>(step)) : -1.0;
  const double bc2 = step > 0 ? 1.0 - pow(static_cast<double>(beta2), static_cast<double>(step)) : 1.0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = static_cast<int64_t>(sms) * 8;
  const int grid = static_cast<int>(n_chunks < want ? n_chunks : want);
  plora::launch_pdl(adamw_kernel, dim3(grid), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      n_chunks, reinterpret_cast<const longlong4*>(chunks), param, grad, exp_avg, exp_avg_sq,
      static_cast<__nv_bfloat16*>(shadow), reinterpret_cast<const float4*>(hp), beta1, beta2, eps,
      static_cast<float>(bc1), static_cast<float>(sqrt(bc2)));
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return plora::set_error(std::string("adamw launch: ") + cudaGetErrorString(e));
  return 0;
}
