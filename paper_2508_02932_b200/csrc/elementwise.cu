// elementwise.cu -- fused HBM-bound kernels around the packed-LoRA GEMMs:
// RMSNorm fwd/recompute/bwd, SwiGLU fwd/bwd, RoPE (with layout change) and the
// chunked cross-entropy forward+backward.  Each reads and writes every element
// once with 16-byte vector accesses and fp32 math (bf16 storage).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/plora.h"
#include "pdl.cuh"
#include "swiglu_math.cuh"

namespace plora {
int set_error(const std::string& msg);
}

namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ void load8(const bf16* p, float (&f)[8]) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void store8(bf16* p, const float (&f)[8]) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  *reinterpret_cast<uint4*>(p) = v;
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) s += red[i];
  return s;
}

// ---------------------------------------------------------------- RMSNorm
// y = x * rstd * w, rstd = rsqrt(mean(x^2) + eps).  One CTA per row; the row is
// held in registers (d <= 8 * 256 * kMaxV).  mode 0: compute rstd; 1: use given rstd.
constexpr int kNormThreads = 256;
constexpr int kMaxV = 4;  // up to 8192 columns

__global__ void __launch_bounds__(kNormThreads) rmsnorm_fwd_kernel(const bf16* __restrict__ x,
                                                                   const bf16* __restrict__ w,
                                                                   bf16* __restrict__ y,
                                                                   float* __restrict__ rstd, int d,
                                                                   float eps, int use_given) {
  plora::pdl_wait();
  plora::pdl_trigger();
  __shared__ float red[kNormThreads / 32];
  const int64_t row = blockIdx.x;
  const bf16* xr = x + row * d;
  float v[kMaxV][8];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kMaxV; ++j) {
    const int c = (j * kNormThreads + threadIdx.x) * 8;
    if (c < d) {
      load8(xr + c, v[j]);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += v[j][e] * v[j][e];
    }
  }
  float r;
  if (use_given) {
    r = rstd[row];
  } else {
    ss = block_sum<kNormThreads>(ss, red);
    r = rsqrtf(ss / d + eps);
    if (threadIdx.x == 0) rstd[row] = r;
  }
#pragma unroll
  for (int j = 0; j < kMaxV; ++j) {
    const int c = (j * kNormThreads + threadIdx.x) * 8;
    if (c < d) {
      float wf[8], o[8];
      load8(w + c, wf);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = v[j][e] * r * wf[e];
      store8(y + row * d + c, o);
    }
  }
}

// Fused residual add + RMSNorm: s = a + b (written to sum), y = s * rstd * w.
__global__ void __launch_bounds__(kNormThreads) add_rmsnorm_kernel(const bf16* __restrict__ a,
                                                                   const bf16* __restrict__ b,
                                                                   const bf16* __restrict__ w,
                                                                   bf16* __restrict__ sum, bf16* __restrict__ y,
                                                                   float* __restrict__ rstd, int d, float eps) {
  plora::pdl_wait();
  plora::pdl_trigger();
  __shared__ float red[kNormThreads / 32];
  const int64_t row = blockIdx.x;
  float v[kMaxV][8];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kMaxV; ++j) {
    const int c = (j * kNormThreads + threadIdx.x) * 8;
    if (c < d) {
      float bf[8];
      load8(a + row * d + c, v[j]);
      load8(b + row * d + c, bf);
#pragma unroll
      for (int e = 0; e < 8; ++e)   // normalise the bf16-rounded sum (what the backward sees)
        v[j][e] = __bfloat162float(__float2bfloat16_rn(v[j][e] + bf[e]));
      store8(sum + row * d + c, v[j]);
#pragma unroll
      for (int e = 0; e < 8; ++e) ss += v[j][e] * v[j][e];
    }
  }
  ss = block_sum<kNormThreads>(ss, red);
  const float r = rsqrtf(ss / d + eps);
  if (threadIdx.x == 0) rstd[row] = r;
#pragma unroll
  for (int j = 0; j < kMaxV; ++j) {
    const int c = (j * kNormThreads + threadIdx.x) * 8;
    if (c < d) {
      float wf[8], o[8];
      load8(w + c, wf);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = v[j][e] * r * wf[e];
      store8(y + row * d + c, o);
    }
  }
}

// dx = rstd * (g - xhat * mean(g * xhat)) (+ residual), g = dy * w, xhat = x * rstd.
// All three row inputs (x, dy, residual) are loaded before the block reduction so their
// latencies overlap; V = vectors of 8 per thread (d <= 2048 V).
template <int V>
__global__ void __launch_bounds__(kNormThreads) rmsnorm_bwd_kernel(const bf16* __restrict__ dy,
                                                                   const bf16* __restrict__ x,
                                                                   const float* __restrict__ rstd,
                                                                   const bf16* __restrict__ w,
                                                                   const bf16* __restrict__ res,
                                                                   bf16* __restrict__ dx, int d) {
  plora::pdl_wait();
  plora::pdl_trigger();
  __shared__ float red[kNormThreads / 32];
  const int64_t row = blockIdx.x;
  const float r = rstd[row];
  float xh[V][8], g[V][8], rf[V][8];
  float dot = 0.f;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int c = (j * kNormThreads + threadIdx.x) * 8;
    if (c < d) {
      float wf[8], df[8];
      load8(x + row * d + c, xh[j]);
      load8(dy + row * d + c, df);
      if (res) load8(res + row * d + c, rf[j]);
      load8(w + c, wf);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xh[j][e] *= r;
        g[j][e] = df[e] * wf[e];
        dot += g[j][e] * xh[j][e];
      }
    }
  }
  const float mean = block_sum<kNormThreads>(dot, red) / d;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int c = (j * kNormThreads + threadIdx.x) * 8;
    if (c < d) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = r * (g[j][e] - xh[j][e] * mean) + (res ? rf[j][e] : 0.f);
      store8(dx + row * d + c, o);
    }
  }
}

// ---------------------------------------------------------------- SwiGLU
__global__ void swiglu_fwd_kernel(const bf16* __restrict__ g, const bf16* __restrict__ u,
                                  bf16* __restrict__ a, int64_t n8) {
  plora::pdl_wait();
  plora::pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float gf[8], uf[8], o[8];
    load8(g + i * 8, gf);
    load8(u + i * 8, uf);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = plora::swiglu_act(gf[e], uf[e]);
    store8(a + i * 8, o);
  }
}

__global__ void swiglu_bwd_kernel(const bf16* __restrict__ da, const bf16* g, const bf16* u, bf16* dg,
                                  bf16* du, bf16* __restrict__ act,
                                  int64_t n8) {
  plora::pdl_wait();
  plora::pdl_trigger();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    float af[8], gf[8], uf[8], og[8], ou[8], oa[8];
    load8(da + i * 8, af);
    load8(g + i * 8, gf);
    load8(u + i * 8, uf);
#pragma unroll
    for (int e = 0; e < 8; ++e) plora::swiglu_bwd_elem(af[e], gf[e], uf[e], og[e], ou[e], oa[e]);
    if (act) store8(act + i * 8, oa);   // the arithmetic of swiglu_fwd: bit-identical activation
    store8(dg + i * 8, og);
    store8(du + i * 8, ou);
  }
}

// ---------------------------------------------------------------- RoPE (+ layout change)
// out[t][h][:] (contiguous [T][H][hd]) = rot(in[b][h][p][:]) with t = b*s + p, strided in.
// Half-rotation convention: (x1, x2) -> (x1 c - x2 s, x2 c + x1 s); inverse uses -sin.
// rotate = 0: plain strided copy.  One thread handles 8 consecutive pairs (16 elements).
__global__ void rope_kernel(const bf16* __restrict__ in, bf16* __restrict__ out,
                            const float* __restrict__ cosv, const float* __restrict__ sinv, int64_t T,
                            int s, int H, int hd, int64_t sb, int64_t sp, int64_t sh, int rotate,
                            float sign) {
  plora::pdl_wait();
  plora::pdl_trigger();
  const int half = hd / 2;
  const int per_head = half / 8;
  const int64_t total = T * H * per_head;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int q = static_cast<int>(i % per_head);
    const int64_t th = i / per_head;
    const int h = static_cast<int>(th % H);
    const int64_t t = th / H;
    const int64_t b = t / s;
    const int p = static_cast<int>(t - b * s);
    const bf16* src = in + b * sb + p * sp + h * sh;
    bf16* dst = out + (t * H + h) * hd;
    float x1[8], x2[8];
    load8(src + q * 8, x1);
    load8(src + half + q * 8, x2);
    if (rotate) {
      float o1[8], o2[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float c = cosv[p * half + q * 8 + e];
        const float sn = sign * sinv[p * half + q * 8 + e];
        o1[e] = x1[e] * c - x2[e] * sn;
        o2[e] = x2[e] * c + x1[e] * sn;
      }
      store8(dst + q * 8, o1);
      store8(dst + half + q * 8, o2);
    } else {
      store8(dst + q * 8, x1);
      store8(dst + half + q * 8, x2);
    }
  }
}

// ---------------------------------------------------------------- cross entropy
// One CTA per token row of bf16 logits [V]: loss_t = w_t (lse - x[label]); the row is
// overwritten with w_t (softmax - onehot(label)).  w_t = 0 rows are zeroed.
constexpr int kCeThreads = 512;

__global__ void __launch_bounds__(kCeThreads) ce_kernel(bf16* __restrict__ logits, const int64_t* __restrict__ labels,
                                                        const float* __restrict__ weight,
                                                        float* __restrict__ tok_loss, int V) {
  plora::pdl_wait();
  plora::pdl_trigger();
  __shared__ float red[kCeThreads / 32];
  __shared__ float redm[kCeThreads / 32];
  const int64_t row = blockIdx.x;
  bf16* x = logits + row * (int64_t)V;
  const int nv = V / 8;
  float m = -INFINITY, sum = 0.f;
  for (int i = threadIdx.x; i < nv; i += kCeThreads) {
    float f[8];
    load8(x + i * 8, f);
    float lm = f[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) lm = fmaxf(lm, f[e]);
    if (lm > m) {
      sum *= __expf(m - lm);
      m = lm;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) sum += __expf(f[e] - m);
  }
  for (int i = nv * 8 + threadIdx.x; i < V; i += kCeThreads) {
    const float f = __bfloat162float(x[i]);
    if (f > m) {
      sum *= __expf(m - f);
      m = f;
    }
    sum += __expf(f - m);
  }
  // block reduce (max, sum)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o);
    const float os = __shfl_xor_sync(0xffffffffu, sum, o);
    const float nm = fmaxf(m, om);
    sum = (m == -INFINITY ? 0.f : sum * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
    m = nm;
  }
  const int wid = threadIdx.x / 32, lid = threadIdx.x % 32;
  if (lid == 0) {
    redm[wid] = m;
    red[wid] = sum;
  }
  __syncthreads();
  float M = -INFINITY;
#pragma unroll
  for (int i = 0; i < kCeThreads / 32; ++i) M = fmaxf(M, redm[i]);
  float S = 0.f;
#pragma unroll
  for (int i = 0; i < kCeThreads / 32; ++i) S += red[i] * __expf(redm[i] - M);
  const float lse = M + __logf(S);
  const float w = weight[row];
  const int64_t lab = labels[row];
  if (threadIdx.x == 0) tok_loss[row] = (w != 0.f) ? w * (lse - __bfloat162float(x[lab])) : 0.f;
  __syncthreads();  // label logit read before it is overwritten
  for (int i = threadIdx.x; i < nv; i += kCeThreads) {
    float f[8];
    load8(x + i * 8, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = w * __expf(f[e] - lse);
    const int64_t base = (int64_t)i * 8;
    if (lab >= base && lab < base + 8) f[lab - base] -= w;
    store8(x + i * 8, f);
  }
  for (int i = nv * 8 + threadIdx.x; i < V; i += kCeThreads) {
    float f = w * __expf(__bfloat162float(x[i]) - lse);
    if (i == lab) f -= w;
    x[i] = __float2bfloat16_rn(f);
  }
}


// ---------------------------------------------------------------- vocab-parallel cross entropy
// Tensor-parallel lm_head (config C4): each rank holds logits for vocabulary slice
// [v0, v0+V).  Pass 1 writes per-row (max, sum exp(x - max), x[label] if the label is
// in this slice else 0); the host all-reduces them across the TP group (max, then the
// rescaled sums and label logits); pass 2 overwrites the slice with
// w_t (softmax - onehot(label)) given the global lse.
__global__ void __launch_bounds__(kCeThreads) ce_stats_kernel(const bf16* __restrict__ logits,
                                                              const int64_t* __restrict__ labels,
                                                              float* __restrict__ stats, int V, int64_t v0) {
  plora::pdl_wait();
  plora::pdl_trigger();
  __shared__ float red[kCeThreads / 32];
  __shared__ float redm[kCeThreads / 32];
  const int64_t row = blockIdx.x;
  const bf16* x = logits + row * (int64_t)V;
  const int nv = V / 8;
  float m = -INFINITY, sum = 0.f;
  for (int i = threadIdx.x; i < nv; i += kCeThreads) {
    float f[8];
    load8(x + i * 8, f);
    float lm = f[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) lm = fmaxf(lm, f[e]);
    if (lm > m) {
      sum *= __expf(m - lm);
      m = lm;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) sum += __expf(f[e] - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o);
    const float os = __shfl_xor_sync(0xffffffffu, sum, o);
    const float nm = fmaxf(m, om);
    sum = (m == -INFINITY ? 0.f : sum * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
    m = nm;
  }
  const int wid = threadIdx.x / 32, lid = threadIdx.x % 32;
  if (lid == 0) {
    redm[wid] = m;
    red[wid] = sum;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = -INFINITY;
#pragma unroll
    for (int i = 0; i < kCeThreads / 32; ++i) M = fmaxf(M, redm[i]);
    float S = 0.f;
#pragma unroll
    for (int i = 0; i < kCeThreads / 32; ++i) S += (redm[i] == -INFINITY) ? 0.f : red[i] * __expf(redm[i] - M);
    const int64_t lab = labels[row] - v0;
    stats[row * 3 + 0] = M;
    stats[row * 3 + 1] = S;
    stats[row * 3 + 2] = (lab >= 0 && lab < V) ? __bfloat162float(x[lab]) : 0.f;
  }
}

__global__ void ce_apply_kernel(bf16* __restrict__ logits, const int64_t* __restrict__ labels,
                                const float* __restrict__ lse, const float* __restrict__ weight, int V,
                                int64_t v0) {
  plora::pdl_wait();
  plora::pdl_trigger();
  const int64_t row = blockIdx.x;
  bf16* x = logits + row * (int64_t)V;
  const float w = weight[row];
  const float l = lse[row];
  const int64_t lab = labels[row] - v0;
  for (int i = threadIdx.x; i < V / 8; i += blockDim.x) {
    float f[8];
    load8(x + i * 8, f);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = w * __expf(f[e] - l);
    const int64_t base = (int64_t)i * 8;
    if (lab >= base && lab < base + 8) f[lab - base] -= w;
    store8(x + i * 8, f);
  }
}

// y[r][c] = bf16(float(y[r][c]) + float(bias[c])) -- a broadcast row bias (narrow q/k/v shards).
__global__ void add_row_bias_kernel(bf16* __restrict__ y, const bf16* __restrict__ bias, int64_t rows, int64_t n,
                                    int64_t ldy) {
  plora::pdl_wait();
  plora::pdl_trigger();
  const int64_t per = n / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * per; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per, c = (i - r * per) * 8;
    float f[8], b[8];
    load8(y + r * ldy + c, f);
    load8(bias + c, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] += b[e];
    store8(y + r * ldy + c, f);
  }
}

#ifndef PLORA_EW_BLOCKS_PER_SM
#define PLORA_EW_BLOCKS_PER_SM 16   // grid-stride elementwise kernels: resident blocks per SM (build-time knob)
#endif

int grid_for(int64_t n, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(sms) * PLORA_EW_BLOCKS_PER_SM;
  return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}

int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return plora::set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

}  // namespace

extern "C" {

PLORA_API int plora_rmsnorm_fwd(void* stream, int64_t rows, int64_t d, const void* x, const void* w,
                                float eps, void* y, float* rstd, int32_t use_given_rstd) {
  if (d % 8 || d > 8 * kNormThreads * kMaxV) return plora::set_error("rmsnorm: d must be a multiple of 8, <= 8192");
  if (rows <= 0) return 0;
  plora::launch_pdl(rmsnorm_fwd_kernel, dim3(rows), dim3(kNormThreads), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(x), static_cast<const bf16*>(w), static_cast<bf16*>(y), rstd, (int)d, eps,
      use_given_rstd);
  return launch_status("rmsnorm_fwd");
}

PLORA_API int plora_add_rmsnorm_fwd(void* stream, int64_t rows, int64_t d, const void* a, const void* b,
                                    const void* w, float eps, void* sum, void* y, float* rstd) {
  if (d % 8 || d > 8 * kNormThreads * kMaxV) return plora::set_error("rmsnorm: d must be a multiple of 8, <= 8192");
  if (rows <= 0) return 0;
  plora::launch_pdl(add_rmsnorm_kernel, dim3(rows), dim3(kNormThreads), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(a), static_cast<const bf16*>(b), static_cast<const bf16*>(w), static_cast<bf16*>(sum),
      static_cast<bf16*>(y), rstd, (int)d, eps);
  return launch_status("add_rmsnorm_fwd");
}

PLORA_API int plora_rmsnorm_bwd(void* stream, int64_t rows, int64_t d, const void* dy, const void* x,
                                const float* rstd, const void* w, const void* residual, void* dx) {
  if (d % 8 || d > 8 * kNormThreads * kMaxV) return plora::set_error("rmsnorm: d must be a multiple of 8, <= 8192");
  if (rows <= 0) return 0;
  auto kern = d <= 8 * kNormThreads ? rmsnorm_bwd_kernel<1>
            : (d <= 16 * kNormThreads ? rmsnorm_bwd_kernel<2> : rmsnorm_bwd_kernel<kMaxV>);
  plora::launch_pdl(kern, dim3(rows), dim3(kNormThreads), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(dy), static_cast<const bf16*>(x), rstd, static_cast<const bf16*>(w),
      static_cast<const bf16*>(residual), static_cast<bf16*>(dx), (int)d);
  return launch_status("rmsnorm_bwd");
}

PLORA_API int plora_swiglu_fwd(void* stream, int64_t n, const void* g, const void* u, void* a) {
  if (n % 8) return plora::set_error("swiglu: n must be a multiple of 8");
  plora::launch_pdl(swiglu_fwd_kernel, dim3(grid_for(n / 8, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(g), static_cast<const bf16*>(u), static_cast<bf16*>(a), n / 8);
  return launch_status("swiglu_fwd");
}

PLORA_API int plora_swiglu_bwd(void* stream, int64_t n, const void* da, const void* g, const void* u, void* dg,
                               void* du, void* act) {
  if (n % 8) return plora::set_error("swiglu: n must be a multiple of 8");
  plora::launch_pdl(swiglu_bwd_kernel, dim3(grid_for(n / 8, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(da), static_cast<const bf16*>(g), static_cast<const bf16*>(u),
      static_cast<bf16*>(dg), static_cast<bf16*>(du), static_cast<bf16*>(act), n / 8);
  return launch_status("swiglu_bwd");
}

PLORA_API int plora_rope(void* stream, const void* in, void* out, const float* cosv, const float* sinv,
                         int64_t T, int32_t s, int32_t H, int32_t hd, int64_t sb, int64_t sp, int64_t sh,
                         int32_t rotate, int32_t inverse) {
  if (hd % 16) return plora::set_error("rope: head_dim must be a multiple of 16");
  if ((sb | sp | sh) % 8) return plora::set_error("rope: strides must be multiples of 8 elements");
  const int64_t total = T * H * (hd / 16);
  plora::launch_pdl(rope_kernel, dim3(grid_for(total, 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(in), static_cast<bf16*>(out), cosv, sinv, T, s, H, hd, sb, sp, sh, rotate,
      inverse ? -1.f : 1.f);
  return launch_status("rope");
}

PLORA_API int plora_cross_entropy(void* stream, int64_t rows, int64_t V, void* logits, const int64_t* labels,
                                  const float* weight, float* tok_loss) {
  if (rows <= 0) return 0;
  if ((V * 2) % 16) return plora::set_error("cross_entropy: V must be a multiple of 8");
  plora::launch_pdl(ce_kernel, dim3(rows), dim3(kCeThreads), 0, static_cast<cudaStream_t>(stream), 
      static_cast<bf16*>(logits), labels, weight, tok_loss, (int)V);
  return launch_status("cross_entropy");
}

PLORA_API int plora_add_row_bias(void* stream, int64_t rows, int64_t n, void* y, int64_t ldy, const void* bias) {
  if (rows <= 0 || n <= 0) return 0;
  if (n % 8 || ldy % 8) return plora::set_error("add_row_bias: n and ldy must be multiples of 8");
  plora::launch_pdl(add_row_bias_kernel, dim3(grid_for(rows * (n / 8), 256)), dim3(256), 0, static_cast<cudaStream_t>(stream), 
      static_cast<bf16*>(y), static_cast<const bf16*>(bias), rows, n, ldy);
  return launch_status("add_row_bias");
}

PLORA_API int plora_ce_stats(void* stream, int64_t rows, int64_t V, const void* logits, const int64_t* labels,
                             int64_t v0, float* stats) {
  if (rows <= 0) return 0;
  if (V % 8) return plora::set_error("ce_stats: V must be a multiple of 8");
  plora::launch_pdl(ce_stats_kernel, dim3(rows), dim3(kCeThreads), 0, static_cast<cudaStream_t>(stream), 
      static_cast<const bf16*>(logits), labels, stats, (int)V, v0);
  return launch_status("ce_stats");
}

PLORA_API int plora_ce_apply(void* stream, int64_t rows, int64_t V, void* logits, const int64_t* labels,
                             int64_t v0, const float* lse, const float* weight) {
  if (rows <= 0) return 0;
  if (V % 8) return plora::set_error("ce_apply: V must be a multiple of 8");
  plora::launch_pdl(ce_apply_kernel, dim3(rows), dim3(256), 0, static_cast<cudaStream_t>(stream), static_cast<bf16*>(logits), labels, lse,
                                                                     weight, (int)V, v0);
  return launch_status("ce_apply");
}

}  // extern "C"
