// Fixed cost of a 1-CTA/SM kernel launch inside a CUDA graph, by ingredient (148 CTAs x 192 threads).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Big { uint32_t w[3200]; };   // 12.8 KB of kernel parameters

template <int V>
__global__ void __launch_bounds__(192, 1) k_var(int* cnt, const __grid_constant__ Big big) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[8];
  if (V >= 2) {
    if (threadIdx.x / 32 == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(512) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  if (V >= 3) {
    if (threadIdx.x == 0)
      for (int i = 0; i < 8; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (V == 5 && threadIdx.x == 0) smem[0] = (uint8_t)big.w[blockIdx.x];
  if (V >= 4 && threadIdx.x == 0) {
    __threadfence();
    atomicAdd(cnt, 1);
  }
  __syncthreads();
  if (V >= 2) {
    if (threadIdx.x / 32 == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512) : "memory");
  }
}

template <int V>
float run(int smem, int* cnt, const Big& big) {
  auto k = k_var<V>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  k<<<148, 192, smem, s>>>(cnt, big);
  cudaStreamSynchronize(s);
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 64; ++i) k<<<148, 192, smem, s>>>(cnt, big);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return best * 1000.f / 64;
}

int main() {
  int* cnt;
  cudaMalloc(&cnt, 4);
  Big big = {};
  printf("V0 empty, no smem                 %.2f us\n", run<0>(0, cnt, big));
  printf("V1 empty, 200 KB dyn smem         %.2f us\n", run<1>(200 * 1024, cnt, big));
  printf("V2 + TMEM alloc/dealloc 512       %.2f us\n", run<2>(200 * 1024, cnt, big));
  printf("V3 + mbarrier init                %.2f us\n", run<3>(200 * 1024, cnt, big));
  printf("V4 + threadfence + atomic         %.2f us\n", run<4>(200 * 1024, cnt, big));
  printf("V5 V1 + 12.8 KB params            %.2f us\n", run<5>(200 * 1024, cnt, big));
  return 0;
}
