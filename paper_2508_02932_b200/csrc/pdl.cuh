// pdl.cuh -- programmatic dependent launch for every libplora kernel.
//
// Kernels are launched with cudaLaunchAttributeProgrammaticStreamSerialization: the next
// libplora kernel in the stream is scheduled as soon as every CTA of the current one has
// started (pdl_trigger() at kernel entry), so its launch latency and its prologue (barrier
// init, TMEM allocation, tensor-map prefetch) run under the current kernel's tail instead
// of after it.  Every kernel calls pdl_wait() -- which returns once the preceding grid has
// completed and its memory is visible -- before its first global-memory access (read OR
// write), so stream order is preserved exactly.  A preceding kernel that never triggers
// (torch / cuDNN) completes first, as without the attribute.  Inside CUDA graphs the
// dependency becomes a programmatic edge.
#pragma once
#include <cuda_runtime.h>

#include <utility>

#ifndef PLORA_PDL
#define PLORA_PDL 0   // build-time knob, off: same-box A/B -0.9% at C3, -1% at the 8-GPU split (profiles/r2_pdl_ab.log)
#endif

namespace plora {

__device__ __forceinline__ void pdl_wait() {
#if PLORA_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

__device__ __forceinline__ void pdl_trigger() {
#if PLORA_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = PLORA_PDL ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace plora
