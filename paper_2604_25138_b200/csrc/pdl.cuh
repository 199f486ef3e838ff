// Programmatic dependent launch (PDL) for the kernels of one PCG iteration: a kernel
// launched with launch_pdl may be scheduled while its predecessor in the stream is
// still running (in a captured graph the edge becomes a programmatic dependency), so
// its launch latency and prologue overlap the predecessor's tail.  Every such kernel
// runs pdl_prologue() first: the trigger lets its own successor be scheduled (all of
// this grid's CTAs are then already resident, so the successor's CTAs cannot starve
// it), and the wait blocks until the predecessor grid has completed and its writes
// are visible -- nothing produced upstream is read before it.  Launched without the
// attribute, both instructions are no-ops.  Opt-in (LAKER_PDL=1): measured at C3 it
// was slightly slower than plain stream order inside the CUDA graph (2047-2066 vs
// 2106-2111 it/s best, tools/ab_solve.py) -- the persistent one-CTA-per-SM kernels
// cannot start before their predecessor's CTAs leave the SMs anyway.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace laker {

__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char *v = std::getenv("LAKER_PDL");
    on = (v && v[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace laker
