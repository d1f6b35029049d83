// pdl.cuh -- programmatic dependent launch for the per-stage kernel chains.
//
// The step of a family is a chain of small dependent kernels (field solve,
// dt, stage kernels; several per RK stage for the kinetic models), replayed
// from CUDA graphs.  Launched with programmatic stream serialization, a kernel
// may be scheduled while its predecessor drains; its first instruction
// (griddepcontrol.wait) blocks until the predecessor has completed and its
// memory is visible, so the semantics are unchanged and the launch latency of
// the chain overlaps the predecessor's tail.  On by default (measured against
// the graph replays it runs in: C4 -0.7 %, C3 -0.6 %, S2 -0.3 %, C5 +-0; the
// whole GPU test suite passes with it); SGWG_PDL=0 switches it off.
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace sgwg {

// Wait for the predecessor grid (complete, memory visible), then let the
// successor be scheduled as soon as every CTA of this grid has started: its
// own griddepcontrol.wait still holds it until this grid has finished.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SGWG_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  // the stream's priority stated on the launch itself, so that a captured kernel node
  // carries it whatever the capture inherits
  int prio = 0;
  cudaStreamGetPriority(s, &prio);
  at[0].id = cudaLaunchAttributePriority;
  at[0].val.priority = prio;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace sgwg
