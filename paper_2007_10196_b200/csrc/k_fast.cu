// k_fast.cu -- FMA-contracted, divide-reduced instantiation of kernels.cuh
// (SGWG_ARITH_FAST).  Compiled with the default --fmad=true.
#define SGWG_NS fast
#define SGWG_FAST 1
#include "kernels.cuh"

#ifdef SGWG_TRACE
// experiment builds only: copy the phase trace of the persistent kernel out
extern "C" int sgwg_trace_dump(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, sgwg::fast::sgwg_trace, sizeof(sgwg::fast::sgwg_trace));
}
extern "C" int sgwg_p4trace_dump(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, sgwg::fast::sgwg_p4trace, sizeof(sgwg::fast::sgwg_p4trace));
}
#endif
