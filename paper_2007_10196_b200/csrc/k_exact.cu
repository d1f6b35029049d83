// k_exact.cu -- reference-order instantiation of kernels.cuh (SGWG_ARITH_EXACT)
// plus the scalar step-control kernels.  MUST be compiled with --fmad=false:
// every multiply and add rounds separately, exactly like the reference headers
// built without FMA contraction, so results are bitwise
// equal to the reference.
#define SGWG_NS exact
#define SGWG_FAST 0
#include "kernels.cuh"

#include <limits.h>

#include "dt_device.cuh"

namespace sgwg {

__global__ void local_speeds_kernel(const DtParams p) {
  if (!p.ctl->active) return;
  double sp[kMaxD + 1];
  device_local_speeds(p, sp);  // warp-cooperative
  if (threadIdx.x == 0)
    for (int k = 0; k < kMaxD + 1; ++k) p.ctl->speeds[k] = sp[k];
}

__global__ void dt_kernel(const DtParams p) { device_step_dt(p, p.use_reduced != 0); }

cudaError_t launch_local_speeds(const DtParams& p, cudaStream_t s) {
  local_speeds_kernel<<<1, 32, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_dt(const DtParams& p, cudaStream_t s) {
  dt_kernel<<<1, 32, 0, s>>>(p);
  return cudaGetLastError();
}

// detail::max_abs (models.hpp:110-114) of every member, as u64 bit patterns
__global__ void member_max_kernel(const MemberDesc* mem, const int2* tasks, const double* u,
                                  unsigned long long* amax) {
  const int2 tk = tasks[blockIdx.x];
  const MemberDesc* M = mem + tk.x;
  const long long start = (long long)tk.y * 4096;
  const long long end = min(start + 4096, M->npts);
  double v = 0.0;
  for (long long i = start + threadIdx.x; i < end; i += blockDim.x)
    v = fmax(v, fabs(u[M->offset + i]));
  v = exact::warp_max(v);
  if ((threadIdx.x & 31) == 0) atomicMax(amax + tk.x, (unsigned long long)__double_as_longlong(v));
}

cudaError_t launch_member_max(const MemberDesc* mem, int nmembers, const int2* tasks, int ntasks,
                              const double* u, unsigned long long* amax, cudaStream_t s) {
  (void)nmembers;
  if (ntasks <= 0) return cudaSuccess;
  member_max_kernel<<<ntasks, 256, 0, s>>>(mem, tasks, u, amax);
  return cudaGetLastError();
}

// DFMA throughput probe: 8 independent FMA chains per thread.
__global__ void __launch_bounds__(256) fp64_peak_kernel(double* out, int iters) {
  double a[8];
  const double x = 1.0 + 1e-9 * threadIdx.x, y = 1.0 - 1e-9 * blockIdx.x;
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = q * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = __fma_rn(a[q], x, y);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += a[q];
  if (s == 123.456) out[0] = s;
}

cudaError_t launch_fp64_peak(double* out, int iters, int blocks, cudaStream_t s) {
  fp64_peak_kernel<<<blocks, 256, 0, s>>>(out, iters);
  return cudaGetLastError();
}

}  // namespace sgwg
