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
#include "pdl.cuh"

namespace sgwg {

__global__ void local_speeds_kernel(const DtParams p) {
  pdl_wait();
  if (!p.ctl->active) return;
  double sp[kMaxD + 1];
  device_local_speeds(p, sp);  // warp-cooperative
  if (threadIdx.x == 0)
    for (int k = 0; k < kMaxD + 1; ++k) p.ctl->speeds[k] = sp[k];
}

__global__ void dt_kernel(const DtParams p) {
  pdl_wait();
  device_step_dt(p, p.use_reduced != 0);
}

// timing experiments only (SGWG_STAMPS): the device clock at a point of a stream
__global__ void stamp_kernel(long long* tl, int slot) {
  pdl_wait();
  long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  tl[slot] = g;
}

cudaError_t launch_stamp(long long* tl, int slot, cudaStream_t s) {
  return launch_k(stamp_kernel, dim3(1), dim3(1), 0, s, tl, slot);
}

cudaError_t launch_local_speeds(const DtParams& p, cudaStream_t s) {
  return launch_k(local_speeds_kernel, dim3(1), dim3(32), 0, s, p);
}

cudaError_t launch_dt(const DtParams& p, cudaStream_t s) {
  return launch_k(dt_kernel, dim3(1), dim3(32), 0, s, p);
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

// family_wave_speeds, Vlasov-Maxwell branch (models.hpp:816-836), per member:
// s1 = max |E1(x2) + xi2 B3(x2)|, s2 = max |E2(x2) - xi1 B3(x2)| over the
// member's x2 points and velocity coordinates (max is exact in any order)
__global__ void __launch_bounds__(256) vm_speeds_kernel(const VmParams p) {
  pdl_wait();
  if (p.ctl != nullptr && !p.ctl->active) return;
  const MemberDesc* M = p.mem + blockIdx.x;
  const int nx = M->nx, n1 = M->ext[1], n2 = M->ext[2];
  const double* F = p.fin + M->xoff * 3;
  double s1 = 0.0, s2 = 0.0;
  for (int q = threadIdx.x; q < nx * n2; q += blockDim.x) {
    const int ix = q / n2, i2 = q % n2;
    const double xi2 = __dadd_rn(M->lower[2], __dmul_rn((double)i2, M->h[2]));
    const double v = fabs(__dadd_rn(F[ix], __dmul_rn(xi2, F[2 * nx + ix])));
    s1 = (s1 < v) ? v : s1;
  }
  for (int q = threadIdx.x; q < nx * n1; q += blockDim.x) {
    const int ix = q / n1, i1 = q % n1;
    const double xi1 = __dadd_rn(M->lower[1], __dmul_rn((double)i1, M->h[1]));
    const double v = fabs(__dsub_rn(F[nx + ix], __dmul_rn(xi1, F[2 * nx + ix])));
    s2 = (s2 < v) ? v : s2;
  }
  s1 = warp_allmax(s1);
  s2 = warp_allmax(s2);
  __shared__ double r[2][8];
  if ((threadIdx.x & 31) == 0) {
    r[0][threadIdx.x >> 5] = s1;
    r[1][threadIdx.x >> 5] = s2;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double m = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = (m < r[threadIdx.x][w]) ? r[threadIdx.x][w] : m;
    p.speeds[2 * blockIdx.x + threadIdx.x] = m;
  }
}

cudaError_t launch_vm_speeds(const VmParams& p, int nmembers, cudaStream_t s) {
  if (nmembers <= 0) return cudaSuccess;
  return launch_k(vm_speeds_kernel, dim3(nmembers), dim3(256), 0, s, p);
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
