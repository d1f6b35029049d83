// k_exact.cu -- reference-order instantiation of kernels.cuh (SGWG_ARITH_EXACT)
// plus the scalar step-control kernels.  MUST be compiled with --fmad=false:
// every multiply and add rounds separately, exactly like the reference headers
// built without FMA contraction, so results are bitwise
// equal to the reference.
#define SGWG_NS exact
#define SGWG_FAST 0
#include "kernels.cuh"

#include <limits.h>

namespace sgwg {

// FamilyModel::family_wave_speeds (models.hpp:791-839) over the local members;
// speeds[d] carries the failure flag so one all-reduce(max) propagates it.
__device__ void local_speeds(const DtParams& p, double* sp) {
  for (int k = 0; k < kMaxD + 1; ++k) sp[k] = 0.0;
  if (p.kind == 1) {  // Burgers: family max|u^n| (models.hpp:798-802)
    double umax = 0.0;
    for (int m = 0; m < p.nmembers; ++m) {
      const double a = __longlong_as_double((long long)p.amax[m]);
      umax = (umax < a) ? a : umax;
    }
    for (int k = 0; k < p.d; ++k) sp[k] = umax;
  } else {
    for (int k = 0; k < p.d; ++k) sp[k] = p.const_speeds[k];
    if (p.kind == 3) {  // Vlasov-Poisson: v-directions from the family max|E_j|
      for (int m = 0; m < p.nmembers; ++m)
        for (int j = 0; j < p.space_dim; ++j) {
          const double a = p.emax[m * p.space_dim + j];
          sp[p.space_dim + j] = (sp[p.space_dim + j] < a) ? a : sp[p.space_dim + j];
        }
    }
  }
  double failed = 0.0;
  for (int m = 0; m < p.nmembers; ++m)
    if (p.fail[m] != ULLONG_MAX) failed = 1.0;
  sp[kMaxD] = failed;
}

__global__ void local_speeds_kernel(const DtParams p) {
  if (!p.ctl->active) return;
  local_speeds(p, p.ctl->speeds);
}

// one iteration of evolve_family's step loop (timestep.hpp:152-168) with
// compute_dt (timestep.hpp:47-67) and exact landing (timestep.hpp:155).
__global__ void dt_kernel(const DtParams p) {
  StepCtl* c = p.ctl;
  if (!c->active) return;
  double sp[kMaxD + 1];
  if (p.use_reduced) {
    for (int k = 0; k < kMaxD + 1; ++k) sp[k] = c->speeds[k];
  } else {
    local_speeds(p, sp);
  }
  if (sp[kMaxD] > 0.0) {
    c->active = 0;
    c->failed = 1;
    return;
  }
  if (!(c->stop - c->t > c->eps_t)) {
    c->active = 0;
    return;
  }
  const double remaining = c->stop - c->t;
  double dt;
  if (p.mode == 0) {
    double inv = 0.0;
    for (int k = 0; k < p.d; ++k) inv += sp[k] / p.fine_h[k];
    if (inv == 0.0) {
      dt = remaining;
    } else {
      dt = p.cfl / inv;
      dt = (remaining < dt) ? remaining : dt;  // std::min(dt, remaining)
    }
  } else {
    dt = p.base_dt;
    dt = (remaining < dt) ? remaining : dt;
  }
  if (c->stop - (c->t + dt) <= c->eps_t) dt = c->stop - c->t;
  c->dt = dt;
  c->cur_step = c->step;
  if (p.dts != nullptr && c->step < p.dts_cap) p.dts[c->step] = dt;
  c->step = c->step + 1;
  c->t = c->t + dt;
}

cudaError_t launch_local_speeds(const DtParams& p, cudaStream_t s) {
  local_speeds_kernel<<<1, 1, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_dt(const DtParams& p, cudaStream_t s) {
  dt_kernel<<<1, 1, 0, s>>>(p);
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
