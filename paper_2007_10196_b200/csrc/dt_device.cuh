// dt_device.cuh -- device-side compute_dt + stop landing, exact IEEE arithmetic
// through explicit round-to-nearest intrinsics (never FMA-contracted, whatever
// the TU's --fmad setting), so the dt sequence is bitwise the reference's.
#pragma once
#include <limits.h>

#include "sgwg_internal.h"

namespace sgwg {

__device__ __forceinline__ double vload(const double* p) { return *(volatile const double*)p; }
__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
  return *(volatile const unsigned long long*)p;
}

__device__ __forceinline__ double warp_allmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double w = __shfl_xor_sync(0xffffffffu, v, o);
    v = (v < w) ? w : v;
  }
  return v;
}

// FamilyModel::family_wave_speeds (models.hpp:791-839) over the local members;
// sp[kMaxD] carries the failure flag so one all-reduce(max) propagates it.
// Warp-cooperative: all 32 lanes call, each loads a strided subset of the
// per-member values (through L2) and the maxima are reduced across the warp
// (max is exact and order-independent); every lane gets the result.
__device__ inline void device_local_speeds(const DtParams& p, double* sp) {
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < kMaxD + 1; ++k) sp[k] = 0.0;
  double failed = 0.0;
  for (int m = lane; m < p.nmembers; m += 32)
    if (__ldcg(p.fail + m) != ULLONG_MAX) failed = 1.0;
  if (p.kind == 1) {  // Burgers: family max|u^n| (models.hpp:798-802)
    double umax = 0.0;
    for (int m = lane; m < p.nmembers; m += 32) {
      const double a = __longlong_as_double((long long)__ldcg(p.amax + m));
      umax = (umax < a) ? a : umax;
    }
    umax = warp_allmax(umax);
    for (int k = 0; k < p.d; ++k) sp[k] = umax;
  } else {
    for (int k = 0; k < p.d; ++k) sp[k] = p.const_speeds[k];
    if (p.kind == 4) {  // Vlasov-Maxwell (models.hpp:816-836): s0 constant, s1, s2 per member
      for (int j = 1; j <= 2; ++j) {
        double e = 0.0;
        for (int m = lane; m < p.nmembers; m += 32) {
          const double a = __ldcg(p.vmspd + 2 * m + (j - 1));
          e = (e < a) ? a : e;
        }
        sp[j] = warp_allmax(e);
      }
    }
    if (p.kind == 3) {  // Vlasov-Poisson: v-directions from the family max|E_j|
      for (int j = 0; j < p.space_dim; ++j) {
        double e = 0.0;
        for (int m = lane; m < p.nmembers; m += 32) {
          const double a = __ldcg(p.emax + m * p.space_dim + j);
          e = (e < a) ? a : e;
        }
        sp[p.space_dim + j] = warp_allmax(e);
      }
    }
  }
  sp[kMaxD] = warp_allmax(failed);
}

// one iteration of evolve_family's step loop (timestep.hpp:152-168):
// compute_dt (timestep.hpp:47-67) and the exact landing (timestep.hpp:155),
// applied to the step-control block c (global, or a CTA-local copy).
__device__ inline void device_step_dt_on(const DtParams& p, StepCtl* c, bool use_reduced,
                                         bool write_dts);

__device__ inline void device_step_dt(const DtParams& p, bool use_reduced) {
  device_step_dt_on(p, p.ctl, use_reduced, true);
}

// Warp-cooperative: all 32 lanes of one warp call it; lane 0 writes c.
__device__ inline void device_step_dt_on(const DtParams& p, StepCtl* c, bool use_reduced,
                                         bool write_dts) {
  const bool lead = (threadIdx.x & 31) == 0;
  const int active = c->active;
  const double t = c->t, stop = c->stop, eps_t = c->eps_t;
  const long long step = c->step;
  __syncwarp();
  if (!active) return;
  double sp[kMaxD + 1];
  if (use_reduced) {
    for (int k = 0; k < kMaxD + 1; ++k) sp[k] = vload(&c->speeds[k]);
  } else {
    device_local_speeds(p, sp);
  }
  if (!lead) return;
  if (sp[kMaxD] > 0.0) {
    c->active = 0;
    c->failed = 1;
    return;
  }
  if (!(__dsub_rn(stop, t) > eps_t)) {
    c->active = 0;
    return;
  }
  const double remaining = __dsub_rn(stop, t);
  double dt;
  if (p.mode == 0) {
    double inv = 0.0;
    for (int k = 0; k < p.d; ++k) inv = __dadd_rn(inv, __ddiv_rn(sp[k], p.fine_h[k]));
    if (inv == 0.0) {
      dt = remaining;
    } else {
      dt = __ddiv_rn(p.cfl, inv);
      dt = (remaining < dt) ? remaining : dt;  // std::min(dt, remaining)
    }
  } else {
    dt = p.base_dt;
    dt = (remaining < dt) ? remaining : dt;
  }
  if (__dsub_rn(stop, __dadd_rn(t, dt)) <= eps_t) dt = __dsub_rn(stop, t);
  c->dt = dt;
  c->cur_step = step;
  if (write_dts && p.dts != nullptr && step < p.dts_cap) p.dts[step] = dt;
  c->step = step + 1;
  c->t = __dadd_rn(t, dt);
}

// Last-CTA-done epilogue of the stage-3 kernel: once every CTA of the grid
// has published its max|u| / failure atomics, the last one computes the next
// step's dt, so a step is three kernel launches.
__device__ inline void fused_step_dt(const DtParams* dtp, unsigned int* counter) {
  __shared__ unsigned int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int prev = atomicAdd(counter, 1u);
    s_last = (prev == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    if (threadIdx.x == 0) *counter = 0u;
    device_step_dt(*dtp, false);
  }
}

}  // namespace sgwg
