// kernels.cuh -- sm_100a fp64 kernels of the sparse-grid WENO5 hot path.
//
// Included twice: k_exact.cu (SGWG_FAST=0, compiled with --fmad=false) keeps
// the reference's expression order and IEEE divides so results are bitwise
// equal to the reference built without FMA; k_fast.cu (SGWG_FAST=1) contracts
// to DFMA, uses one divide per reconstruction (common denominator of the three
// nonlinear weights) and reciprocal spacings -- within 1e-10 of the reference.
//
// Kernels
//   pass_kernel<BURGERS>  one dimension-by-dimension WENO5 sweep of every member
//                         of the family (batched), accumulating the tendency in
//                         the reference's order; the last pass of an RK stage
//                         fuses the SSP-RK3 stage update, the non-finite check
//                         and the per-member max|u| of the stage output.
//                         Replaces advective_sweep / flux_sweep (models.hpp:142-177)
//                         -> advect_derivative_line / weno_derivative_line
//                         (weno.hpp:118-192) and SspRk3::step (timestep.hpp:86-104).
//   upsample_kernel       one dimension of prolong (interp.hpp:217-244) for all
//                         members at once (upsample_line, interp.hpp:151-189).
//   final_kernel          the last dimension of prolong fused with the signed
//                         combination sum in sorted member order (combine.hpp:113-120).
#pragma once
#include <cooperative_groups.h>

#include "dt_device.cuh"
#include "pdl.cuh"
#include "sgwg_internal.h"

#ifndef SGWG_FAST
#error "define SGWG_FAST"
#endif

namespace sgwg {
namespace SGWG_NS {

constexpr double kSixth = 1.0 / 6.0;  // weno.hpp:30

__device__ __forceinline__ double sq(double x) { return x * x; }

// weno5_flux_positive (weno.hpp:60-72) with smoothness_indicators (weno.hpp:36-44),
// reference expression order.
__device__ __forceinline__ double recon_ref(double s0, double s1, double s2, double s3, double s4,
                                            double eps, int linear) {
  const double c0 = kSixth * (2.0 * s0 - 7.0 * s1 + 11.0 * s2);
  const double c1 = kSixth * (-s1 + 5.0 * s2 + 2.0 * s3);
  const double c2 = kSixth * (2.0 * s2 + 5.0 * s3 - s4);
  if (linear) return 0.1 * c0 + 0.6 * c1 + 0.3 * c2;
  const double b0 = (13.0 / 12.0) * sq(s0 - 2.0 * s1 + s2) + 0.25 * sq(s0 - 4.0 * s1 + 3.0 * s2);
  const double b1 = (13.0 / 12.0) * sq(s1 - 2.0 * s2 + s3) + 0.25 * sq(s1 - s3);
  const double b2 = (13.0 / 12.0) * sq(s2 - 2.0 * s3 + s4) + 0.25 * sq(3.0 * s2 - 4.0 * s3 + s4);
  const double a0 = 0.1 / sq(eps + b0);
  const double a1 = 0.6 / sq(eps + b1);
  const double a2 = 0.3 / sq(eps + b2);
  return (a0 * c0 + a1 * c1 + a2 * c2) / (a0 + a1 + a2);
}

#if SGWG_FAST
// Same reconstruction with the three weights over a common denominator:
//   sum_r d_r c_r / q_r / sum_r d_r / q_r = sum_r d_r c_r Q_r / sum_r d_r Q_r,
//   q_r = (eps+b_r)^2, Q_0 = q_1 q_2, Q_1 = q_0 q_2, Q_2 = q_0 q_1.
// One divide instead of four.  Q_r overflows only for b_r ~ 1e77; then the
// reference form is used.
__device__ __forceinline__ double recon(double s0, double s1, double s2, double s3, double s4,
                                        double eps, int linear) {
  const double c0 = fma(2.0, s0, fma(-7.0, s1, 11.0 * s2));
  const double c1 = fma(5.0, s2, fma(2.0, s3, -s1));
  const double c2 = fma(2.0, s2, fma(5.0, s3, -s4));
  if (linear) return kSixth * fma(0.1, c0, fma(0.6, c1, 0.3 * c2));
  const double d0 = s0 - 2.0 * s1 + s2, g0 = s0 - 4.0 * s1 + 3.0 * s2;
  const double d1 = s1 - 2.0 * s2 + s3, g1 = s1 - s3;
  const double d2 = s2 - 2.0 * s3 + s4, g2 = 3.0 * s2 - 4.0 * s3 + s4;
  const double e0 = fma(13.0 / 12.0 * d0, d0, fma(0.25 * g0, g0, eps));
  const double e1 = fma(13.0 / 12.0 * d1, d1, fma(0.25 * g1, g1, eps));
  const double e2 = fma(13.0 / 12.0 * d2, d2, fma(0.25 * g2, g2, eps));
  const double q0 = e0 * e0, q1 = e1 * e1, q2 = e2 * e2;
  const double w0 = 0.1 * (q1 * q2), w1 = 0.6 * (q0 * q2), w2 = 0.3 * (q0 * q1);
  const double den = 6.0 * (w0 + w1 + w2);
  if (!(den < 1.0e300)) return recon_ref(s0, s1, s2, s3, s4, eps, linear);
  return fma(w0, c0, fma(w1, c1, w2 * c2)) / den;
}
#else
__device__ __forceinline__ double recon(double s0, double s1, double s2, double s3, double s4,
                                        double eps, int linear) {
  return recon_ref(s0, s1, s2, s3, s4, eps, linear);
}
#endif

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

#if SGWG_FAST
#ifndef SGWG_SWEEP_ATTR
#define SGWG_SWEEP_ATTR __noinline__
#endif
template <bool BURGERS, int RUN, bool LINEAR, bool NEWTON = false>
__device__ SGWG_SWEEP_ATTR void sweep_run(const double* __restrict__ P,
                                       const double* __restrict__ Mv, int st, int p0, double c,
                                       double eps4, double inv_h, double* __restrict__ out,
                                       int ost);
#endif

// Lines of dimension k of a member: line L -> (outer o, inner i), base offset
// o*n*inner + i, element j at base + j*inner (grid.hpp:202-217, line_at order).
template <bool BURGERS>
__global__ void __launch_bounds__(kPassThreads) pass_kernel(const PassParams p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  const int4 tk = p.tasks[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  const int k = p.kdim;
  const int n = M->ext[k];
  const long long inner = M->stride[k];
  const int S = M->segS[k], P = M->runP[k], W = M->linesW[k], pitch = M->pitch[k];
  const long long nlines = M->npts / n;
  const long long L0 = tk.y;
  const int seg0 = tk.z;
  const int Weff = (int)min((long long)W, nlines - L0);
  const int Seff = min(S, n - seg0);
  const int bc = M->bc[k];
  const int tid = threadIdx.x;

  extern __shared__ double smem[];
  double* sfp = smem;
  double* sfm = smem + p.dyn_smem_doubles;
  double* scoef = smem + (BURGERS ? 2 : 1) * p.dyn_smem_doubles;
  long long* sbase = reinterpret_cast<long long*>(scoef + W);  // member-local line bases

  if (p.amax_zero != nullptr && blockIdx.x == 0)
    for (int i = tid; i < p.nmembers; i += blockDim.x) p.amax_zero[i] = 0ull;

  // fixed (line, run) coordinates of this thread: lane-consecutive lines
  const int R = (S + P - 1) / P;
  const int w = tid % W;
  const int r = tid / W;
  const int in32 = (int)inner;  // member-local offsets fit in 32 bits

  // line bases and per-line coefficients (advective_sweep coef_of_line)
  if (tid < Weff) {
    const long long L = L0 + tid;
    const long long o = L / inner, i = L % inner;
    const long long base = o * (long long)n * inner + i;
    sbase[tid] = base;
    double c = p.c_const;
    if (p.flux == kFluxKinX) {  // models.hpp:341-344: coefficient v_j
      const int q = p.space_dim + k;
      const int idx = (int)((base / M->stride[q]) % M->ext[q]);
      c = M->lower[q] + idx * M->h[q];
    } else if (p.flux == kFluxKinVB) {  // models.hpp:346-349: coefficient -x_j
      const int q = k - p.space_dim;
      const int idx = (int)((base / M->stride[q]) % M->ext[q]);
      c = -(M->lower[q] + idx * M->h[q]);
    } else if (p.flux == kFluxKinVP) {  // -E_j(x) of this member's Poisson field
      const int comp = k - p.space_dim;
      const long long xi = base / M->vn;
      c = -p.efield[M->xoff * p.space_dim + (long long)comp * M->nx + xi];
    } else if (p.flux >= kFluxVM0) {  // Vlasov-Maxwell (models.hpp:456-480)
      const int ix = (int)(base / M->stride[0]);
      const int i1 = (int)((base / M->stride[1]) % M->ext[1]);
      const int i2 = (int)(base % M->ext[2]);
      const double* F = p.efield + M->xoff * 3;  // E1, E2, B3 of the stage input
      const double xi1 = M->lower[1] + i1 * M->h[1], xi2 = M->lower[2] + i2 * M->h[2];
      if (p.flux == kFluxVM0)
        c = xi2;
      else if (p.flux == kFluxVM1)
        c = F[ix] + xi2 * F[2 * M->nx + ix];
      else
        c = F[M->nx + ix] - xi1 * F[2 * M->nx + ix];
    }
    scoef[tid] = c;
  }
  __syncthreads();

  // gather the padded segment [seg0-3, seg0+Seff+3) of every line; periodic
  // wrap ((j%n)+n)%n or zero ghosts (weno.hpp:131-141); split fluxes.
  const double* u = p.uin + M->offset;
  const int len = Seff + 6;
  const double alpha = BURGERS ? __longlong_as_double((long long)p.amax_in[tk.x]) : 0.0;
  auto load_in = [&](int ww, int jj) -> double {
    int j = seg0 - 3 + jj;
    if (bc == 0) {  // |excursion| <= 3 < n (periodic lines have n >= 6)
      j = (j < 0) ? j + n : (j >= n ? j - n : j);
      return __ldg(u + (int)sbase[ww] + j * in32);
    }
    return (j >= 0 && j < n) ? __ldg(u + (int)sbase[ww] + j * in32) : 0.0;
  };
  auto stage_in = [&](int ww, int jj, double uj) {
    if (BURGERS) {
      const double f = 0.5 * uj * uj;           // models.hpp:194
      const double fpj = 0.5 * (f + alpha * uj);  // weno.hpp:138-140
      sfp[ww * pitch + jj] = fpj;
      sfm[ww * pitch + jj] = f - fpj;
    } else {
#if SGWG_FAST
      sfp[ww * pitch + jj] = uj;  // sweep_run applies the line coefficient
#else
      sfp[ww * pitch + jj] = scoef[ww] * uj;  // weno.hpp:176
#endif
    }
  };
  // loads are issued in batches of kBatch before any of them is used
  constexpr int kBatch = 8;
  if (inner > 1) {  // strided lines: lanes walk adjacent lines (coalesced), rows by run
    if (w < Weff && r < R) {
      for (int jb = r; jb < len; jb += kBatch * R) {
        double v[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
          const int jj = jb + b * R;
          v[b] = (jj < len) ? load_in(w, jj) : 0.0;
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
          const int jj = jb + b * R;
          if (jj < len) stage_in(w, jj, v[b]);
        }
      }
    }
  } else {  // contiguous lines: lanes walk along the line
    const float inv_len = 1.0f / (float)len;
    const int tot = Weff * len;
    for (int qb = tid; qb < tot; qb += kBatch * blockDim.x) {
      double v[kBatch];
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
        const int q = qb + b * blockDim.x;
        const int ww = (int)(((float)q + 0.5f) * inv_len);
        v[b] = (q < tot) ? load_in(ww, q - ww * len) : 0.0;
      }
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
        const int q = qb + b * blockDim.x;
        const int ww = (int)(((float)q + 0.5f) * inv_len);
        if (q < tot) stage_in(ww, q - ww * len, v[b]);
      }
    }
  }
  __syncthreads();

  // interfaces and flux differences: thread (w, r) owns points [r*P, r*P+P)
  // of line w and recomputes the interface left of its run.
  const int j0 = r * P;
  const bool mine = (r < R) && (w < Weff) && (j0 < Seff);
  const double eps = p.eps;
  const int linear = p.linear;
#if SGWG_FAST
  // shared-term sliding sweep over whole runs of P (4 or 8) points; outputs
  // past the segment end are computed on padding and discarded
  double* sdu = reinterpret_cast<double*>(sbase + W);
  if (mine) {
    const double c = BURGERS ? 0.0 : scoef[w];
    const double* Pl = sfp + w * pitch;
    const double* Ml = (BURGERS ? sfm : sfp) + w * pitch;
    double* o = sdu + w * pitch + j0;
    const double eps4 = 4.0 * eps, inv_h = M->inv_h[k];
    if (P == 8) {
      if (linear)
        sweep_run<BURGERS, 8, true>(Pl, Ml, 1, j0, c, eps4, inv_h, o, 1);
      else
        sweep_run<BURGERS, 8, false>(Pl, Ml, 1, j0, c, eps4, inv_h, o, 1);
    } else {
      if (linear)
        sweep_run<BURGERS, 4, true>(Pl, Ml, 1, j0, c, eps4, inv_h, o, 1);
      else
        sweep_run<BURGERS, 4, false>(Pl, Ml, 1, j0, c, eps4, inv_h, o, 1);
    }
  }
  __syncthreads();
  const double* dub = sdu;
  const int dpitch = pitch;
#else
  double du[kMaxRun];
  if (mine) {
    const double* fp = sfp + w * pitch;
    const double* fm = sfm + w * pitch;
    const double c = scoef[w];
    const int bdir = (c < 0.0) ? 5 : 0;  // downwind: reversed window (weno.hpp:178-183)
    const int sdir = (c < 0.0) ? -1 : 1;
    auto flux_at = [&](int jl) -> double {  // interface jl+1/2 (local index)
      if (BURGERS) {
        const double* a = fp + jl + 1;
        const double* b = fm + jl + 2;
        return recon(a[0], a[1], a[2], a[3], a[4], eps, linear) +
               recon(b[4], b[3], b[2], b[1], b[0], eps, linear);
      } else {
        const double* a = fp + jl + 1 + bdir;
        return recon(a[0], a[sdir], a[2 * sdir], a[3 * sdir], a[4 * sdir], eps, linear);
      }
    };
#if SGWG_FAST
    const double inv_h = M->inv_h[k];
#else
    const double h = M->h[k];
#endif
    double fprev = flux_at(j0 - 1);
#pragma unroll
    for (int t = 0; t < kMaxRun; ++t) {
      const int jl = j0 + t;
      if (t < P && jl < Seff) {
        const double f = flux_at(jl);
#if SGWG_FAST
        du[t] = (f - fprev) * inv_h;
#else
        du[t] = (f - fprev) / h;  // weno.hpp:147,152
#endif
        fprev = f;
      }
    }
  }
  __syncthreads();
  if (mine) {
#pragma unroll
    for (int t = 0; t < kMaxRun; ++t)
      if (t < P && j0 + t < Seff) sfp[w * S + j0 + t] = du[t];
  }
  __syncthreads();
  const double* dub = sfp;
  const int dpitch = S;
#endif

  // accumulate out -= du in dimension order (models.hpp:155,175,187-197) and,
  // on the last pass, the SSP-RK3 stage update (timestep.hpp:93,98,103).
  double lmax = 0.0;
  const double dt = (ctl != nullptr) ? ctl->dt : 0.0;
  double* kb = p.kbuf + M->offset;
  const double* ub = p.uin + M->offset;
  const double* nb = p.un + M->offset;
  double* ob = p.out + M->offset;
  // phase 1 of a batch: the global values this point needs (k accumulator,
  // u_in, u^n); phase 2: accumulate / RK update / store
  struct Pre {
    double k, ui, un;
  };
  auto prefetch = [&](int ww, int jl) -> Pre {
    const int gi = (int)sbase[ww] + (seg0 + jl) * in32;
    Pre v{0.0, 0.0, 0.0};
    if (!p.first) v.k = kb[gi];
    if (p.last && p.stage > 0) {
      v.ui = ub[gi];
      if (p.stage > 1) v.un = nb[gi];
    }
    return v;
  };
  auto finish = [&](int ww, int jl, const Pre& v) {
    const int gi = (int)sbase[ww] + (seg0 + jl) * in32;
    const double d = dub[ww * dpitch + jl];
    const double kv = p.first ? (0.0 - d) : (v.k - d);
    if (!p.last) {
      kb[gi] = kv;
      return;
    }
    double o;
    if (p.stage == 0) {
      o = kv;
    } else {
      if (!isfinite(kv)) {  // tendency_finite (timestep.hpp:71-75)
        const unsigned long long code =
            (unsigned long long)ctl->cur_step * 4ull + (unsigned long long)p.stage;
        atomicMin(p.fail + tk.x, code);
      }
      const double ui = v.ui;
      if (p.stage == 1) {
        o = ui + dt * kv;
      } else if (p.stage == 2) {
        o = 0.75 * v.un + 0.25 * (ui + dt * kv);
      } else {
        o = (1.0 / 3.0) * v.un + (2.0 / 3.0) * (ui + dt * kv);
      }
    }
    ob[gi] = o;
    lmax = fmax(lmax, fabs(o));
  };
  constexpr int kEpi = 4;
  if (inner > 1) {
    if (w < Weff && r < R) {
      for (int jb = r; jb < Seff; jb += kEpi * R) {
        Pre v[kEpi];
#pragma unroll
        for (int b = 0; b < kEpi; ++b)
          if (jb + b * R < Seff) v[b] = prefetch(w, jb + b * R);
#pragma unroll
        for (int b = 0; b < kEpi; ++b)
          if (jb + b * R < Seff) finish(w, jb + b * R, v[b]);
      }
    }
  } else {
    const float inv_s = 1.0f / (float)Seff;
    const int tot = Weff * Seff;
    for (int qb = tid; qb < tot; qb += kEpi * blockDim.x) {
      Pre v[kEpi];
#pragma unroll
      for (int b = 0; b < kEpi; ++b) {
        const int q = qb + b * blockDim.x;
        const int ww = (int)(((float)q + 0.5f) * inv_s);
        if (q < tot) v[b] = prefetch(ww, q - ww * Seff);
      }
#pragma unroll
      for (int b = 0; b < kEpi; ++b) {
        const int q = qb + b * blockDim.x;
        const int ww = (int)(((float)q + 0.5f) * inv_s);
        if (q < tot) finish(ww, q - ww * Seff, v[b]);
      }
    }
  }
  if (p.last && p.track_max) {
    lmax = warp_max(lmax);
    if ((tid & 31) == 0)
      atomicMax(p.amax_out + tk.x, (unsigned long long)__double_as_longlong(lmax));
  }
  if (p.last && p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

// ---------------------------------------------------------------------------
// fused 2D stage: both sweeps + SSP-RK3 stage update in one launch
// ---------------------------------------------------------------------------
// A CTA owns a TX x TY tile of one member (thread per point).  It stages the
// tile plus 3-point halos along each axis (no corners) in shared memory,
// computes every x-interface flux F(i+1/2, j) and y-interface flux
// G(i, j+1/2) of the tile exactly once, then forms
//   k = (0 - (F(i+1/2)-F(i-1/2))/h0) - (G(j+1/2)-G(j-1/2))/h1
// in the reference's accumulation order (models.hpp:187-197) and applies the
// RK stage.  Same arithmetic per interface as pass_kernel, so both are
// bitwise equal to the reference in the exact build.
__device__ __forceinline__ double line_coef(int flux, const MemberDesc* M, int k, int space_dim,
                                            int idx_other, double c_const,
                                            const double* efield) {
  if (flux == kFluxKinX) return M->lower[space_dim + k] + idx_other * M->h[space_dim + k];
  if (flux == kFluxKinVB) return -(M->lower[k - space_dim] + idx_other * M->h[k - space_dim]);
  if (flux == kFluxKinVP) return -efield[M->xoff * space_dim + (long long)(k - space_dim) * M->nx +
                                         idx_other];
  return c_const;
}

template <bool BURGERS>
__global__ void __launch_bounds__(256) stage2d_kernel(const Stage2DParams p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  const int4 tk = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  const int n0 = M->ext[0], n1 = M->ext[1];
  const int TX = M->tx, TY = M->ty;
  const int i0 = tk.y, j0 = tk.z;
  const int TXe = min(TX, n0 - i0), TYe = min(TY, n1 - j0);
  const int PY = TY + 6;
  const int tid = threadIdx.x, nt = blockDim.x;
  extern __shared__ double sm[];
  double* A = sm;                                      // fp (Burgers) or u
  double* Bm = A + (TX + 6) * PY;                      // fm (Burgers)
  double* Fx = BURGERS ? Bm + (TX + 6) * PY : Bm;      // (TX+1) x TY
  double* Fy = Fx + (TX + 1) * TY;                     // TX x (TY+1)
  double* cx = Fy + TX * (TY + 1);                     // per column (x-lines)
  double* cy = cx + TY;                                // per row (y-lines)

  if (p.amax_zero != nullptr && blockIdx.x == 0)
    for (int i = tid; i < p.nmembers; i += nt) p.amax_zero[i] = 0ull;
  if (!BURGERS) {
    for (int j = tid; j < TYe; j += nt)
      cx[j] = line_coef(p.flux0, M, 0, p.space_dim, j0 + j, p.c0, p.efield);
    for (int i = tid; i < TXe; i += nt)
      cy[i] = line_coef(p.flux1, M, 1, p.space_dim, i0 + i, p.c1, p.efield);
  }
  const double* u = p.uin + M->offset;
  const double alpha = BURGERS ? __longlong_as_double((long long)p.amax_in[tk.x]) : 0.0;
  const int bc0 = M->bc[0], bc1 = M->bc[1];
  const int LX = TXe + 6, LY = TYe + 6;
  for (int q = tid; q < LX * LY; q += nt) {
    const int a = q / LY, b = q - a * LY;
    if ((a < 3 || a >= TXe + 3) && (b < 3 || b >= TYe + 3)) continue;  // corners unused
    int gi = i0 - 3 + a, gj = j0 - 3 + b;
    bool zero = false;
    if (bc0 == 0) {
      gi %= n0;
      if (gi < 0) gi += n0;
    } else if (gi < 0 || gi >= n0) {
      zero = true;
    }
    if (bc1 == 0) {
      gj %= n1;
      if (gj < 0) gj += n1;
    } else if (gj < 0 || gj >= n1) {
      zero = true;
    }
    const double uj = zero ? 0.0 : __ldg(u + (long long)gi * n1 + gj);
    if (BURGERS) {
      const double f = 0.5 * uj * uj;             // models.hpp:194
      const double fpj = 0.5 * (f + alpha * uj);  // weno.hpp:138-140
      A[a * PY + b] = fpj;
      Bm[a * PY + b] = f - fpj;
    } else {
      A[a * PY + b] = uj;
    }
  }
  __syncthreads();

  const double eps = p.eps;
  const int linear = p.linear;
  // x-interfaces: (TXe+1) x TYe, F[ia][j] = flux at (i0+ia-1)+1/2, column j
  for (int q = tid; q < (TXe + 1) * TYe; q += nt) {
    const int ia = q / TYe, j = q - ia * TYe;
    const double* col = A + j + 3;
    double F;
    if (BURGERS) {
      const double* colm = Bm + j + 3;
      F = recon(col[ia * PY], col[(ia + 1) * PY], col[(ia + 2) * PY], col[(ia + 3) * PY],
                col[(ia + 4) * PY], eps, linear) +
          recon(colm[(ia + 5) * PY], colm[(ia + 4) * PY], colm[(ia + 3) * PY],
                colm[(ia + 2) * PY], colm[(ia + 1) * PY], eps, linear);
    } else {
      const double c = cx[j];
      const int b0 = (c < 0.0) ? ia + 5 : ia;  // downwind: reversed window (weno.hpp:178-183)
      const int s = (c < 0.0) ? -PY : PY;
      const double* w = col + b0 * PY;
      F = recon(c * w[0], c * w[s], c * w[2 * s], c * w[3 * s], c * w[4 * s], eps, linear);
    }
    Fx[ia * TY + j] = F;
  }
  // y-interfaces: TXe x (TYe+1), G[i][jb] = flux at row i, (j0+jb-1)+1/2
  for (int q = tid; q < TXe * (TYe + 1); q += nt) {
    const int i = q / (TYe + 1), jb = q - i * (TYe + 1);
    const double* row = A + (i + 3) * PY;
    double G;
    if (BURGERS) {
      const double* rowm = Bm + (i + 3) * PY;
      G = recon(row[jb], row[jb + 1], row[jb + 2], row[jb + 3], row[jb + 4], eps, linear) +
          recon(rowm[jb + 5], rowm[jb + 4], rowm[jb + 3], rowm[jb + 2], rowm[jb + 1], eps,
                linear);
    } else {
      const double c = cy[i];
      const int b0 = (c < 0.0) ? jb + 5 : jb;
      const int s = (c < 0.0) ? -1 : 1;
      const double* w = row + b0;
      G = recon(c * w[0], c * w[s], c * w[2 * s], c * w[3 * s], c * w[4 * s], eps, linear);
    }
    Fy[i * (TY + 1) + jb] = G;
  }
  __syncthreads();

  double lmax = 0.0;
  const int ti = tid / TY, tj = tid - (tid / TY) * TY;
  if (ti < TXe && tj < TYe) {
#if SGWG_FAST
    const double dux = (Fx[(ti + 1) * TY + tj] - Fx[ti * TY + tj]) * M->inv_h[0];
    const double duy = (Fy[ti * (TY + 1) + tj + 1] - Fy[ti * (TY + 1) + tj]) * M->inv_h[1];
#else
    const double dux = (Fx[(ti + 1) * TY + tj] - Fx[ti * TY + tj]) / M->h[0];
    const double duy = (Fy[ti * (TY + 1) + tj + 1] - Fy[ti * (TY + 1) + tj]) / M->h[1];
#endif
    const double kv = (0.0 - dux) - duy;
    const long long gi = M->offset + (long long)(i0 + ti) * n1 + (j0 + tj);
    double o;
    if (p.stage == 0) {
      o = kv;
    } else {
      if (!isfinite(kv)) {
        const unsigned long long code =
            (unsigned long long)ctl->cur_step * 4ull + (unsigned long long)p.stage;
        atomicMin(p.fail + tk.x, code);
      }
      const double dt = ctl->dt;
      const double ui = p.uin[gi];
      if (p.stage == 1)
        o = ui + dt * kv;
      else if (p.stage == 2)
        o = 0.75 * p.un[gi] + 0.25 * (ui + dt * kv);
      else
        o = (1.0 / 3.0) * p.un[gi] + (2.0 / 3.0) * (ui + dt * kv);
    }
    p.out[gi] = o;
    lmax = fabs(o);
  }
  if (p.track_max) {
    lmax = warp_max(lmax);
    if ((tid & 31) == 0) {
      atomicMax(p.amax_out + tk.x, (unsigned long long)__double_as_longlong(lmax));
    }
  }
  if (p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

#if SGWG_FAST
// ---------------------------------------------------------------------------
// fast 2D stage: sliding-window reconstructions with shared smoothness terms
// ---------------------------------------------------------------------------
// With D(j) = f_{j-1} - 2 f_j + f_{j+1} and d(j) = f_j - f_{j-1}, the
// positive reconstruction at x_{i+1/2} (weno.hpp:60-72) is exactly
//   f_i + sum_r w_r c_r / (6 sum_r w_r),
//   c_0 = 2D(i-1) + 3d(i),  c_1 = -D(i) + 3d(i+1),  c_2 = -D(i+1) + 3d(i+1),
//   4(eps+b_0) = (2d(i)+D(i-1))^2 + K(i-1),  4(eps+b_1) = (d(i)+d(i+1))^2 + K(i),
//   4(eps+b_2) = (D(i+1)-2d(i+1))^2 + K(i+1),   K(j) = 13/3 D(j)^2 + 4 eps,
//   w_r ~ (1, 6, 3)_r * prod_{s != r} (4(eps+b_s))^2,
// and the negative one is its mirror about x_{i+1/2}.  D, d and K of a point
// are shared by the three interfaces that see it, so a thread that slides
// along RUN consecutive interfaces computes them once.  One reciprocal per
// reconstruction (rcp.approx + Newton).  Rounding differs from the reference
// at the 1e-16 level; the parity bar for this build is 1e-10.

// NEWTON: two Newton steps (4 DFMA) instead of one third-order step (3 DFMA) -- measured
// faster in the Burgers stage kernel of large families (S2 evolve 25.8 vs 27.3 ms), slower
// everywhere else (C2 persistent 34.3 vs 33.5 ms, C3 144.3 vs 143.3 ms, the C5 planes, the
// combination).
template <bool NEWTON = false>
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  if (NEWTON) {
    r = fma(r, fma(-x, r, 1.0), r);
    r = fma(r, fma(-x, r, 1.0), r);
    return r;
  }
  // one third-order step from the ~2^-20 seed: r (1 + e + e^2), e = 1 - x r (error e^3)
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// generic role form: A,B,C = D at the three substencil centres, a,b = the two
// first differences, fc = centre value; returns the reconstruction.
template <bool LINEAR, bool NEWTON = false>
__device__ __forceinline__ double recon_roles(double fc, double A, double B, double C, double KA,
                                              double KB, double KC, double a, double b) {
  const double g0 = fma(2.0, a, A);
  const double c0 = fma(2.0, g0, -a);  // 2A + 3a
  const double c1 = fma(3.0, b, -B);
  const double c2 = fma(3.0, b, -C);
  if (LINEAR) return fc + kSixth * fma(0.1, c0, fma(0.6, c1, 0.3 * c2));
  const double g1 = a + b;
  const double g2 = fma(-2.0, b, C);
  const double e0 = fma(g0, g0, KA), e1 = fma(g1, g1, KB), e2 = fma(g2, g2, KC);
  const double q0 = e0 * e0, q1 = e1 * e1, q2 = e2 * e2;
  const double w0 = q1 * q2;
  const double w1 = (6.0 * q0) * q2;
  const double w2 = (3.0 * q0) * q1;
  const double num = fma(w0, c0, fma(w1, c1, w2 * c2));
  const double den = 6.0 * (w0 + w1 + w2);
  return fc + num * fast_rcp<NEWTON>(den);
}

// du = (F(i+1/2) - F(i-1/2)) / h for RUN consecutive points of one line held
// in shared memory (padded index q -> base[q * st]; the run's first point has
// padded index p0+3).  BURGERS: F = pos(fp) + neg(fm); else F = upwind recon
// of c*u (direction from the sign of c, weno.hpp:178-183).
// Not inlined: one copy of the (large, fully unrolled) line sweep serves the
// x and y sweeps of every tile shape, keeping the hot code in the i-cache.
// du[t] is written to out[t * ost] (shared memory).
template <bool BURGERS, int RUN, bool LINEAR, bool NEWTON>
__device__ SGWG_SWEEP_ATTR void sweep_run(const double* __restrict__ P,
                                          const double* __restrict__ Mv, int st, int p0,
                                          double c, double eps4, double inv_h,
                                          double* __restrict__ out, int ost) {
  // Fully unrolled sliding window: interface t has left point q = t + 2
  // (q = padded index relative to p0); D, d, K of a point are computed once and
  // reused by the three interfaces that see it.  For advection Mv == P and the
  // upwind side is selected per line.
  constexpr int NV = RUN + 6;
  const double sc = BURGERS ? 1.0 : c;
  // advection: a downwind line (c < 0, weno.hpp:178-183) is the positive
  // reconstruction of the reversed line, so only the addressing depends on
  // the direction (no per-value selects)
  const bool rev = !BURGERS && (c < 0.0);
  double fp[NV], fm[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    fp[q] = sc * P[(p0 + (rev ? NV - 1 - q : q)) * st];
    if (BURGERS) fm[q] = Mv[(p0 + q) * st];
  }
  // second differences from the first differences they share a, b with
  auto Kof = [&](double Dq) { return fma(13.0 / 3.0 * Dq, Dq, eps4); };
  double Dp[NV], Kp[NV], dp[NV], Dm[NV], Km[NV], dm[NV];
#pragma unroll
  for (int q = 1; q < NV; ++q) {
    dp[q] = fp[q] - fp[q - 1];
    if (BURGERS) dm[q] = fm[q] - fm[q - 1];
  }
#pragma unroll
  for (int q = 1; q < NV - 1; ++q) {
    // (NEWTON -- the Burgers stage kernel of large families -- keeps the direct form: with
    // both splittings' differences live first it was 8 % slower on S2)
    Dp[q] = NEWTON ? fma(-2.0, fp[q], fp[q - 1] + fp[q + 1]) : dp[q + 1] - dp[q];
    Kp[q] = Kof(Dp[q]);
    if (BURGERS) {
      Dm[q] = NEWTON ? fma(-2.0, fm[q], fm[q - 1] + fm[q + 1]) : dm[q + 1] - dm[q];
      Km[q] = Kof(Dm[q]);
    }
  }
  double fprev = 0.0;
#pragma unroll
  for (int t = 0; t <= RUN; ++t) {
    const int i = t + 2, m = t + 3;
    double F = recon_roles<LINEAR, NEWTON>(fp[i], Dp[i - 1], Dp[i], Dp[i + 1], Kp[i - 1], Kp[i],
                                           Kp[i + 1], dp[i], dp[i + 1]);
    if (BURGERS)
      F += recon_roles<LINEAR, NEWTON>(fm[m], Dm[m + 1], Dm[m], Dm[m - 1], Km[m + 1], Km[m],
                                       Km[m - 1], -dm[m + 1], -dm[m]);
    if (t > 0) {
      // reversed: step t yields the flux left of padded point RUN+3-t, so
      // du(local RUN-t) = (F_{t-1} - F_t) / h
      if (rev)
        out[(RUN - t) * ost] = (fprev - F) * inv_h;
      else
        out[(t - 1) * ost] = (F - fprev) * inv_h;
    }
    fprev = F;
  }
}

template <bool PERSIST>
__device__ __forceinline__ double ldx(const double* p) {
  return PERSIST ? __ldcg(p) : __ldg(p);
}

// run length of the fast 2D sweeps: 8 points per thread -> 512 threads per
// 2048-point tile.  (4 -> 1024 threads at <= 64 registers was measured slower:
// spills plus 25% redundant interfaces outweigh the doubled warp count.)
#ifndef SGWG_FAST_RUN
#define SGWG_FAST_RUN 8
#endif
constexpr int kFastRun = SGWG_FAST_RUN;
constexpr int kFastThreads = 2 * 2048 / kFastRun;

#ifdef SGWG_TRACE
// phase timestamps of the persistent kernel (experiment builds only)
__device__ long long sgwg_trace[4][600][5];
__device__ __forceinline__ void trace_mark(int slot, int step_stage, int ph) {
  const int b = blockIdx.x;
  const int w = (b == 0) ? 0 : (b == 40) ? 1 : (b == 80) ? 2 : (b == 120) ? 3 : -1;
  if (w >= 0 && threadIdx.x == 0 && step_stage >= 0 && step_stage < 600)
    sgwg_trace[w][step_stage][ph] = clock64();
  (void)slot;
}
#define SGWG_MARK(ss, ph) trace_mark(0, ss, ph)
#else
#define SGWG_MARK(ss, ph)
#endif

template <bool BURGERS, bool PERSIST, int TX, int TY>
__device__ __forceinline__ void stage2d_fast_body(const Stage2DParams& p, const MemberDesc* M,
                                                  int mi, int i0, int j0, double* sm) {
  constexpr int RUN = kFastRun;
  constexpr int PY = ((TY + 6) % 2 == 0) ? TY + 7 : TY + 6;  // odd pitch
  constexpr int DP = TY + 1;                                  // du pitch (odd for TY even)
  constexpr int NS = TX * TY / RUN;  // threads per sweep; x and y sweeps run concurrently
  constexpr int NT = 2 * NS;
  double* FP = sm;
  double* FM = FP + (TX + 6) * PY;
  double* DX = FM + (BURGERS ? (TX + 6) * PY : 0);
  double* DY = DX + TX * DP;
  double* cx = DY + TX * DP;
  double* cy = cx + TY;
  const int n0 = M->ext[0], n1 = M->ext[1];
  const int tid = threadIdx.x;
  if (!BURGERS) {
    for (int j = tid; j < TY; j += NT)
      cx[j] = line_coef(p.flux0, M, 0, p.space_dim, min(j0 + j, n1 - 1), p.c0, p.efield);
    for (int i = tid; i < TX; i += NT)
      cy[i] = line_coef(p.flux1, M, 1, p.space_dim, min(i0 + i, n0 - 1), p.c1, p.efield);
  }
  const double* u = p.uin + M->offset;
  const double alpha = BURGERS ? __longlong_as_double((long long)p.amax_in[mi]) : 0.0;
  const int bc0 = M->bc[0], bc1 = M->bc[1];
  // global row offset / column of tile-relative padded position a / b with the
  // boundary treatment of weno.hpp:131-136 (periodic wrap / zero ghosts), -1 =
  // zero.  Valid outputs read at most 3 points past a member edge (periodic
  // lines have n >= 6); positions further out are padding of a partial tile
  // and read as zero.  Branch-free: no modulo on the runtime extents.
  auto grow = [&](int a) -> int {
    const int gi = i0 - 3 + a;
    const int w = (gi < 0) ? gi + n0 : (gi >= n0 ? gi - n0 : gi);
    const bool z = (gi < 0 || gi >= n0) && (bc0 != 0 || gi >= n0 + 3);
    return z ? -1 : w * n1;
  };
  auto gcol = [&](int b) -> int {
    const int gj = j0 - 3 + b;
    const int w = (gj < 0) ? gj + n1 : (gj >= n1 ? gj - n1 : gj);
    const bool z = (gj < 0 || gj >= n1) && (bc1 != 0 || gj >= n1 + 3);
    return z ? -1 : w;
  };
  auto split_store = [&](int a, int b, double uj) {
    if (BURGERS) {
      const double f = 0.5 * uj * uj;              // models.hpp:194
      const double fpj = 0.5 * (f + alpha * uj);   // weno.hpp:138-140
      FP[a * PY + b] = fpj;
      FM[a * PY + b] = f - fpj;
    } else {
      FP[a * PY + b] = uj;
    }
  };
  // tile interior: NE points per thread in one column (j = tid % TY, rows
  // tid / TY + e * RS; also the epilogue's points and u_in), then the 3-wide
  // halos of the two axes; all loads issued before any use
  constexpr int NE = TX * TY / NT;
  constexpr int RS = NT / TY;  // row step of a thread's interior points
  static_assert(NT % TY == 0, "tile width must divide the thread count");
  constexpr int NHR = 6 * TY, NH = 6 * (TX + TY);
  constexpr int NHL = (NH + NT - 1) / NT;
  const int tj = tid % TY, tr = tid / TY;
  const int ccol = gcol(tj + 3);
  double vin[NE], pre_n[NE], vh[NHL];
  int ih[NHL];
  // resident tile (persistent launch, one tile per CTA): the tile's own stage
  // input and u^n stay in shared memory between stages; only halos and
  // out-of-member padding come from L2
  double* UC = cy + TX;
  double* UN = UC + TX * TY;
  const bool resident = PERSIST && p.resident;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int q = tid + e * NT, ti = tr + e * RS;
    const bool inside = (i0 + ti < n0) && (j0 + tj < n1);
    if (resident && !p.resident_load && inside) {
      vin[e] = UC[q];
      pre_n[e] = UN[q];
    } else {
      const int ro = grow(ti + 3);
      const bool ok = ro >= 0 && ccol >= 0;
      const int g = ro + ccol;
      vin[e] = ok ? ldx<PERSIST>(u + g) : 0.0;
      pre_n[e] = (p.stage > 1 && ok) ? ldx<PERSIST>(p.un + M->offset + g) : 0.0;
      if (resident && inside) {
        UC[q] = vin[e];
        UN[q] = (p.stage == 1) ? vin[e] : pre_n[e];
      }
    }
  }
#pragma unroll
  for (int e = 0; e < NHL; ++e) {
    const int h = tid + e * NT;
    int a, b;
    if (h < NHR) {  // 3 rows above / below: (r6, column), columns fastest
      const int r6 = h / TY;
      a = (r6 < 3) ? r6 : TX + r6;
      b = h % TY + 3;
    } else {  // 3 columns left / right: (row, c6), c6 fastest
      const int h2 = h - NHR, c6 = h2 % 6;
      a = h2 / 6 + 3;
      b = (c6 < 3) ? c6 : TY + c6;
    }
    const int ro = (h < NH) ? grow(a) : -1, co = gcol(b);
    ih[e] = (h < NH) ? a * PY + b : -1;
    vh[e] = (ro >= 0 && co >= 0) ? ldx<PERSIST>(u + ro + co) : 0.0;
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) split_store(tr + e * RS + 3, tj + 3, vin[e]);
#pragma unroll
  for (int e = 0; e < NHL; ++e)
    if (ih[e] >= 0) {
      const double uj = vh[e];
      if (BURGERS) {
        const double f = 0.5 * uj * uj;
        const double fpj = 0.5 * (f + alpha * uj);
        FP[ih[e]] = fpj;
        FM[ih[e]] = f - fpj;
      } else {
        FP[ih[e]] = uj;
      }
    }
  __syncthreads();
  if (PERSIST) SGWG_MARK(p.trace_ss, 1);
  const double eps4 = 4.0 * p.eps;
  // Arithmetic form of the reconstructions (fast_rcp / second differences): a property of
  // the FAMILY (p.newton: Burgers families too large for the persistent kernel), not of the
  // kernel -- the stage kernel and the persistent kernel of one family stay bitwise equal
  // (a sharded small family runs the stage kernel: option B compares it with the
  // unsharded run).
  const bool nw = BURGERS && !PERSIST && p.newton;
  if (tid < NS) {  // x-sweep warps: thread = (column j, run of RUN rows)
    const int j = tid % TY, r = tid / TY;
    const double c = BURGERS ? 0.0 : cx[j];
    const double* P = FP + j + 3;
    const double* Mv = (BURGERS ? FM : FP) + j + 3;
    double* o = DX + r * RUN * DP + j;
    if (p.linear) {
      if (nw)
        sweep_run<BURGERS, RUN, true, true>(P, Mv, PY, r * RUN, c, eps4, M->inv_h[0], o, DP);
      else
        sweep_run<BURGERS, RUN, true, false>(P, Mv, PY, r * RUN, c, eps4, M->inv_h[0], o, DP);
    } else {
      if (nw)
        sweep_run<BURGERS, RUN, false, true>(P, Mv, PY, r * RUN, c, eps4, M->inv_h[0], o, DP);
      else
        sweep_run<BURGERS, RUN, false, false>(P, Mv, PY, r * RUN, c, eps4, M->inv_h[0], o, DP);
    }
  } else {  // y-sweep warps: thread = (row i, run of RUN columns)
    const int i = (tid - NS) % TX, r = (tid - NS) / TX;
    const double c = BURGERS ? 0.0 : cy[i];
    const double* P = FP + (i + 3) * PY;
    const double* Mv = (BURGERS ? FM : FP) + (i + 3) * PY;
    double* o = DY + i * DP + r * RUN;
    if (p.linear) {
      if (nw)
        sweep_run<BURGERS, RUN, true, true>(P, Mv, 1, r * RUN, c, eps4, M->inv_h[1], o, 1);
      else
        sweep_run<BURGERS, RUN, true, false>(P, Mv, 1, r * RUN, c, eps4, M->inv_h[1], o, 1);
    } else {
      if (nw)
        sweep_run<BURGERS, RUN, false, true>(P, Mv, 1, r * RUN, c, eps4, M->inv_h[1], o, 1);
      else
        sweep_run<BURGERS, RUN, false, false>(P, Mv, 1, r * RUN, c, eps4, M->inv_h[1], o, 1);
    }
  }
  __syncthreads();
  if (PERSIST) SGWG_MARK(p.trace_ss, 2);
  // epilogue: k = (0 - du_x) - du_y, RK stage, coalesced along j
  // max|out| as the u64 bit pattern (non-negative doubles order as integers)
  unsigned long long lmax = 0ull;
  const StepCtl* ctl = p.ctl;
  const double dt = PERSIST ? p.dt_value : ((ctl != nullptr) ? ctl->dt : 0.0);
  double* outp = p.out + M->offset + (long long)(i0 + tr) * n1 + (j0 + tj);
  const bool colok = j0 + tj < n1;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int ti = tr + e * RS;
    if (!colok || i0 + ti >= n0) continue;
    const double kv = (0.0 - DX[ti * DP + tj]) - DY[ti * DP + tj];
    double o;
    if (p.stage == 0) {
      o = kv;
    } else {
      if (!isfinite(kv)) {
        const unsigned long long cs = PERSIST ? p.cur_step : (unsigned long long)ctl->cur_step;
        atomicMin(p.fail + mi, cs * 4ull + (unsigned long long)p.stage);
      }
      const double ui = vin[e];
      if (p.stage == 1)
        o = fma(dt, kv, ui);
      else if (p.stage == 2)
        o = fma(0.75, pre_n[e], 0.25 * fma(dt, kv, ui));
      else
        o = fma(1.0 / 3.0, pre_n[e], (2.0 / 3.0) * fma(dt, kv, ui));
    }
    outp[(long long)e * RS * n1] = o;
    if (resident) {  // next stage's input (and u^{n+1} after stage 3) stay on chip
      const int q = tid + e * NT;
      UC[q] = o;
      if (p.stage == 3) UN[q] = o;
    }
    const unsigned long long ob = (unsigned long long)__double_as_longlong(fabs(o));
    lmax = (ob > lmax) ? ob : lmax;
  }
  if (p.track_max) {  // one atomic per CTA (max is exact in any order)
    __shared__ unsigned long long wmax[kFastThreads / 32];
    // exact u64 warp max from two 32-bit reductions (high word, then the low
    // word among the lanes holding the maximal high word)
    const unsigned hi = (unsigned)(lmax >> 32);
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? (unsigned)lmax : 0u);
    if ((tid & 31) == 0) wmax[tid >> 5] = ((unsigned long long)mh << 32) | ml;
    __syncthreads();
    if (tid == 0) {
      unsigned long long m = 0ull;
      for (int w = 0; w < NT / 32; ++w) m = (wmax[w] > m) ? wmax[w] : m;
      atomicMax(p.amax_out + mi, m);
    }
  }
}

template <bool BURGERS, bool PERSIST>
__device__ __forceinline__ void tile_body(const Stage2DParams& p, const MemberDesc* M, int4 tk,
                                          double* sm) {
  switch (tk.w) {  // tile shape (TX, TY), TX*TY = 2048, 512 threads (x and y sweep warps)
    case 0: stage2d_fast_body<BURGERS, PERSIST, 32, 64>(p, M, tk.x, tk.y, tk.z, sm); break;
    case 1: stage2d_fast_body<BURGERS, PERSIST, 64, 32>(p, M, tk.x, tk.y, tk.z, sm); break;
    case 2: stage2d_fast_body<BURGERS, PERSIST, 16, 128>(p, M, tk.x, tk.y, tk.z, sm); break;
    default: stage2d_fast_body<BURGERS, PERSIST, 128, 16>(p, M, tk.x, tk.y, tk.z, sm); break;
  }
}

// half-size tiles (1024 points, 256 threads): two CTAs per SM, so one CTA's
// staging / epilogue overlaps the other's sweeps (large families; the
// 2048-point tiles above stay for the persistent small-family kernel)
template <bool BURGERS, bool PERSIST = false>
__device__ __forceinline__ void tile_body_half(const Stage2DParams& p, const MemberDesc* M,
                                               int4 tk, double* sm) {
  switch (tk.w) {  // TX*TY = 1024, 256 threads
    case 4: stage2d_fast_body<BURGERS, PERSIST, 32, 32>(p, M, tk.x, tk.y, tk.z, sm); break;
    case 5: stage2d_fast_body<BURGERS, PERSIST, 16, 64>(p, M, tk.x, tk.y, tk.z, sm); break;
    case 6: stage2d_fast_body<BURGERS, PERSIST, 64, 16>(p, M, tk.x, tk.y, tk.z, sm); break;
    case 7: stage2d_fast_body<BURGERS, PERSIST, 8, 128>(p, M, tk.x, tk.y, tk.z, sm); break;
    default: stage2d_fast_body<BURGERS, PERSIST, 128, 8>(p, M, tk.x, tk.y, tk.z, sm); break;
  }
}
constexpr int kHalfThreads = kFastThreads / 2;

// quarter-size tiles (512 points, 128 threads): four CTAs per SM
template <bool BURGERS, bool PERSIST = false>
__device__ __forceinline__ void tile_body_quarter(const Stage2DParams& p, const MemberDesc* M,
                                                  int4 tk, double* sm) {
  switch (tk.w) {  // TX*TY = 512, 128 threads
    case 8: stage2d_fast_body<BURGERS, PERSIST, 16, 32>(p, M, tk.x, tk.y, tk.z, sm); break;
    case 9: stage2d_fast_body<BURGERS, PERSIST, 32, 16>(p, M, tk.x, tk.y, tk.z, sm); break;
    case 10: stage2d_fast_body<BURGERS, PERSIST, 8, 64>(p, M, tk.x, tk.y, tk.z, sm); break;
    default: stage2d_fast_body<BURGERS, PERSIST, 64, 8>(p, M, tk.x, tk.y, tk.z, sm); break;
  }
}
constexpr int kQuarterThreads = kFastThreads / 4;

template <bool BURGERS>
__global__ void __launch_bounds__(kQuarterThreads, 4)
    stage2d_quarter_kernel(const Stage2DParams p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  const int4 tk = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  extern __shared__ double sm[];
  if (p.amax_zero != nullptr && blockIdx.x == 0)
    for (int i = threadIdx.x; i < p.nmembers; i += blockDim.x) p.amax_zero[i] = 0ull;
  tile_body_quarter<BURGERS>(p, M, tk, sm);
  if (p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

template <bool BURGERS, bool HALF>
__global__ void __launch_bounds__(HALF ? kHalfThreads : kFastThreads, HALF ? 2 : 1)
    stage2d_fast_kernel(const Stage2DParams p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  const int4 tk = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  extern __shared__ double sm[];
  if (p.amax_zero != nullptr && blockIdx.x == 0)
    for (int i = threadIdx.x; i < p.nmembers; i += blockDim.x) p.amax_zero[i] = 0ull;
  if (HALF)
    tile_body_half<BURGERS>(p, M, tk, sm);
  else
    tile_body<BURGERS, false>(p, M, tk, sm);
  if (p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

// ---------------------------------------------------------------------------
// fast 3D stage (advection / kinetic transport): all three sweeps in one launch
// ---------------------------------------------------------------------------
// A CTA owns a TX x TY x TZ = 2048-point tile, staged with 3-point halos on
// the six faces (padded box, odd z pitch); three 256-thread warp groups run the
// x, y and z sweeps concurrently (runs of 8 points), each writing its du to
// shared memory; the epilogue forms k = ((0 - du_x) - du_y) - du_z in the
// reference's order and applies the RK stage.  <= 85 registers (768 threads).
template <int TX, int TY, int TZ>
__device__ __forceinline__ void stage3d_fast_body(const Stage2DParams& p, const MemberDesc* M,
                                                  int mi, int i0, int j0, int l0, double* sm) {
  constexpr int RUN = 8;
  constexpr int PZ = ((TZ + 6) % 2 == 0) ? TZ + 7 : TZ + 6;  // odd pitches
  constexpr int PY = TY + 6;
  constexpr int BOX = (TX + 6) * PY * PZ;
  constexpr int NPTS = TX * TY * TZ;
  constexpr int NS = NPTS / RUN;  // threads per sweep
  constexpr int NT = 3 * NS;
  constexpr int DZP = TZ + 1;     // du arrays: (i*TY + j)*DZP + l, odd pitch for the z-sweep
  constexpr int DN = TX * TY * DZP;
  double* U = sm;                 // padded box (u, times the line coefficient in the sweep)
  double* DX = U + BOX;
  double* DY = DX + DN;
  double* DZ = DY + DN;
  double* cxs = DZ + DN;          // per (j, l) x-line coefficient
  double* cys = cxs + TY * TZ;    // per (i, l)
  double* czs = cys + TX * TZ;    // per (i, j)
  const int n0 = M->ext[0], n1 = M->ext[1], n2 = M->ext[2];
  const int tid = threadIdx.x;
  for (int q = tid; q < TY * TZ; q += NT)
    cxs[q] = line_coef(p.flux0, M, 0, p.space_dim, 0, p.c0, p.efield);
  for (int q = tid; q < TX * TZ; q += NT)
    cys[q] = line_coef(p.flux1, M, 1, p.space_dim, 0, p.c1, p.efield);
  for (int q = tid; q < TX * TY; q += NT)
    czs[q] = line_coef(p.flux2, M, 2, p.space_dim, 0, p.c2, p.efield);
  const double* u = p.uin + M->offset;
  auto gindex = [&](int a, int b, int c) -> int {
    int gi = i0 - 3 + a, gj = j0 - 3 + b, gl = l0 - 3 + c;
    if (gi < 0 || gi >= n0) {
      if (M->bc[0] != 0) return -1;
      gi %= n0;
      if (gi < 0) gi += n0;
    }
    if (gj < 0 || gj >= n1) {
      if (M->bc[1] != 0) return -1;
      gj %= n1;
      if (gj < 0) gj += n1;
    }
    if (gl < 0 || gl >= n2) {
      if (M->bc[2] != 0) return -1;
      gl %= n2;
      if (gl < 0) gl += n2;
    }
    return (gi * n1 + gj) * n2 + gl;
  };
  // interior (also the epilogue's u_in), then the six 3-wide faces
  constexpr int NE = (NPTS + NT - 1) / NT;
  double vin[NE], pre_n[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int q = tid + e * NT;
    vin[e] = 0.0;
    pre_n[e] = 0.0;
    if (q < NPTS) {
      const int a = q / (TY * TZ), b = (q / TZ) % TY, c = q % TZ;
      const int g = gindex(a + 3, b + 3, c + 3);
      vin[e] = (g >= 0) ? __ldg(u + g) : 0.0;
      if (p.stage > 1 && g >= 0) pre_n[e] = __ldg(p.un + M->offset + g);
    }
  }
  constexpr int FX = 6 * TY * TZ, FY = 6 * TX * TZ, FZ = 6 * TX * TY;
  constexpr int NH = FX + FY + FZ;
  constexpr int NHL = (NH + NT - 1) / NT;
  double vh[NHL];
  int ih[NHL];
#pragma unroll
  for (int e = 0; e < NHL; ++e) {
    const int h = tid + e * NT;
    int a = 0, b = 0, c = 0;
    if (h < FX) {
      const int r6 = h / (TY * TZ), rem = h % (TY * TZ);
      a = (r6 < 3) ? r6 : TX + r6;
      b = rem / TZ + 3;
      c = rem % TZ + 3;
    } else if (h < FX + FY) {
      const int h2 = h - FX, r6 = h2 / (TX * TZ), rem = h2 % (TX * TZ);
      b = (r6 < 3) ? r6 : TY + r6;
      a = rem / TZ + 3;
      c = rem % TZ + 3;
    } else {
      const int h3 = h - FX - FY, r6 = h3 / (TX * TY), rem = h3 % (TX * TY);
      c = (r6 < 3) ? r6 : TZ + r6;
      a = rem / TY + 3;
      b = rem % TY + 3;
    }
    const bool ok = h < NH;
    ih[e] = ok ? (a * PY + b) * PZ + c : -1;
    const int g = ok ? gindex(a, b, c) : -1;
    vh[e] = (g >= 0) ? __ldg(u + g) : 0.0;
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int q = tid + e * NT;
    if (q < NPTS) {
      const int a = q / (TY * TZ), b = (q / TZ) % TY, c = q % TZ;
      U[((a + 3) * PY + (b + 3)) * PZ + (c + 3)] = vin[e];
    }
  }
#pragma unroll
  for (int e = 0; e < NHL; ++e)
    if (ih[e] >= 0) U[ih[e]] = vh[e];
  __syncthreads();
  const double eps4 = 4.0 * p.eps;
  if (tid < NS) {  // x-sweep: lines (j, l), runs along i
    const int l = tid % TZ, j = (tid / TZ) % TY, r = tid / (TY * TZ);
    const double* base = U + ((j + 3) * PZ) + (l + 3);
    double* out = DX + ((r * RUN) * TY + j) * DZP + l;
    if (p.linear)
      sweep_run<false, RUN, true>(base, base, PY * PZ, r * RUN, cxs[j * TZ + l], eps4,
                                  M->inv_h[0], out, TY * DZP);
    else
      sweep_run<false, RUN, false>(base, base, PY * PZ, r * RUN, cxs[j * TZ + l], eps4,
                                   M->inv_h[0], out, TY * DZP);
  } else if (tid < 2 * NS) {  // y-sweep: lines (i, l), runs along j
    const int t2 = tid - NS;
    const int l = t2 % TZ, i = (t2 / TZ) % TX, r = t2 / (TX * TZ);
    const double* base = U + ((i + 3) * PY) * PZ + (l + 3);
    double* out = DY + (i * TY + r * RUN) * DZP + l;
    if (p.linear)
      sweep_run<false, RUN, true>(base, base, PZ, r * RUN, cys[i * TZ + l], eps4, M->inv_h[1],
                                  out, DZP);
    else
      sweep_run<false, RUN, false>(base, base, PZ, r * RUN, cys[i * TZ + l], eps4, M->inv_h[1],
                                   out, DZP);
  } else {  // z-sweep: lines (i, j), runs along l; lanes walk j (odd z pitch)
    const int t3 = tid - 2 * NS;
    const int j = t3 % TY, i = (t3 / TY) % TX, r = t3 / (TX * TY);
    const double* base = U + ((i + 3) * PY + (j + 3)) * PZ;
    double* out = DZ + (i * TY + j) * DZP + r * RUN;
    if (p.linear)
      sweep_run<false, RUN, true>(base, base, 1, r * RUN, czs[i * TY + j], eps4, M->inv_h[2],
                                  out, 1);
    else
      sweep_run<false, RUN, false>(base, base, 1, r * RUN, czs[i * TY + j], eps4, M->inv_h[2],
                                   out, 1);
  }
  __syncthreads();
  double lmax = 0.0;
  const StepCtl* ctl = p.ctl;
  const double dt = (ctl != nullptr) ? ctl->dt : 0.0;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int q = tid + e * NT;
    if (q >= NPTS) continue;
    const int a = q / (TY * TZ), b = (q / TZ) % TY, c = q % TZ;
    if (i0 + a >= n0 || j0 + b >= n1 || l0 + c >= n2) continue;
    const int dq = (a * TY + b) * DZP + c;
    const double kv = ((0.0 - DX[dq]) - DY[dq]) - DZ[dq];
    const long long gi = M->offset + ((long long)(i0 + a) * n1 + (j0 + b)) * n2 + (l0 + c);
    double o;
    if (p.stage == 0) {
      o = kv;
    } else {
      if (!isfinite(kv)) {
        const unsigned long long code =
            (unsigned long long)ctl->cur_step * 4ull + (unsigned long long)p.stage;
        atomicMin(p.fail + mi, code);
      }
      const double ui = vin[e];
      if (p.stage == 1)
        o = fma(dt, kv, ui);
      else if (p.stage == 2)
        o = fma(0.75, pre_n[e], 0.25 * fma(dt, kv, ui));
      else
        o = fma(1.0 / 3.0, pre_n[e], (2.0 / 3.0) * fma(dt, kv, ui));
    }
    p.out[gi] = o;
    lmax = fmax(lmax, fabs(o));
  }
  (void)lmax;  // advection / kinetic: no Burgers alpha to track
}

constexpr int kStage3DThreads = 768;

__global__ void __launch_bounds__(kStage3DThreads, 1) stage3d_fast_kernel(const Stage2DParams p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  const int4 tk = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  extern __shared__ double sm[];
  const int i0 = tk.y >> 16, j0 = tk.y & 0xffff, l0 = tk.z >> 8, shape = tk.z & 0xff;
  switch (shape) {  // (TX, TY, TZ), 2048 points
    case 0: stage3d_fast_body<8, 16, 16>(p, M, tk.x, i0, j0, l0, sm); break;
    case 1: stage3d_fast_body<16, 8, 16>(p, M, tk.x, i0, j0, l0, sm); break;
    default: stage3d_fast_body<16, 16, 8>(p, M, tk.x, i0, j0, l0, sm); break;
  }
  if (p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

// Persistent, software-pipelined variant (advection): each CTA walks its
// tiles in order and stages tile k+1 with asynchronous 8-byte copies
// (cp.async, zero-filled ghosts) into the second of two padded boxes while
// the sweeps of tile k run, so the halo/interior load latency overlaps the
// fp64 work instead of preceding it.
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int TX, int TY, int TZ>
struct Box3 {
  static constexpr int PZ = ((TZ + 6) % 2 == 0) ? TZ + 7 : TZ + 6;
  static constexpr int PY = TY + 6;
  static constexpr int BOX = (TX + 6) * PY * PZ;
  static constexpr int NPTS = TX * TY * TZ;
  static constexpr int NS = NPTS / 8;
  static constexpr int NT = 3 * NS;
  static constexpr int DZP = TZ + 1;
  static constexpr int DN = TX * TY * DZP;
};
constexpr int kPipe3DBox = 7260;   // max Box3::BOX of the three tile shapes
constexpr int kPipe3DDn = 2304;    // max Box3::DN
constexpr int kPipe3DBoxH = 4620;  // 1024-point tiles (8,8,16), (8,16,8), (16,8,8)
constexpr int kPipe3DDnH = 1152;

// gindex of the padded box position (a, b, c) (weno.hpp:131-141 boundary rule)
__device__ __forceinline__ int gidx3(const MemberDesc* M, int i0, int j0, int l0, int a, int b,
                                     int c) {
  const int n0 = M->ext[0], n1 = M->ext[1], n2 = M->ext[2];
  int gi = i0 - 3 + a, gj = j0 - 3 + b, gl = l0 - 3 + c;
  if (gi < 0 || gi >= n0) {
    if (M->bc[0] != 0) return -1;
    gi = (gi < 0) ? gi + n0 : gi - n0;  // |excursion| <= 3 < n (periodic n >= 6)
  }
  if (gj < 0 || gj >= n1) {
    if (M->bc[1] != 0) return -1;
    gj = (gj < 0) ? gj + n1 : gj - n1;
  }
  if (gl < 0 || gl >= n2) {
    if (M->bc[2] != 0) return -1;
    gl = (gl < 0) ? gl + n2 : gl - n2;
  }
  return (gi * n1 + gj) * n2 + gl;
}

// one padded coordinate of a 3D box: member index (periodic wrap, |excursion|
// <= 3 < n) or -1 (zero ghost)
__device__ __forceinline__ int wrap1(int g, int n, int bc) {
  if (g >= 0 && g < n) return g;
  if (bc != 0) return -1;
  return (g < 0) ? g + n : g - n;
}

template <int TX, int TY, int TZ>
__device__ __forceinline__ void stage3d_issue(const Stage2DParams& p, const MemberDesc* M, int i0,
                                              int j0, int l0, double* U) {
  using G = Box3<TX, TY, TZ>;
  const double* u = p.uin + M->offset;
  const int tid = threadIdx.x;
  const int n0 = M->ext[0], n1 = M->ext[1], n2 = M->ext[2];
  const int s0 = n1 * n2;
  // a box inside its member (every tile of the BASELINE families): interior
  // points need no boundary rule, a face point only the rule of its face axis
  const bool full = (i0 + TX <= n0) && (j0 + TY <= n1) && (l0 + TZ <= n2);
  const int base = (i0 * n1 + j0) * n2 + l0;
#pragma unroll
  for (int e = 0; e < (G::NPTS + G::NT - 1) / G::NT; ++e) {
    const int q = tid + e * G::NT;
    if (q < G::NPTS) {
      const int a = q / (TY * TZ), b = (q / TZ) % TY, c = q % TZ;
      const int g = full ? base + a * s0 + b * n2 + c : gidx3(M, i0, j0, l0, a + 3, b + 3, c + 3);
      cp_async8(U + ((a + 3) * G::PY + (b + 3)) * G::PZ + (c + 3), u + max(g, 0), g >= 0);
    }
  }
  constexpr int FX = 6 * TY * TZ, FY = 6 * TX * TZ, FZ = 6 * TX * TY;
  const int bc0 = M->bc[0], bc1 = M->bc[1], bc2 = M->bc[2];
  for (int h = tid; h < FX + FY + FZ; h += G::NT) {
    int a, b, c, g;
    if (h < FX) {
      const int r6 = h / (TY * TZ), rem = h % (TY * TZ);
      a = (r6 < 3) ? r6 : TX + r6;
      b = rem / TZ + 3;
      c = rem % TZ + 3;
      const int gi = wrap1(i0 - 3 + a, n0, bc0);
      g = (gi >= 0) ? (gi * n1 + j0 + b - 3) * n2 + l0 + c - 3 : -1;
    } else if (h < FX + FY) {
      const int h2 = h - FX, r6 = h2 / (TX * TZ), rem = h2 % (TX * TZ);
      b = (r6 < 3) ? r6 : TY + r6;
      a = rem / TZ + 3;
      c = rem % TZ + 3;
      const int gj = wrap1(j0 - 3 + b, n1, bc1);
      g = (gj >= 0) ? ((i0 + a - 3) * n1 + gj) * n2 + l0 + c - 3 : -1;
    } else {
      const int h3 = h - FX - FY, r6 = h3 / (TX * TY), rem = h3 % (TX * TY);
      c = (r6 < 3) ? r6 : TZ + r6;
      a = rem / TY + 3;
      b = rem % TY + 3;
      const int gl = wrap1(l0 - 3 + c, n2, bc2);
      g = (gl >= 0) ? ((i0 + a - 3) * n1 + j0 + b - 3) * n2 + gl : -1;
    }
    if (!full) g = gidx3(M, i0, j0, l0, a, b, c);
    cp_async8(U + (a * G::PY + b) * G::PZ + c, u + max(g, 0), g >= 0);
  }
}

template <int TX, int TY, int TZ>
__device__ __forceinline__ void stage3d_compute(const Stage2DParams& p, const MemberDesc* M,
                                                int mi, int i0, int j0, int l0, const double* U,
                                                double* D) {
  using G = Box3<TX, TY, TZ>;
  constexpr int RUN = 8, PY = G::PY, PZ = G::PZ, NS = G::NS, DZP = G::DZP, DN = G::DN;
  double* DX = D;
  double* DY = DX + DN;
  double* DZ = DY + DN;
  const int tid = threadIdx.x;
  const double eps4 = 4.0 * p.eps;
  if (tid < NS) {  // x-sweep: lines (j, l), runs along i
    const int l = tid % TZ, j = (tid / TZ) % TY, r = tid / (TY * TZ);
    const double* base = U + ((j + 3) * PZ) + (l + 3);
    double* out = DX + ((r * RUN) * TY + j) * DZP + l;
    if (p.linear)
      sweep_run<false, RUN, true>(base, base, PY * PZ, r * RUN, p.c0, eps4, M->inv_h[0], out,
                                  TY * DZP);
    else
      sweep_run<false, RUN, false>(base, base, PY * PZ, r * RUN, p.c0, eps4, M->inv_h[0], out,
                                   TY * DZP);
  } else if (tid < 2 * NS) {  // y-sweep: lines (i, l), runs along j
    const int t2 = tid - NS;
    const int l = t2 % TZ, i = (t2 / TZ) % TX, r = t2 / (TX * TZ);
    const double* base = U + ((i + 3) * PY) * PZ + (l + 3);
    double* out = DY + (i * TY + r * RUN) * DZP + l;
    if (p.linear)
      sweep_run<false, RUN, true>(base, base, PZ, r * RUN, p.c1, eps4, M->inv_h[1], out, DZP);
    else
      sweep_run<false, RUN, false>(base, base, PZ, r * RUN, p.c1, eps4, M->inv_h[1], out, DZP);
  } else {  // z-sweep: lines (i, j), runs along l; lanes walk j (odd z pitch)
    const int t3 = tid - 2 * NS;
    const int j = t3 % TY, i = (t3 / TY) % TX, r = t3 / (TX * TY);
    const double* base = U + ((i + 3) * PY + (j + 3)) * PZ;
    double* out = DZ + (i * TY + j) * DZP + r * RUN;
    if (p.linear)
      sweep_run<false, RUN, true>(base, base, 1, r * RUN, p.c2, eps4, M->inv_h[2], out, 1);
    else
      sweep_run<false, RUN, false>(base, base, 1, r * RUN, p.c2, eps4, M->inv_h[2], out, 1);
  }
  __syncthreads();
  const StepCtl* ctl = p.ctl;
  const double dt = (ctl != nullptr) ? ctl->dt : 0.0;
  const int n0 = M->ext[0], n1 = M->ext[1], n2 = M->ext[2];
  // all u^n loads of the thread's points in flight before any use
  constexpr int NE = (G::NPTS + G::NT - 1) / G::NT;
  const double* unb = p.un + M->offset;
  double* outb = p.out + M->offset;
  int gq[NE];
  double unv[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int q = tid + e * G::NT;
    const int a = q / (TY * TZ), b = (q / TZ) % TY, c = q % TZ;
    const bool ok = q < G::NPTS && i0 + a < n0 && j0 + b < n1 && l0 + c < n2;
    gq[e] = ok ? ((i0 + a) * n1 + (j0 + b)) * n2 + (l0 + c) : -1;
    unv[e] = (ok && p.stage > 1) ? __ldg(unb + gq[e]) : 0.0;
  }
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    if (gq[e] < 0) continue;
    const int q = tid + e * G::NT;
    const int a = q / (TY * TZ), b = (q / TZ) % TY, c = q % TZ;
    const int dq = (a * TY + b) * DZP + c;
    const double kv = ((0.0 - DX[dq]) - DY[dq]) - DZ[dq];
    double o;
    if (p.stage == 0) {
      o = kv;
    } else {
      if (!isfinite(kv)) {
        const unsigned long long code =
            (unsigned long long)ctl->cur_step * 4ull + (unsigned long long)p.stage;
        atomicMin(p.fail + mi, code);
      }
      const double ui = U[((a + 3) * PY + (b + 3)) * PZ + (c + 3)];
      if (p.stage == 1)
        o = fma(dt, kv, ui);
      else if (p.stage == 2)
        o = fma(0.75, unv[e], 0.25 * fma(dt, kv, ui));
      else
        o = fma(1.0 / 3.0, unv[e], (2.0 / 3.0) * fma(dt, kv, ui));
    }
    outb[gq[e]] = o;
  }
}

__device__ __forceinline__ void stage3d_issue_any(const Stage2DParams& p, int4 tk, double* U) {
  const MemberDesc* M = p.mem + tk.x;
  const int i0 = tk.y >> 16, j0 = tk.y & 0xffff, l0 = tk.z >> 8;
  switch (tk.z & 0xff) {
    case 0: stage3d_issue<8, 16, 16>(p, M, i0, j0, l0, U); break;
    case 1: stage3d_issue<16, 8, 16>(p, M, i0, j0, l0, U); break;
    case 2: stage3d_issue<16, 16, 8>(p, M, i0, j0, l0, U); break;
    case 3: stage3d_issue<8, 8, 16>(p, M, i0, j0, l0, U); break;
    case 4: stage3d_issue<8, 16, 8>(p, M, i0, j0, l0, U); break;
    default: stage3d_issue<16, 8, 8>(p, M, i0, j0, l0, U); break;
  }
}

// Q = 1: 2048-point tiles, 768 threads, one CTA per SM; Q = 2: 1024-point
// tiles (shape codes 3..5), 384 threads, two CTAs per SM
template <int Q>
__global__ void __launch_bounds__(kStage3DThreads / Q, Q) stage3d_pipe_kernel(const Stage2DParams p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  extern __shared__ double sm[];
  constexpr int BOX = (Q == 1) ? kPipe3DBox : kPipe3DBoxH;
  double* Ub[2] = {sm, sm + BOX};
  double* D = sm + 2 * BOX;
  int t = blockIdx.x;
  if (t < p.ntiles) stage3d_issue_any(p, p.tiles[t], Ub[0]);
  cp_async_commit();
  for (int k = 0; t < p.ntiles; t += gridDim.x, ++k) {
    const int tn = t + gridDim.x;
    if (tn < p.ntiles) stage3d_issue_any(p, p.tiles[tn], Ub[(k + 1) & 1]);
    cp_async_commit();
    cp_async_wait<1>();  // tile t's copies have landed (the newest group may be in flight)
    __syncthreads();
    const int4 tk = p.tiles[t];
    const MemberDesc* M = p.mem + tk.x;
    const int i0 = tk.y >> 16, j0 = tk.y & 0xffff, l0 = tk.z >> 8;
    if (Q == 1) {
      switch (tk.z & 0xff) {
        case 0: stage3d_compute<8, 16, 16>(p, M, tk.x, i0, j0, l0, Ub[k & 1], D); break;
        case 1: stage3d_compute<16, 8, 16>(p, M, tk.x, i0, j0, l0, Ub[k & 1], D); break;
        default: stage3d_compute<16, 16, 8>(p, M, tk.x, i0, j0, l0, Ub[k & 1], D); break;
      }
    } else {
      switch (tk.z & 0xff) {
        case 3: stage3d_compute<8, 8, 16>(p, M, tk.x, i0, j0, l0, Ub[k & 1], D); break;
        case 4: stage3d_compute<8, 16, 8>(p, M, tk.x, i0, j0, l0, Ub[k & 1], D); break;
        default: stage3d_compute<16, 8, 8>(p, M, tk.x, i0, j0, l0, Ub[k & 1], D); break;
      }
    }
    __syncthreads();  // box k&1 and D are reused by the next tiles
  }
  cp_async_wait<0>();
  if (p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

// ---------------------------------------------------------------------------
// fast 4D stage (kinetic transport / advection) as two plane launches
// ---------------------------------------------------------------------------
// A 4D member splits into planes of the dimension pairs (0,1) and (2,3): for
// the kinetic models the x-lines of a fixed velocity point carry the constant
// coefficients (v_1, v_2) (models.hpp:341-344) and the v-lines of a fixed x
// point the constants (-E_1(x), -E_2(x)), so each plane is a 2D constant-speed
// advection problem.  Launch pr = 0 sweeps dims 0 and 1 of every plane and
// stores K = (0 - du_0) - du_1; launch pr = 1 sweeps dims 2 and 3, forms
// k = (K - du_2) - du_3 and applies the RK stage (and, for Vlasov-Poisson, the
// charge-density partial sums of the stage output).  A tile is nv consecutive
// planes restricted to a window, staged with 3-point halos (periodic wrap or
// zero ghosts, weno.hpp:131-141); the two sweeps run concurrently in two
// 128-thread halves over runs of 8 points (a line of 8m+1 points: m runs and a
// 1-point tail).  Compulsory traffic 16 B (pr 0) + 24..32 B (pr 1) per point.
#ifndef SGWG_PLANE_MINB
#define SGWG_PLANE_MINB 3
#endif
#ifndef SGWG_PLANE_THREADS
#define SGWG_PLANE_THREADS 256
#endif
constexpr int kPlaneThreads = SGWG_PLANE_THREADS;
constexpr int kPlaneMaxE = 8;  // tile points <= kPlaneThreads * kPlaneMaxE

// q / n for 0 <= q < 2^21, 0 < n < 2^12 via a float reciprocal (exact: the quotient
// (q + 1/2) / n is >= 1/(2n) away from an integer; float error < q 2^-23 / n)
__device__ __forceinline__ int qdiv(int q, float inv_n) {
  return (int)(((float)q + 0.5f) * inv_n);
}

struct PlaneGeom {
  int TX, TY, V;
  int RA, RB, tailA, tailB, TXr, TYr, PA, PB, DPB;
  __host__ __device__ PlaneGeom(int nv, int tx, int ty) : TX(tx), TY(ty), V(nv) {
    tailA = (TX & 7) == 1;
    tailB = (TY & 7) == 1;
    RA = tailA ? TX >> 3 : (TX + 7) >> 3;
    RB = tailB ? TY >> 3 : (TY + 7) >> 3;
    TXr = tailA ? TX : RA * 8;
    TYr = tailB ? TY : RB * 8;
    PA = TXr + 6;
    PB = (TYr + 6) | 1;  // odd pitches
    DPB = TYr | 1;
  }
  __host__ __device__ int smem_doubles() const {
    return V * PA * PB + 2 * V * TXr * DPB + 2 * kPlaneMaxV + TXr + TYr;
  }
};

template <bool LINEAR>
__device__ __forceinline__ void plane_sweeps(const PlaneGeom& G, const double* FP, double* DX,
                                             double* DY, const double* sca, const double* scb,
                                             double eps4, double inv_ha, double inv_hb) {
  constexpr int NSW = kPlaneThreads / 2;
  const int tid = threadIdx.x;
  const int plane = G.PA * G.PB;
  const float iTX = 1.0f / (float)G.TX, iTY = 1.0f / (float)G.TY, iV = 1.0f / (float)G.V;
  if (tid < NSW) {  // a-sweep: lines (v, j), runs along a; lanes walk j
    const int nit = G.V * G.TY * G.RA;
#pragma unroll 1
    for (int w = tid; w < nit; w += NSW) {
      const int r2 = qdiv(w, iTY), j = w - r2 * G.TY, r = qdiv(r2, iV), v = r2 - r * G.V;
      const double* P = FP + v * plane + j + 3;
      sweep_run<false, 8, LINEAR>(P, P, G.PB, r * 8, sca[v], eps4, inv_ha,
                                  DX + (v * G.TXr + r * 8) * G.DPB + j, G.DPB);
    }
    if (G.tailA)
#pragma unroll 1
      for (int w = tid; w < G.V * G.TY; w += NSW) {
        const int v = qdiv(w, iTY), j = w - v * G.TY;
        const double* P = FP + v * plane + j + 3;
        sweep_run<false, 1, LINEAR>(P, P, G.PB, G.TX - 1, sca[v], eps4, inv_ha,
                                    DX + (v * G.TXr + G.TX - 1) * G.DPB + j, G.DPB);
      }
  } else {  // b-sweep: lines (v, i), runs along b; lanes walk i (odd pitch)
    const int t = tid - NSW;
    const int nit = G.V * G.TX * G.RB;
#pragma unroll 1
    for (int w = t; w < nit; w += NSW) {
      const int r2 = qdiv(w, iTX), i = w - r2 * G.TX, r = qdiv(r2, iV), v = r2 - r * G.V;
      const double* P = FP + v * plane + (i + 3) * G.PB;
      sweep_run<false, 8, LINEAR>(P, P, 1, r * 8, scb[v], eps4, inv_hb,
                                  DY + (v * G.TXr + i) * G.DPB + r * 8, 1);
    }
    if (G.tailB)
#pragma unroll 1
      for (int w = t; w < G.V * G.TX; w += NSW) {
        const int v = qdiv(w, iTX), i = w - v * G.TX;
        const double* P = FP + v * plane + (i + 3) * G.PB;
        sweep_run<false, 1, LINEAR>(P, P, 1, G.TY - 1, scb[v], eps4, inv_hb,
                                    DY + (v * G.TXr + i) * G.DPB + G.TY - 1, 1);
      }
  }
}

__global__ void __launch_bounds__(kPlaneThreads, SGWG_PLANE_MINB) plane_fast_kernel(const PlaneParams p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  const PlaneTile tl = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tl.mi;
  const int a = 2 * p.pr, b = a + 1;
  const PlaneGeom G(tl.nv, tl.tx, tl.ty);
  const int na = M->ext[a], nb = M->ext[b];
  const int sa = (int)M->stride[a], sb = (int)M->stride[b];
  const int ps = (p.pr == 0) ? 1 : M->ext[2] * M->ext[3];  // plane -> memory offset
  const bool vfast = (p.pr == 0);  // consecutive planes are adjacent in memory
  const int bca = M->bc[a], bcb = M->bc[b];
  const int TX = G.TX, TY = G.TY, V = G.V;
  const int NP = V * TX * TY;
  const int plane = G.PA * G.PB;
  extern __shared__ double sm[];
  double* FP = sm;
  double* DX = FP + V * plane;
  double* DY = DX + V * G.TXr * G.DPB;
  double* sca = DY + V * G.TXr * G.DPB;
  double* scb = sca + kPlaneMaxV;
  double* WA = scb + kPlaneMaxV;  // pr = 1: trapezoid weights of the window rows / columns
  double* WB = WA + G.TXr;
  const int tid = threadIdx.x;
  if (tid < V) {  // per-plane line coefficients (line_coef)
    const int pl = tl.plane0 + tid;
    if (p.pr == 0) {  // x_j lines at velocity point pl: v_j (models.hpp:341-344)
      const int n3 = M->ext[3];
      sca[tid] = line_coef(p.flux_a, M, 0, p.space_dim, pl / n3, p.c_a, p.efield);
      scb[tid] = line_coef(p.flux_b, M, 1, p.space_dim, pl % n3, p.c_b, p.efield);
    } else {  // v_j lines at x point pl: -E_j(x)
      sca[tid] = line_coef(p.flux_a, M, 2, p.space_dim, pl, p.c_a, p.efield);
      scb[tid] = line_coef(p.flux_b, M, 3, p.space_dim, pl, p.c_b, p.efield);
    }
  }
  if (p.pr == 1 && p.rho_parts != nullptr) {  // models.hpp:64-71,240-257
    for (int i = tid; i < TX; i += kPlaneThreads) {
      const int ia = tl.i0 + i;
      WA[i] = (bca == 1 && (ia == 0 || ia == na - 1)) ? 0.5 * M->h[a] : M->h[a];
    }
    for (int j = tid; j < TY; j += kPlaneThreads) {
      const int jb = tl.j0 + j;
      WB[j] = (bcb == 1 && (jb == 0 || jb == nb - 1)) ? 0.5 * M->h[b] : M->h[b];
    }
  }
  const double* u = p.uin + M->offset;
  // tile point q -> (v, i, j): planes fastest when adjacent in memory, else j
  const float iTX = 1.0f / (float)TX, iTY = 1.0f / (float)TY, iV = 1.0f / (float)V;
  auto decode = [&](int q, int& v, int& i, int& j) {
    if (vfast) {
      const int r = qdiv(q, iV);
      v = q - r * V;
      i = qdiv(r, iTY);
      j = r - i * TY;
    } else {
      const int r = qdiv(q, iTY);
      j = q - r * TY;
      v = qdiv(r, iTX);
      i = r - v * TX;
    }
  };
  // interior: one load per point (all in flight before any use)
  const bool wholeA = (TX == na), wholeB = (TY == nb);
  double vin[kPlaneMaxE];
  int sidx[kPlaneMaxE], ij[kPlaneMaxE];
#pragma unroll
  for (int e = 0; e < kPlaneMaxE; ++e) {
    const int q = tid + e * kPlaneThreads;
    vin[e] = 0.0;
    sidx[e] = -1;
    ij[e] = 0;
    if (q < NP) {
      int v, i, j;
      decode(q, v, i, j);
      vin[e] = __ldg(u + (tl.plane0 + v) * ps + (tl.i0 + i) * sa + (tl.j0 + j) * sb);
      sidx[e] = v * plane + (i + 3) * G.PB + j + 3;
      ij[e] = (i << 16) | j;
    }
  }
  // zero ghosts of a whole zero-BC dimension (the velocity planes): one
  // vectorised clear of the staging planes instead of per-point edge tests
  const bool zA = wholeA && bca != 0, zB = wholeB && bcb != 0;
  if (zA || zB) {
    double2* z = reinterpret_cast<double2*>(FP);
    const int n2 = (V * plane + 1) / 2;  // (one spare double of DX, rewritten by the sweeps)
    for (int q = tid; q < n2; q += kPlaneThreads) z[q] = make_double2(0.0, 0.0);
    __syncthreads();
  }
  // halos along a window-split dimension: 3 rows above/below (a), 3 columns
  // left/right (b) of every plane, from L2/HBM (periodic wrap or zero ghosts)
  const int HA = wholeA ? 0 : 6 * TY, HB = wholeB ? 0 : 6 * TX;
  const int HP = HA + HB;
  const int NH = V * HP;
  if (NH > 0) {
    const float iHP = 1.0f / (float)HP;
#pragma unroll 1
    for (int h0 = tid; h0 < NH; h0 += 4 * kPlaneThreads) {
      double hv[4];
      int hs[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int h = h0 + e * kPlaneThreads;
        hv[e] = 0.0;
        hs[e] = -1;
        if (h < NH) {
          int v, hh;
          if (vfast) {
            hh = qdiv(h, iV);
            v = h - hh * V;
          } else {
            v = qdiv(h, iHP);
            hh = h - v * HP;
          }
          int ia, jb;  // padded tile coordinates
          if (hh < HA) {
            const int r6 = qdiv(hh, iTY);
            ia = (r6 < 3) ? r6 : TX + r6;
            jb = hh - r6 * TY + 3;
          } else {
            const int h2 = hh - HA, r6 = qdiv(h2, 1.0f / 6.0f), c6 = h2 - r6 * 6;
            ia = r6 + 3;
            jb = (c6 < 3) ? c6 : TY + c6;
          }
          hs[e] = v * plane + ia * G.PB + jb;
          int gi = tl.i0 - 3 + ia, gj = tl.j0 - 3 + jb;
          bool zero = false;
          if (gi < 0 || gi >= na) {
            if (bca != 0) zero = true;
            gi = (gi < 0) ? gi + na : gi - na;  // |excursion| <= 3 < n
          }
          if (gj < 0 || gj >= nb) {
            if (bcb != 0) zero = true;
            gj = (gj < 0) ? gj + nb : gj - nb;
          }
          if (!zero) hv[e] = __ldg(u + (tl.plane0 + v) * ps + gi * sa + gj * sb);
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (hs[e] >= 0) FP[hs[e]] = hv[e];
    }
  }
  // interior stores; along a whole dimension a point near an edge also fills
  // its halo copy: the periodic image (weno.hpp:131-136) or a zero ghost
  const int upA = ((bca != 0) ? -3 : TX) * G.PB, dnA = ((bca != 0) ? 3 : -TX) * G.PB;
  const int upB = (bcb != 0) ? -3 : TY, dnB = (bcb != 0) ? 3 : -TY;
#pragma unroll
  for (int e = 0; e < kPlaneMaxE; ++e) {
    if (sidx[e] < 0) continue;
    const double val = vin[e];
    const int si = sidx[e], i = ij[e] >> 16, j = ij[e] & 0xffff;
    FP[si] = val;
    if (wholeA && !zA) {  // periodic image
      if (i < 3) FP[si + upA] = val;
      if (i >= TX - 3) FP[si + dnA] = val;
    }
    if (wholeB && !zB) {
      if (j < 3) FP[si + upB] = val;
      if (j >= TY - 3) FP[si + dnB] = val;
    }
  }
  __syncthreads();
  const double eps4 = 4.0 * p.eps;
  if (p.linear)
    plane_sweeps<true>(G, FP, DX, DY, sca, scb, eps4, M->inv_h[a], M->inv_h[b]);
  else
    plane_sweeps<false>(G, FP, DX, DY, sca, scb, eps4, M->inv_h[a], M->inv_h[b]);
  __syncthreads();
  // epilogue: coalesced in the staging order; loads of a batch before use
  double* kb = p.kbuf + M->offset;
  const double dt = (ctl != nullptr) ? ctl->dt : 0.0;
  const bool moment = (p.pr == 1) && (p.rho_parts != nullptr) && (p.stage > 0);
#pragma unroll
  for (int e0 = 0; e0 < kPlaneMaxE; e0 += 4) {
    double kin[4], unv[4];
    int gq[4], pk[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int q = tid + (e0 + e) * kPlaneThreads;
      kin[e] = 0.0;
      unv[e] = 0.0;
      gq[e] = -1;
      pk[e] = 0;
      if (q < NP) {
        int v, i, j;
        decode(q, v, i, j);
        pk[e] = (v << 22) | (i << 11) | j;  // v < 32, i, j < 2048
        gq[e] = (tl.plane0 + v) * ps + (tl.i0 + i) * sa + (tl.j0 + j) * sb;
        if (p.pr == 1) {
          kin[e] = __ldg(kb + gq[e]);
          if (p.stage > 1) unv[e] = __ldg(p.un + M->offset + gq[e]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (gq[e] < 0) continue;
      const int v = pk[e] >> 22, i = (pk[e] >> 11) & 2047, j = pk[e] & 2047;
      const int dq = (v * G.TXr + i) * G.DPB + j;
      const double dx = DX[dq], dy = DY[dq];
      if (p.pr == 0) {
        kb[gq[e]] = (0.0 - dx) - dy;
        continue;
      }
      const double kv = (kin[e] - dx) - dy;
      double o;
      if (p.stage == 0) {
        o = kv;
      } else {
        if (!isfinite(kv)) {
          const unsigned long long code =
              (unsigned long long)ctl->cur_step * 4ull + (unsigned long long)p.stage;
          atomicMin(p.fail + tl.mi, code);
        }
        const double ui = FP[v * plane + (i + 3) * G.PB + j + 3];
        if (p.stage == 1)
          o = fma(dt, kv, ui);
        else if (p.stage == 2)
          o = fma(0.75, unv[e], 0.25 * fma(dt, kv, ui));
        else
          o = fma(1.0 / 3.0, unv[e], (2.0 / 3.0) * fma(dt, kv, ui));
      }
      p.out[M->offset + gq[e]] = o;
      if (moment) DX[dq] = (WA[i] * WB[j]) * o;  // trapezoid weights of the velocity block
    }
  }
  if (moment) {  // per-plane sums in a fixed order: one warp per plane
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5;
    const int di = qdiv(32, iTY), dj = 32 - di * TY;  // lane stride 32 in (i, j)
    const int i0 = qdiv(lane, iTY), j0 = lane - i0 * TY;
    for (int v = warp; v < V; v += kPlaneThreads / 32) {
      double acc = 0.0;
      const double* D = DX + v * G.TXr * G.DPB;
      for (int i = i0, j = j0; i < TX;) {
        acc += D[i * G.DPB + j];
        i += di;
        j += dj;
        if (j >= TY) {
          j -= TY;
          ++i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) p.rho_parts[(M->xoff + tl.plane0 + v) * kRhoParts + tl.part] = acc;
    }
  }
  if (p.pr == 1 && p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

// Persistent cooperative variant for small families (C1/C2/C4-sized): one
// launch runs up to `nsteps` RK steps.  Stages are separated by grid-wide
// barriers; every CTA computes the step's dt redundantly from the same
// post-barrier data (deterministic, so all CTAs agree) on its own copy of the
// step-control block, and CTA 0 publishes it.  Loads of data written by other
// CTAs in this launch go through L2 (ld.global.cg).
// Q = tile divisor: 2048 / Q-point tiles, Q CTAs of kFastThreads / Q threads per SM
template <bool BURGERS, int Q>
__global__ void __launch_bounds__(kFastThreads / Q, Q)
    evolve2d_persistent_kernel(const PersistParams pp) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  __shared__ StepCtl sctl;
  __shared__ DtParams sdt;
  if (threadIdx.x == 0) {
    sdt = *pp.base.dtp;
    const volatile unsigned long long* src = (const volatile unsigned long long*)pp.base.ctl;
    unsigned long long* dst = (unsigned long long*)&sctl;
    for (int w = 0; w < (int)(sizeof(StepCtl) / 8); ++w) dst[w] = src[w];
  }
  __syncthreads();
  const int nm = pp.base.nmembers;
  for (int step = 0; step < pp.nsteps; ++step) {
    if (threadIdx.x < 32) device_step_dt_on(sdt, &sctl, false, blockIdx.x == 0);
    __syncthreads();
    if (!sctl.active) break;  // identical decision in every CTA
    for (int s = 1; s <= 3; ++s) {
      Stage2DParams p = pp.base;
      p.stage = s;
      p.uin = (s == 1) ? pp.u : (s == 2 ? pp.A : pp.B);
      p.un = pp.u;
      p.out = (s == 1) ? pp.A : (s == 2 ? pp.B : pp.u);
      p.amax_in = pp.base.amax_in + (size_t)(s - 1) * nm;
      p.amax_out = pp.base.amax_zero + (size_t)(s % 3) * nm;
      p.dt_value = sctl.dt;
      p.cur_step = (unsigned long long)sctl.cur_step;
      p.resident = pp.base.resident && (pp.base.ntiles <= (int)gridDim.x);
      p.resident_load = (step == 0 && s == 1);
      p.trace_ss = step * 3 + (s - 1);
      SGWG_MARK(p.trace_ss, 0);
      if (BURGERS && blockIdx.x == 0)  // stage s clears the slot stage s+1 writes
        for (int i = threadIdx.x; i < nm; i += blockDim.x)
          pp.base.amax_zero[(size_t)((s + 1) % 3) * nm + i] = 0ull;
      for (int t = blockIdx.x; t < pp.base.ntiles; t += gridDim.x) {
        const int4 tk = pp.base.tiles[t];
        if (Q == 4)
          tile_body_quarter<BURGERS, true>(p, pp.base.mem + tk.x, tk, sm);
        else if (Q == 2)
          tile_body_half<BURGERS, true>(p, pp.base.mem + tk.x, tk, sm);
        else
          tile_body<BURGERS, true>(p, pp.base.mem + tk.x, tk, sm);
        if (t + (int)gridDim.x < pp.base.ntiles) __syncthreads();  // (grid.sync has one)
      }
      SGWG_MARK(p.trace_ss, 3);
      grid.sync();
      SGWG_MARK(p.trace_ss, 4);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    StepCtl* g = const_cast<StepCtl*>(pp.base.ctl);
    g->t = sctl.t;
    g->dt = sctl.dt;
    g->step = sctl.step;
    g->cur_step = sctl.cur_step;
    g->active = sctl.active;
    g->failed = sctl.failed;
  }
}

// 512-point tiles (8 x 8 x 8), one per CTA, 192 threads, four CTAs per SM: the
// staging of one CTA overlaps the others' sweeps (no software pipeline)
constexpr int kSmall3DSmem = Box3<8, 8, 8>::BOX + 3 * Box3<8, 8, 8>::DN;
__global__ void __launch_bounds__(kStage3DThreads / 4, 4) stage3d_small_kernel(const Stage2DParams p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  extern __shared__ double sm[];
  const int4 tk = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  const int i0 = tk.y >> 16, j0 = tk.y & 0xffff, l0 = tk.z >> 8;
  double* U = sm;
  double* D = sm + Box3<8, 8, 8>::BOX;
  stage3d_issue<8, 8, 8>(p, M, i0, j0, l0, U);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  stage3d_compute<8, 8, 8>(p, M, tk.x, i0, j0, l0, U, D);
  if (p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

cudaError_t launch_stage3d(const Stage2DParams& p, int nblocks, size_t smem, cudaStream_t s) {
  if (nblocks <= 0) return cudaSuccess;
  if (p.half_tiles == 2)
    return launch_k(stage3d_small_kernel, dim3(nblocks), dim3(kStage3DThreads / 4),
                    kSmall3DSmem * sizeof(double), s, p);
  const char* e = getenv("SGWG_3D_PIPE");
  if (p.half_tiles || !(e && e[0] == '0')) {  // persistent, pipelined
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    Stage2DParams q = p;
    q.ntiles = nblocks;
    if (p.half_tiles)  // 1024-point tiles, two CTAs per SM
      return launch_k(stage3d_pipe_kernel<2>, dim3(min(nblocks, 2 * sms)),
                      dim3(kStage3DThreads / 2),
                      (2 * kPipe3DBoxH + 3 * kPipe3DDnH) * sizeof(double), s, q);
    return launch_k(stage3d_pipe_kernel<1>, dim3(min(nblocks, sms)), dim3(kStage3DThreads),
                    (2 * kPipe3DBox + 3 * kPipe3DDn) * sizeof(double), s, q);
  }
  return launch_k(stage3d_fast_kernel, dim3(nblocks), dim3(kStage3DThreads), smem, s, p);
}

cudaError_t launch_plane(const PlaneParams& p, int nblocks, size_t smem, cudaStream_t s) {
  if (nblocks <= 0) return cudaSuccess;
  return launch_k(plane_fast_kernel, dim3(nblocks), dim3(kPlaneThreads), smem, s, p);
}

int plane_smem_doubles(int nv, int tx, int ty) { return PlaneGeom(nv, tx, ty).smem_doubles(); }

template <bool B>
const void* persist_fn(int q) {
  return (q == 4) ? (const void*)evolve2d_persistent_kernel<B, 4>
                  : (q == 2) ? (const void*)evolve2d_persistent_kernel<B, 2>
                             : (const void*)evolve2d_persistent_kernel<B, 1>;
}

// p.base.half_tiles: 0 = 2048-point tiles, 1 = 1024, 2 = 512
cudaError_t launch_persist2d(const PersistParams& p, int nblocks, size_t smem, cudaStream_t s) {
  void* args[] = {(void*)&p};
  const int q = 1 << p.base.half_tiles;
  const void* fn = p.base.burgers ? persist_fn<true>(q) : persist_fn<false>(q);
  return cudaLaunchCooperativeKernel(fn, nblocks, kFastThreads / q, args, smem, s);
}

int persist2d_max_blocks(int burgers, int half, size_t smem) {
  int per_sm = 0;
  const int q = 1 << half;
  const void* fn = burgers ? persist_fn<true>(q) : persist_fn<false>(q);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kFastThreads / q, smem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;
}
#endif  // SGWG_FAST

// ---------------------------------------------------------------------------
// prolongation / combination
// ---------------------------------------------------------------------------

// One point of upsample_line (interp.hpp:151-189) with OffsetTable::make
// (interp.hpp:124-146): fine index j of a line of n_src source values at
// src[base + i*stride], refinement 2^m.
// Interpolation weights of fine index j on a line refined by 2^m (r = j mod 2^m
// != 0): stencil centre i, offset t and linear weights c (OffsetTable::make,
// interp.hpp:124-146; linear_interp_weights interp.hpp:36-40).
struct InterpAt {
  int i;
  double t, c0, c1, c2;
};

__device__ __forceinline__ InterpAt interp_at(int j, int m, int mode) {
  const int f = 1 << m;
  const int r = j & (f - 1);
  int di;
  double t;
  if (mode == 1) {  // InterpMode::weno
    di = (r >= f / 2) ? 1 : 0;
    t = (double)r / f - di;
  } else {
    di = 0;
    t = (double)r / f;
  }
  InterpAt a;
  a.c0 = (t - 1.0) * (t - 2.0) / 12.0;  // interp.hpp:39 / 120-121
  a.c1 = (4.0 - t * t) / 6.0;
  a.c2 = (t + 2.0) * (t + 1.0) / 12.0;
  a.i = (j >> m) + di;
  a.t = t;
  return a;
}

// the value from the 5 stencil values s[0..4] around a.i (upsample_line,
// interp.hpp:179-187 with substencil_values interp.hpp:45-53)
__device__ __forceinline__ double interp_vals(const double* s, const InterpAt& a, int mode,
                                              double eps) {
  const double t = a.t, c0 = a.c0, c1 = a.c1, c2 = a.c2;
  const double p0 = s[0] * 0.5 * (t + 1.0) * t - s[1] * (t + 2.0) * t +
                    s[2] * 0.5 * (t + 2.0) * (t + 1.0);
  const double p1 = s[1] * 0.5 * t * (t - 1.0) - s[2] * (t + 1.0) * (t - 1.0) +
                    s[3] * 0.5 * (t + 1.0) * t;
  const double p2 = s[2] * 0.5 * (t - 1.0) * (t - 2.0) - s[3] * t * (t - 2.0) +
                    s[4] * 0.5 * t * (t - 1.0);
  if (mode == 0) return c0 * p0 + c1 * p1 + c2 * p2;
  const double b0 = (13.0 / 12.0) * sq(s[0] - 2.0 * s[1] + s[2]) +
                    0.25 * sq(s[0] - 4.0 * s[1] + 3.0 * s[2]);
  const double b1 = (13.0 / 12.0) * sq(s[1] - 2.0 * s[2] + s[3]) + 0.25 * sq(s[1] - s[3]);
  const double b2 = (13.0 / 12.0) * sq(s[2] - 2.0 * s[3] + s[4]) +
                    0.25 * sq(3.0 * s[2] - 4.0 * s[3] + s[4]);
#if SGWG_FAST
  const double q0 = sq(eps + b0), q1 = sq(eps + b1), q2 = sq(eps + b2);
  const double w0 = c0 * (q1 * q2), w1 = c1 * (q0 * q2), w2 = c2 * (q0 * q1);
  const double den = w0 + w1 + w2;
  if (den < 1.0e300)  // else: fall through to the reference form
    return fma(w0, p0, fma(w1, p1, w2 * p2)) / den;
#endif
  const double a0 = c0 / sq(eps + b0);
  const double a1 = c1 / sq(eps + b1);
  const double a2 = c2 / sq(eps + b2);
  return (a0 * p0 + a1 * p1 + a2 * p2) / (a0 + a1 + a2);
}

__device__ __forceinline__ double interp_point(const double* __restrict__ src, long long base,
                                               long long stride, int n_src, int j, int m, int bc,
                                               int mode, double eps) {
  const int f = 1 << m;
  const int r = j & (f - 1);
  if (r == 0) return src[base + (long long)((j >> m) % n_src) * stride];
  const InterpAt a = interp_at(j, m, mode);
  double s[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int ii = a.i - 2 + q;
    if (bc == 0) {
      int iw = ii % n_src;
      if (iw < 0) iw += n_src;
      s[q] = src[base + (long long)iw * stride];
    } else {
      s[q] = (ii >= 0 && ii < n_src) ? src[base + (long long)ii * stride] : 0.0;
    }
  }
  return interp_vals(s, a, mode, eps);
}

// Combined value at single finest-grid points (cut planes, probes): for each
// member, prolong restricted to the point -- the dimension-by-dimension
// interpolation (interp.hpp:217-244) evaluated recursively on the 5^k source
// values it depends on, with the same arithmetic as upsample_kernel /
// final_kernel, so a point equals the same point of the full combination --
// then acc = acc + c*P(u) in member order (combine.hpp:113-120).
struct EvalDim {
  int copy;  // 1: the point's source index along this dimension is i (no interpolation)
  int i, n, bc;
  long long stride;
  InterpAt a;
};

template <int K>
struct EvalRec {
  static __device__ double go(const double* u, const EvalDim* D, long long off, int mode,
                              double eps) {
    const EvalDim& e = D[K];
    if (e.copy) return EvalRec<K - 1>::go(u, D, off + (long long)e.i * e.stride, mode, eps);
    double s[5];
    for (int q = 0; q < 5; ++q) {
      int ii = e.a.i - 2 + q;
      if (e.bc == 0) {
        ii %= e.n;
        if (ii < 0) ii += e.n;
      } else if (ii < 0 || ii >= e.n) {
        s[q] = 0.0;
        continue;
      }
      s[q] = EvalRec<K - 1>::go(u, D, off + (long long)ii * e.stride, mode, eps);
    }
    return interp_vals(s, e.a, mode, eps);
  }
};
template <>
struct EvalRec<-1> {
  static __device__ double go(const double* u, const EvalDim*, long long off, int, double) {
    return u[off];
  }
};

__global__ void __launch_bounds__(128) eval_points_kernel(const EvalParams p) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= p.npts) return;
  const int d = p.d;
  int j[kMaxD];
  for (int k = 0; k < d; ++k) j[k] = p.idx[q * d + k];
  double acc = 0.0;
  for (int mi = 0; mi < p.nm; ++mi) {
    const MemberDesc* M = p.mem + mi;
    EvalDim D[kMaxD];
    for (int k = 0; k < d; ++k) {
      const int m = p.nl - M->level[k];
      EvalDim& e = D[k];
      e.n = M->ext[k];
      e.bc = M->bc[k];
      e.stride = M->stride[k];
      e.copy = 1;
      if (m == 0) {
        e.i = j[k];
      } else if ((j[k] & ((1 << m) - 1)) == 0) {
        e.i = (j[k] >> m) % e.n;
      } else {
        e.copy = 0;
        e.a = interp_at(j[k], m, p.mode);
      }
    }
    const double* u = p.u + M->offset;
    double v;
    switch (d) {
      case 1: v = EvalRec<0>::go(u, D, 0, p.mode, p.eps); break;
      case 2: v = EvalRec<1>::go(u, D, 0, p.mode, p.eps); break;
      case 3: v = EvalRec<2>::go(u, D, 0, p.mode, p.eps); break;
      default: v = EvalRec<3>::go(u, D, 0, p.mode, p.eps); break;
    }
    acc = acc + p.coef[mi] * v;  // combine.hpp:119
  }
  p.out[q] = acc;
}

cudaError_t launch_eval_points(const EvalParams& p, cudaStream_t s) {
  if (p.npts <= 0) return cudaSuccess;
  eval_points_kernel<<<(unsigned)((p.npts + 127) / 128), 128, 0, s>>>(p);
  return cudaGetLastError();
}

// dimension k of prolong for a batch of members: dst has finest extent along
// k, src the member's current extents (finest for dims < k).
__global__ void __launch_bounds__(256) upsample_kernel(const UpsampleParams p) {
  pdl_wait();
  const int2 tk = p.tasks[blockIdx.x];
  const int slot = tk.x;
  const int mi = p.slot_member[slot];
  const MemberDesc* M = p.mem + mi;
  const int k = p.kdim;
  const int* ext = p.slot_ext + 4 * slot;
  long long inner = 1;
  for (int q = k + 1; q < 4; ++q) inner *= ext[q];
  const int n_src = ext[k];
  const int n_dst = p.fine_ext;
  const int m = p.nl - M->level[k];
  const double* src = p.src[slot];
  double* dst = p.dst[slot];
  const long long ndst = p.slot_n[slot];
  const long long start = (long long)tk.y * p.chunk;
  const long long end = min(start + (long long)p.chunk, ndst);
  for (long long q = start + threadIdx.x; q < end; q += blockDim.x) {
    const long long o = q / ((long long)n_dst * inner);
    const long long rem = q - o * (long long)n_dst * inner;
    const int jl = (int)(rem / inner);  // local row (slab of dimension 0: + jrow0)
    const long long i = rem - (long long)jl * inner;
    const long long base = o * (long long)n_src * inner + i;
    dst[q] = interp_point(src, base, inner, n_src, jl + p.jrow0, m, p.bc, p.mode, p.eps);
  }
}

// last dimension of prolong fused with acc += c*p over members in sorted order.
__global__ void __launch_bounds__(256) final_kernel(const FinalParams p) {
  pdl_wait();
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long first = p.row0 * (long long)p.fine_last;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < p.nfine; q += stride) {
    // sources are local to this launch's rows: q indexes them, first + q the grid
    const long long o = q / p.fine_last;
    const int j = (int)(q - o * p.fine_last);
    (void)first;
    double acc = 0.0;
    for (int mi = 0; mi < p.nm; ++mi) {
      const int m = p.mrefine[mi];
      const double* src = p.src[mi];
      double v;
      if (m == 0) {
        v = src[q];
      } else {
        const int n_src = p.msrc_ext[mi];
        v = interp_point(src, o * (long long)n_src, 1, n_src, j, m, p.bc_last, p.mode, p.eps);
      }
      if (p.assign)
        acc = v;
      else
        acc = acc + p.coef[mi] * v;  // combine.hpp:119
    }
    p.out[q] = acc;
  }
}

#if SGWG_FAST
// ---------------------------------------------------------------------------
// Fast final pass of the combination (last dimension of prolong fused with
// acc += c p over members, combine.hpp:113-120 / interp.hpp:151-189).
// A thread owns 8 consecutive fine points of one finest row; a warp takes the
// same 8-point chunk of 32 rows, so the refinement phase of the chunk (which
// fine points are copies, which stencil centre and offset t each uses) is a
// compile-time property of the instantiation <M, PH> (2^M refinement, chunk
// phase PH = (8 c mod 2^M) / 8).  Per stencil centre the smoothness
// indicators are computed once and the three nonlinear weights are put over a
// common denominator; the linear weights C_k(t) and substencil coefficients
// are literals.  ~24 fp64 operations per interpolated fine point.
// ---------------------------------------------------------------------------
template <int M, int PH, int MODE>
__device__ __forceinline__ void final_chunk(const double* __restrict__ line, long long st, int n_src,
                                            int bc, int ib, double coef, double eps, double* acc) {
  constexpr int F = 1 << M;
  constexpr int W0 = 8 * PH;  // offset of the chunk's first fine point within its block
  // window offsets (relative to ib) of every source value the chunk reads
  constexpr int OMIN = -2;
  constexpr int OMAX = ((W0 + 7) >> M) + 1 + 2;
  constexpr int NW = OMAX - OMIN + 1;
  double s[NW];
#pragma unroll
  for (int o = 0; o < NW; ++o) {
    int q = ib + OMIN + o;
    if (q < 0 || q >= n_src) {
      if (bc == 0) {
        q = (q < 0) ? q + n_src : q - n_src;
        s[o] = __ldg(line + q * st);
      } else {
        s[o] = 0.0;
      }
    } else {
      s[o] = __ldg(line + q * st);
    }
  }
  // per stencil centre (window index c - OMIN): Q_k = prod_{l != k} (eps + b_l)^2
  constexpr int NC = ((W0 + 7) >> M) + 2;
  double Q0[NC], Q1[NC], Q2[NC];
  if (MODE == 1) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int z = c - OMIN;
      const double s0 = s[z - 2], s1 = s[z - 1], s2 = s[z], s3 = s[z + 1], s4 = s[z + 2];
      const double d0 = s0 - 2.0 * s1 + s2, g0 = s0 - 4.0 * s1 + 3.0 * s2;
      const double d1 = s1 - 2.0 * s2 + s3, g1 = s1 - s3;
      const double d2 = s2 - 2.0 * s3 + s4, g2 = 3.0 * s2 - 4.0 * s3 + s4;
      const double e0 = fma(13.0 / 12.0 * d0, d0, fma(0.25 * g0, g0, eps));
      const double e1 = fma(13.0 / 12.0 * d1, d1, fma(0.25 * g1, g1, eps));
      const double e2 = fma(13.0 / 12.0 * d2, d2, fma(0.25 * g2, g2, eps));
      const double q0 = e0 * e0, q1 = e1 * e1, q2 = e2 * e2;
      Q0[c] = q1 * q2;
      Q1[c] = q0 * q2;
      Q2[c] = q0 * q1;
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int w = W0 + u;
    const int r = w & (F - 1);
    const int jj = w >> M;
    if (r == 0) {  // copy: src[(j >> m) % n_src]
      acc[u] = fma(coef, s[jj - OMIN], acc[u]);
      continue;
    }
    const int di = (MODE == 1 && r >= F / 2) ? 1 : 0;
    const double t = (double)r / F - di;
    const int co = jj + di;
    const int z = co - OMIN;
    const double s0 = s[z - 2], s1 = s[z - 1], s2 = s[z], s3 = s[z + 1], s4 = s[z + 2];
    const double p0 =
        s0 * (0.5 * (t + 1.0) * t) - s1 * ((t + 2.0) * t) + s2 * (0.5 * (t + 2.0) * (t + 1.0));
    const double p1 =
        s1 * (0.5 * t * (t - 1.0)) - s2 * ((t + 1.0) * (t - 1.0)) + s3 * (0.5 * (t + 1.0) * t);
    const double p2 =
        s2 * (0.5 * (t - 1.0) * (t - 2.0)) - s3 * (t * (t - 2.0)) + s4 * (0.5 * t * (t - 1.0));
    const double c0 = (t - 1.0) * (t - 2.0) / 12.0, c1 = (4.0 - t * t) / 6.0,
                 c2 = (t + 2.0) * (t + 1.0) / 12.0;
    double v;
    if (MODE == 1) {
      const double a0 = c0 * Q0[co], a1 = c1 * Q1[co], a2 = c2 * Q2[co];
      v = fma(a0, p0, fma(a1, p1, a2 * p2)) * fast_rcp(a0 + a1 + a2);
    } else {
      v = fma(c0, p0, fma(c1, p1, c2 * p2));
    }
    acc[u] = fma(coef, v, acc[u]);
  }
}

// Chunk of 8 fine points [j0, j0 + 8) along a line refined by 2^m >= 8: every
// point lies in the source interval [ib, ib + 1), ib = j0 >> m, so the window
// is the 6 values ib-2 .. ib+3 and the stencil centre is ib or ib + 1 (WENO:
// r >= 2^m / 2, interp.hpp:124-146).  The per-offset coefficients -- the
// substencil polynomials p_k(t) as point weights and the linear weights C_k(t)
// (interp.hpp:36-53, 119-122) -- come from a constant table indexed by the
// warp-uniform (m, r), so one body serves every m in 3..7 and chunk phase
// (the per-phase instantiations of final_chunk were the final pass's
// instruction-cache stall).  The smoothness indicators of the two centres are
// computed once per chunk.
constexpr int kInterpTabMaxM = 7;
__constant__ double c_itab[2][256][12];  // [mode][(1 << m) + r]: a0..a2 b1..b3 e2..e4 c0..c2

void fill_interp_table(double* tab /* [2][256][12] */) {
  for (int mode = 0; mode < 2; ++mode)
    for (int m = 1; m <= kInterpTabMaxM; ++m) {
      const int F = 1 << m;
      for (int r = 1; r < F; ++r) {
        const int di = (mode == 1 && r >= F / 2) ? 1 : 0;
        const double t = (double)r / F - di;
        double* e = tab + ((mode * 256) + F + r) * 12;
        e[0] = 0.5 * (t + 1.0) * t;
        e[1] = -(t + 2.0) * t;
        e[2] = 0.5 * (t + 2.0) * (t + 1.0);
        e[3] = 0.5 * t * (t - 1.0);
        e[4] = -(t + 1.0) * (t - 1.0);
        e[5] = 0.5 * (t + 1.0) * t;
        e[6] = 0.5 * (t - 1.0) * (t - 2.0);
        e[7] = -t * (t - 2.0);
        e[8] = 0.5 * t * (t - 1.0);
        e[9] = (t - 1.0) * (t - 2.0) / 12.0;
        e[10] = (4.0 - t * t) / 6.0;
        e[11] = (t + 2.0) * (t + 1.0) / 12.0;
      }
    }
}

template <int MODE>
__device__ __forceinline__ void weno_q(const double* s, double eps, double& Q0, double& Q1,
                                       double& Q2) {
  const double s0 = s[0], s1 = s[1], s2 = s[2], s3 = s[3], s4 = s[4];
  const double d0 = s0 - 2.0 * s1 + s2, g0 = s0 - 4.0 * s1 + 3.0 * s2;
  const double d1 = s1 - 2.0 * s2 + s3, g1 = s1 - s3;
  const double d2 = s2 - 2.0 * s3 + s4, g2 = 3.0 * s2 - 4.0 * s3 + s4;
  const double e0 = fma(13.0 / 12.0 * d0, d0, fma(0.25 * g0, g0, eps));
  const double e1 = fma(13.0 / 12.0 * d1, d1, fma(0.25 * g1, g1, eps));
  const double e2 = fma(13.0 / 12.0 * d2, d2, fma(0.25 * g2, g2, eps));
  const double q0 = e0 * e0, q1 = e1 * e1, q2 = e2 * e2;
  Q0 = q1 * q2;
  Q1 = q0 * q2;
  Q2 = q0 * q1;
}

// the points u in [U0, U1) of the chunk with stencil values s0..s4 and weights
// Q (one centre): acc[u] += coef * P(u)
template <int MODE, int U0, int U1>
__device__ __forceinline__ void chunk_points(const double* __restrict__ tab, int j0, int F, int np,
                                             double s0, double s1, double s2, double s3, double s4,
                                             double Q0, double Q1, double Q2, double coef,
                                             double* acc) {
#pragma unroll
  for (int u = U0; u < U1; ++u) {
    if (u >= np) break;
    const int r = (j0 + u) & (F - 1);
    if (r == 0) {  // copy: src[j >> m] (the window's centre ib)
      acc[u] = fma(coef, s2, acc[u]);
      continue;
    }
    const double* e = tab + r * 12;
    const double p0 = fma(s0, e[0], fma(s1, e[1], s2 * e[2]));
    const double p1 = fma(s1, e[3], fma(s2, e[4], s3 * e[5]));
    const double p2 = fma(s2, e[6], fma(s3, e[7], s4 * e[8]));
    double v;
    if (MODE == 1) {
      const double a0 = e[9] * Q0, a1 = e[10] * Q1, a2 = e[11] * Q2;
      v = fma(a0, p0, fma(a1, p1, a2 * p2)) * fast_rcp(a0 + a1 + a2);
    } else {
      v = fma(e[9], p0, fma(e[10], p1, e[11] * p2));
    }
    acc[u] = fma(coef, v, acc[u]);
  }
}

// NP <= 8 points of the chunk are formed (line tails); acc[u] += coef * P(u).
// For m >= 4 the chunk lies in one half of its source interval, so one stencil
// centre (ib, or ib + 1 when WENO's r >= 2^m / 2) serves all 8 points; for m = 3
// points 0-3 use ib and 4-7 use ib + 1.
template <int MODE>
__device__ __forceinline__ void chunk_generic(const double* __restrict__ line, long long st,
                                              int n_src, int bc, int m, int j0, int np,
                                              double coef, double eps, double* acc) {
  const int F = 1 << m;
  const int ib = j0 >> m;
  double s[6];
#pragma unroll
  for (int o = 0; o < 6; ++o) {
    int q = ib - 2 + o;
    const bool out = (q < 0 || q >= n_src);
    if (out && bc == 0) q = (q < 0) ? q + n_src : q - n_src;
    s[o] = (out && bc != 0) ? 0.0 : __ldg(line + q * st);
  }
  const double* tab = &c_itab[MODE][F][0];
  double Q0 = 0.0, Q1 = 0.0, Q2 = 0.0;
  if (m > 3) {
    const bool hi = (MODE == 1) && (((j0 & (F - 1)) << 1) >= F);  // chunk-uniform centre
    const double s0 = hi ? s[1] : s[0], s1 = hi ? s[2] : s[1], s2 = hi ? s[3] : s[2],
                 s3 = hi ? s[4] : s[3], s4 = hi ? s[5] : s[4];
    if (MODE == 1) {
      const double w[5] = {s0, s1, s2, s3, s4};
      weno_q<MODE>(w, eps, Q0, Q1, Q2);
    }
    // r == 0 copies (j0 % F == 0) take the centre ib: hi is false there
    chunk_points<MODE, 0, 8>(tab, j0, F, np, s0, s1, s2, s3, s4, Q0, Q1, Q2, coef, acc);
  } else {
    if (MODE == 1) weno_q<MODE>(s, eps, Q0, Q1, Q2);
    chunk_points<MODE, 0, 4>(tab, j0, F, np, s[0], s[1], s[2], s[3], s[4], Q0, Q1, Q2, coef, acc);
    if (MODE == 1) {
      weno_q<MODE>(s + 1, eps, Q0, Q1, Q2);
      chunk_points<MODE, 4, 8>(tab, j0, F, np, s[1], s[2], s[3], s[4], s[5], Q0, Q1, Q2, coef,
                               acc);
    } else {
      chunk_points<MODE, 4, 8>(tab, j0, F, np, s[0], s[1], s[2], s[3], s[4], Q0, Q1, Q2, coef,
                               acc);
    }
  }
}

// chunk [j0, j0 + np) of a line refined by 2^m (1 <= m <= 7, j0 % 8 == 0)
template <int MODE>
__device__ __forceinline__ void interp_chunk(int m, int j0, int np, const double* line,
                                             long long st, int n_src, int bc, double coef,
                                             double eps, double* acc) {
  if (m >= 3) {
    chunk_generic<MODE>(line, st, n_src, bc, m, j0, np, coef, eps, acc);
  } else {
    // np < 8 only at a zero-ghost line's last point (fine extent 8k + 1): the
    // full chunk's extra points read in-range or zero windows and are discarded
    if (m == 1)
      final_chunk<1, 0, MODE>(line, st, n_src, bc, j0 >> 1, coef, eps, acc);
    else
      final_chunk<2, 0, MODE>(line, st, n_src, bc, j0 >> 2, coef, eps, acc);
  }
}

// the chunk in the reference form (interp_point), when the common-denominator
// weights overflowed (|u| >~ 1e38)
template <int MODE>
__device__ __noinline__ void final_chunk_ref(const double* const* srcs, const double* coef,
                                             const int* mref, const int* mext, int nm,
                                             int fine_last, int bc, double eps, double* out,
                                             long long row, int c) {
  for (int u = 0; u < 8; ++u) {
    const int j = 8 * c + u;
    if (j >= fine_last) break;
    double a = 0.0;
    for (int mi = 0; mi < nm; ++mi) {
      const int m = mref[mi];
      const double* src = srcs[mi];
      const double v = (m == 0) ? src[row * fine_last + j]
                                : interp_point(src, row * mext[mi], 1, mext[mi], j, m, bc, MODE,
                                               eps);
      a = fma(coef[mi], v, a);
    }
    out[row * fine_last + j] = a;
  }
}

// grid-stride over (32-row block, chunk) warp items
#ifndef SGWG_FINAL_MINB
#define SGWG_FINAL_MINB 3
#endif
template <int MODE>
__global__ void __launch_bounds__(256, SGWG_FINAL_MINB) final_fast_kernel(const FinalParams p) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int nch = (p.fine_last + 7) >> 3;  // chunks per row (the last may be partial)
  const long long rows = p.nfine / p.fine_last;
  const long long rblocks = (rows + 31) >> 5;
  const long long items = rblocks * nch;
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long it = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < items;
       it += wstride) {
    const int c = (int)(it % nch);  // warp-uniform chunk
    const long long row = (it / nch) * 32 + lane;
    if (row >= rows) continue;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    for (int mi = 0; mi < p.nm; ++mi) {
      const int m = p.mrefine[mi];
      const double cf = p.coef[mi];
      if (m == 0) {  // member at the finest level along the last dimension: copy
        const double* src = p.src[mi] + row * p.fine_last + 8 * c;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (8 * c + u < p.fine_last) acc[u] = fma(cf, __ldg(src + u), acc[u]);
        continue;
      }
      const int n_src = p.msrc_ext[mi];
      SGWG_DCHECK(m >= 1 && m <= kInterpTabMaxM && ((n_src - (p.bc_last != 0 ? 1 : 0)) << m) ==
                                                        p.fine_last - (p.bc_last != 0 ? 1 : 0),
                  "final pass refinement");
      interp_chunk<MODE>(m, 8 * c, min(8, p.fine_last - 8 * c), p.src[mi] + row * n_src, 1, n_src,
                         p.bc_last, cf, p.eps, acc);
    }
    int ex = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) ex = max(ex, __double2hiint(acc[u]) & 0x7ff00000);
    if (ex == 0x7ff00000) {  // overflowed common-denominator weights
      final_chunk_ref<MODE>(p.src, p.coef, p.mrefine, p.msrc_ext, p.nm, p.fine_last, p.bc_last,
                            p.eps, p.out, row, c);
      continue;
    }
    double* out = p.out + row * p.fine_last + 8 * c;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (8 * c + u < p.fine_last) out[u] = acc[u];
  }
}

// Fast prolongation of dimension k < d-1 (interp.hpp:217-244) for all member
// slots of a plan: a thread forms one 8-point chunk of one line along k, a
// warp the same chunk of 32 consecutive lines (consecutive inner index: the
// loads and stores of a warp are unit-stride across lanes), the chunk phase
// is warp-uniform.  Work item = (slot, chunk, 32-line block), chunk-major
// within a slot; slot found by binary search of the item prefix.
template <int MODE>
__global__ void __launch_bounds__(256) upsample_fast_kernel(const UpsampleParams p) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const long long wstride = (long long)gridDim.x * (blockDim.x >> 5);
  const int k = p.kdim;
  for (long long it = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       it < p.nitems; it += wstride) {
    int lo = 0, hi = p.nslots - 1;  // last slot with item0 <= it
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (p.slot_item0[mid] <= it) lo = mid; else hi = mid - 1;
    }
    const int slot = lo;
    const int* ext = p.slot_ext + 4 * slot;
    long long inner = 1, outer = 1;
    for (int q = 0; q < 4; ++q) {
      if (q > k) inner *= ext[q];
      if (q < k) outer *= ext[q];
    }
    const long long nlines = outer * inner;
    const long long nblk = (nlines + 31) >> 5;
    const long long local = it - p.slot_item0[slot];
    const int ci = (int)(local / nblk);
    const long long line = (local - ci * nblk) * 32 + lane;
    if (line >= nlines) continue;
    const int n_src = ext[k];
    const int ndst = (k == 0) ? p.nrows0 : p.fine_ext;      // dst extent along k
    const int jlo = (k == 0) ? p.jrow0 : 0;                 // fine index of dst row 0
    const int j0 = ((jlo >> 3) + ci) * 8;                   // chunk start (fine index)
    const int a = max(j0, jlo), b = min(j0 + 8, jlo + ndst);  // points of this slab
    const int m = p.nl - p.mem[p.slot_member[slot]].level[k];
    const long long o = line / inner, i = line - o * inner;
    const double* src = p.src[slot] + o * (long long)n_src * inner + i;
    double* dst = p.dst[slot] + (o * (long long)ndst - jlo) * inner + i;
    SGWG_DCHECK(m >= 1 && m <= kInterpTabMaxM && j0 + 8 > jlo && j0 < jlo + ndst,
                "upsample chunk outside the slab");
    SGWG_DCHECK((o + 1) * (long long)ndst * inner <= p.slot_n[slot], "upsample dst slot");
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    interp_chunk<MODE>(m, j0, 8, src, inner, n_src, p.bc, 1.0, p.eps, acc);
    int ex = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) ex = max(ex, __double2hiint(acc[u]) & 0x7ff00000);
    if (ex == 0x7ff00000) {  // overflowed common-denominator weights: reference form
      const long long base = o * (long long)n_src * inner + i;
      for (int u = 0; u < 8; ++u)
        if (j0 + u >= a && j0 + u < b)
          acc[u] = interp_point(p.src[slot], base, inner, n_src, j0 + u, m, p.bc, MODE, p.eps);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u >= a && j0 + u < b) dst[(long long)(j0 + u) * inner] = acc[u];
  }
}
#endif

// ---------------------------------------------------------------------------
// Vlasov-Maxwell field lines (vm_rhs_into, models.hpp:437-505 + SspRk3::step)
// ---------------------------------------------------------------------------
// One CTA per member.  Currents j1, j2 = sum_q w_j1/2[q] f(x2, q) over the
// velocity block in the reference's order (vm_currents, models.hpp:420-433;
// block_weights 238-257), the characteristic variables w+- = E1 +- B3 and their
// upwind WENO derivatives along the periodic x2 line (advect_derivative_line,
// weno.hpp:160-192) with speeds -1 / +1, the tendencies
//   E1' = (tp + tm)/2, B3' = (tp - tm)/2, E2' = -j2, tp/m = -dw+-/dx2 - j1,
// and the RK stage update of the three lines (timestep.hpp:93,98,103).
// Dynamic smem: 4 * nx doubles.
__device__ __forceinline__ double vm_fhat(const double* w, int n, int k, double c, double eps,
                                          int linear) {
  // fhat[k] of advect_derivative_line on the periodic line c*w (padded fp[j+3] = c*w[j mod n])
  auto fp = [&](int j) {
    int q = j % n;
    if (q < 0) q += n;
    return c * w[q];
  };
  if (c < 0.0)  // flux_neg5(&fp[k+2]): positive reconstruction of fp[k+6..k+2]
    return recon(fp(k + 3), fp(k + 2), fp(k + 1), fp(k), fp(k - 1), eps, linear);
  return recon(fp(k - 2), fp(k - 1), fp(k), fp(k + 1), fp(k + 2), eps, linear);
}

__global__ void __launch_bounds__(256) vm_fields_kernel(const VmParams p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  const int mi = blockIdx.x;
  const MemberDesc* M = p.mem + mi;
  const int nx = M->nx, n1 = M->ext[1], n2 = M->ext[2], vn = M->vn;
  extern __shared__ double vsm[];
  double* wp = vsm;
  double* wm = wp + nx;
  double* j1 = wm + nx;
  double* j2 = j1 + nx;
  const double* F = p.fin + M->xoff * 3;
  for (int ix = threadIdx.x; ix < nx; ix += blockDim.x) {
    const double* block = p.f + M->offset + (long long)ix * vn;
    double a = 0.0, b = 0.0;
    for (int i1 = 0; i1 < n1; ++i1) {
      const double xi1 = M->lower[1] + i1 * M->h[1];
      double w1 = M->h[1];
      if (M->bc[1] != 0 && (i1 == 0 || i1 == n1 - 1)) w1 *= 0.5;  // trapezoid_weights_1d
      for (int i2 = 0; i2 < n2; ++i2) {
        const double xi2 = M->lower[2] + i2 * M->h[2];
        double w2 = M->h[2];
        if (M->bc[2] != 0 && (i2 == 0 || i2 == n2 - 1)) w2 *= 0.5;
        double wq = 1.0;  // block_weights: p = 1; p *= w_1; p *= w_2
        wq *= w1;
        wq *= w2;
        const double v = block[i1 * n2 + i2];
        a += (wq * xi1) * v;
        b += (wq * xi2) * v;
      }
    }
    j1[ix] = a;
    j2[ix] = b;
    wp[ix] = F[ix] + F[2 * nx + ix];
    wm[ix] = F[ix] - F[2 * nx + ix];
  }
  __syncthreads();
  const double hx = M->h[0];
  const double dt = (ctl != nullptr) ? ctl->dt : 0.0;
  const double* U = p.fun + M->xoff * 3;
  double* O = p.fout + M->xoff * 3;
  for (int ix = threadIdx.x; ix < nx; ix += blockDim.x) {
    const int im = (ix + nx - 1) % nx;
    const double dwp = (vm_fhat(wp, nx, ix, -1.0, p.eps, p.linear) -
                        vm_fhat(wp, nx, im, -1.0, p.eps, p.linear)) / hx;
    const double dwm = (vm_fhat(wm, nx, ix, +1.0, p.eps, p.linear) -
                        vm_fhat(wm, nx, im, +1.0, p.eps, p.linear)) / hx;
    const double tp = -dwp - j1[ix];
    const double tm = -dwm - j1[ix];
    double k3[3];
    k3[0] = 0.5 * (tp + tm);  // E1
    k3[1] = -j2[ix];          // E2
    k3[2] = 0.5 * (tp - tm);  // B3
    for (int c = 0; c < 3; ++c) {
      const double kv = k3[c];
      double o;
      if (p.stage == 0) {
        o = kv;
      } else {
        if (!isfinite(kv)) {
          const unsigned long long code =
              (unsigned long long)ctl->cur_step * 4ull + (unsigned long long)p.stage;
          atomicMin(p.fail + mi, code);
        }
        const double ui = F[c * nx + ix];
        if (p.stage == 1)
          o = ui + dt * kv;
        else if (p.stage == 2)
          o = 0.75 * U[c * nx + ix] + 0.25 * (ui + dt * kv);
        else
          o = (1.0 / 3.0) * U[c * nx + ix] + (2.0 / 3.0) * (ui + dt * kv);
      }
      O[c * nx + ix] = o;
    }
  }
}

cudaError_t launch_vm_fields(const VmParams& p, int nmembers, int smem, cudaStream_t s) {
  if (nmembers <= 0) return cudaSuccess;
  return launch_k(vm_fields_kernel, dim3(nmembers), dim3(256), (size_t)smem, s, p);
}

#if SGWG_FAST
#include "plane4d.cuh"
#endif

cudaError_t configure() {
#if SGWG_FAST
  cudaError_t e0 = cudaFuncSetAttribute(stage2d_fast_kernel<true, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(stage2d_fast_kernel<false, false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(stage2d_quarter_kernel<true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(stage2d_quarter_kernel<false>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(stage2d_fast_kernel<true, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(stage2d_fast_kernel<false, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(stage3d_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            200 * 1024);
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(plane_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            200 * 1024);
  if (e0 != cudaSuccess) return e0;
  e0 = configure_plane4();
  if (e0 != cudaSuccess) return e0;
  {
    static double tab[2 * 256 * 12];
    fill_interp_table(tab);
    e0 = cudaMemcpyToSymbol(c_itab, tab, sizeof(tab));
    if (e0 != cudaSuccess) return e0;
  }
  e0 = cudaFuncSetAttribute(stage3d_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kSmall3DSmem * (int)sizeof(double));
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(stage3d_pipe_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (2 * kPipe3DBox + 3 * kPipe3DDn) * (int)sizeof(double));
  if (e0 != cudaSuccess) return e0;
  e0 = cudaFuncSetAttribute(stage3d_pipe_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (2 * kPipe3DBoxH + 3 * kPipe3DDnH) * (int)sizeof(double));
  if (e0 != cudaSuccess) return e0;
  for (int q = 1; q <= 4; q *= 2) {
    e0 = cudaFuncSetAttribute(persist_fn<true>(q), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              112 * 1024);
    if (e0 != cudaSuccess) return e0;
    e0 = cudaFuncSetAttribute(persist_fn<false>(q), cudaFuncAttributeMaxDynamicSharedMemorySize,
                              112 * 1024);
    if (e0 != cudaSuccess) return e0;
  }
#endif
  cudaError_t e = cudaFuncSetAttribute(pass_kernel<true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              160 * 1024);
}

cudaError_t launch_stage2d(const Stage2DParams& p, int nblocks, size_t smem, cudaStream_t s) {
  if (nblocks <= 0) return cudaSuccess;
#if SGWG_FAST
  if (p.half_tiles == 2) {  // four CTAs per SM
    if (p.burgers)
      return launch_k(stage2d_quarter_kernel<true>, dim3(nblocks), dim3(kQuarterThreads), smem,
                      s, p);
    return launch_k(stage2d_quarter_kernel<false>, dim3(nblocks), dim3(kQuarterThreads), smem, s,
                    p);
  }
  if (p.half_tiles) {  // two CTAs per SM
    if (p.burgers)
      return launch_k(stage2d_fast_kernel<true, true>, dim3(nblocks), dim3(kHalfThreads), smem,
                      s, p);
    return launch_k(stage2d_fast_kernel<false, true>, dim3(nblocks), dim3(kHalfThreads), smem, s,
                    p);
  }
  if (p.burgers)
    return launch_k(stage2d_fast_kernel<true, false>, dim3(nblocks), dim3(kFastThreads), smem, s,
                    p);
  else
    return launch_k(stage2d_fast_kernel<false, false>, dim3(nblocks), dim3(kFastThreads), smem,
                    s, p);
#else
  if (p.burgers)
    return launch_k(stage2d_kernel<true>, dim3(nblocks), dim3(256), smem, s, p);
  else
    return launch_k(stage2d_kernel<false>, dim3(nblocks), dim3(256), smem, s, p);
#endif
  return cudaGetLastError();
}

cudaError_t launch_pass(const PassParams& p, int nblocks, size_t smem, cudaStream_t s) {
  if (nblocks <= 0) return cudaSuccess;
  if (p.flux == kFluxBurgers)
    return launch_k(pass_kernel<true>, dim3(nblocks), dim3(kPassThreads), smem, s, p);
  else
    return launch_k(pass_kernel<false>, dim3(nblocks), dim3(kPassThreads), smem, s, p);
  return cudaGetLastError();
}

cudaError_t launch_upsample(const UpsampleParams& p, int nblocks, cudaStream_t s) {
  if (nblocks <= 0) return cudaSuccess;
#if SGWG_FAST
  if (p.nitems > 0) {  // chunked form (every member refinement of the pass <= 2^7)
    long long blocks = (p.nitems + 7) / 8;
    if (blocks > 148 * 32) blocks = 148 * 32;
    return p.mode == 1 ? launch_k(upsample_fast_kernel<1>, dim3((int)blocks), dim3(256), 0, s, p)
                       : launch_k(upsample_fast_kernel<0>, dim3((int)blocks), dim3(256), 0, s, p);
  }
#endif
  return launch_k(upsample_kernel, dim3(nblocks), dim3(256), 0, s, p);
}

cudaError_t launch_final(const FinalParams& p, cudaStream_t s) {
  if (p.nfine <= 0) return cudaSuccess;
#if SGWG_FAST
  // chunked kernel: rows of 8m (+1) fine points, refinement <= 2^5 in the last
  // dimension; else (or SGWG_FINAL_GENERIC=1) the generic one
  bool chunked = !p.assign && p.nm_host == p.nm &&
                 ((p.fine_last - (p.bc_last != 0 ? 1 : 0)) % 8 == 0) &&
                 std::getenv("SGWG_FINAL_GENERIC") == nullptr;
  for (int mi = 0; chunked && mi < p.nm_host; ++mi) chunked = p.mref_host[mi] <= kInterpTabMaxM;
  if (chunked) {
    const long long rows = p.nfine / p.fine_last;
    const long long items = ((rows + 31) / 32) * ((p.fine_last + 7) / 8);
    long long blocks = (items + 7) / 8;
    if (blocks > 148 * 32) blocks = 148 * 32;
    return p.mode == 1 ? launch_k(final_fast_kernel<1>, dim3((int)blocks), dim3(256), 0, s, p)
                       : launch_k(final_fast_kernel<0>, dim3((int)blocks), dim3(256), 0, s, p);
  }
#endif
  long long blocks = (p.nfine + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_k(final_kernel, dim3((int)blocks), dim3(256), 0, s, p);
}

}  // namespace SGWG_NS
}  // namespace sgwg
