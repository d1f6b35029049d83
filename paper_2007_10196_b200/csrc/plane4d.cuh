// plane4d.cuh -- fast-build 4D kinetic / advection stage on whole planes
// (BASELINE C5: 2D2V Vlasov-Poisson, 121 members, 12M points per stage).
// Included by kernels.cuh inside namespace sgwg::fast.
//
// A member is (x1, x2, v1, v2) row-major (grid.hpp:102-108): the velocity
// plane of an x point is contiguous (V = n3 n4 doubles), the x-plane of a
// velocity point is strided by V.  One RK stage = two launches, each over
// WHOLE planes so that no halo is ever loaded:
//
//   xpass4d_kernel  tile = the whole periodic x-plane (n1 x n2 <= 2048 points)
//                   x C consecutive velocity points (C = 2..64, X*C ~ 4096);
//                   x2 then x1 sweep (coefficients v2, v1: models.hpp:341-344)
//                   with the periodic wrap done by addressing; K = -(dx1+dx2).
//   vpass4d_kernel  tile = G consecutive x points with their whole velocity
//                   planes (one contiguous span, staged by ONE bulk copy
//                   cp.async.bulk + mbarrier); v1 and v2 sweeps (coefficient
//                   -E_j(x), models.hpp:346-349 with the Poisson field) with
//                   the zero ghosts as compile-time zeros; RK stage
//                   (timestep.hpp:86-104) + the charge density of the stage
//                   output per x point (moment_density, models.hpp:294-306).
//
// Sweeps: one thread slides a run of 8 points of a line (14-value window in
// registers, D/d/K shared by the three interfaces that see them, one
// reciprocal per reconstruction -- recon_roles).  A warp takes 32 lines at
// the same position class (first / middle / last run / tail) so the ghost
// pattern is a compile-time property of the instantiation: no per-point
// index decode, no ghost fill, no bank conflicts (lanes on consecutive
// lines: odd row pitch or unit stride).
#pragma once

#ifndef SGWG_P4_THREADS
#define SGWG_P4_THREADS 256
#endif
#ifndef SGWG_P4_MINB
#define SGWG_P4_MINB 2
#endif
constexpr int kP4Threads = SGWG_P4_THREADS;
constexpr int kP4MaxC = 64;   // velocity points per x-pass tile

#ifdef SGWG_TRACE
// experiment builds only: per-CTA phase stamps of the plane kernels
// [pass][cta][0: globaltimer start, 1..7: clock64 at marks 0..6, 8: smid, 9: globaltimer at mark 5]
constexpr int kP4TraceCtas = 8192;
__device__ long long sgwg_p4trace[2][kP4TraceCtas][10];
#define P4MARK(pass, k)                                                      \
  do {                                                                       \
    if (threadIdx.x == 0 && blockIdx.x < kP4TraceCtas) {                     \
      if ((k) == 0) {                                                        \
        long long g;                                                         \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));                \
        unsigned sid;                                                        \
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sid));                     \
        sgwg_p4trace[pass][blockIdx.x][0] = g;                               \
        sgwg_p4trace[pass][blockIdx.x][8] = sid;                             \
      }                                                                      \
      if ((k) == 5) {                                                        \
        long long g;                                                         \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));                \
        sgwg_p4trace[pass][blockIdx.x][9] = g;                               \
      }                                                                      \
      sgwg_p4trace[pass][blockIdx.x][(k) + 1] = clock64();                   \
    }                                                                        \
  } while (0)
#else
#define P4MARK(pass, k) \
  do {                  \
  } while (0)
#endif

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one bulk global -> shared copy completing on `bar` (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// du/dx of c*u (upwind WENO5-JS, advect_derivative_line weno.hpp:160-192) for
// RUN consecutive points of one line.  P: the window's first value (physical
// point 8r - 3 of the line), st: smem stride along the line.  Writes
// out[k*ost] = du.  Downwind lines (c < 0) use the mirrored reconstruction on
// the same physically ordered window.
// Masked form: one instantiation per (RUN, ghost kind) -- the ghost counts
// gl (left) / gr (right) of the run are runtime values (integer selects on the
// six window ends), so every full run of a sweep shares one body: a small hot
// code footprint (the instruction cache was the vpass's second stall reason
// with one body per ghost pattern).  Ghost values are zeros (ZERO) or the
// periodic image at -/+ wrap; a masked zero ghost reads the run's own first
// point (a valid address) and discards it.
template <int RUN, bool ZERO>
__device__ __forceinline__ void load_window_masked(double* f, const double* __restrict__ P, int st,
                                                   int wrap, int gl, int gr, double c) {
  constexpr int NV = RUN + 6;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const bool lg = (q < 3) && (q < gl);
    const bool rg = (q >= NV - 3) && (q >= NV - gr);
    int idx = q * st;
    if (ZERO) {
      if (lg || rg) idx = 3 * st;
    } else {
      if (lg) idx += wrap;
      if (rg) idx -= wrap;
    }
    const double v = c * P[idx];
    f[q] = (ZERO && (lg || rg)) ? 0.0 : v;
  }
}

template <int RUN, bool ZERO, bool LINEAR>
__device__ __noinline__ void adv_run_ref_masked(const double* __restrict__ P, int st, int wrap,
                                                int gl, int gr, double c, double eps,
                                                double inv_h, double* __restrict__ out, int ost) {
  constexpr int NV = RUN + 6;
  double f[NV];
  load_window_masked<RUN, ZERO>(f, P, st, wrap, gl, gr, c);
  const bool rev = c < 0.0;
  double Fp = 0.0;
#pragma unroll
  for (int t = 0; t <= RUN; ++t) {
    const int i = t + 2, m = t + 3;
    const double F = rev ? recon_ref(f[m + 2], f[m + 1], f[m], f[m - 1], f[m - 2], eps, LINEAR)
                         : recon_ref(f[i - 2], f[i - 1], f[i], f[i + 1], f[i + 2], eps, LINEAR);
    if (t > 0) out[(t - 1) * ost] = (F - Fp) * inv_h;
    Fp = F;
  }
}

// Window load of the fast run: the values in upwind order (a downwind line, c < 0, is the
// positive reconstruction of the reversed line, weno.hpp:178-183, so only the addressing
// depends on the direction -- per lane, no divergent branch when the lines of a warp
// differ in sign).
template <int RUN, bool ZERO, int Q0 = 0, int Q1 = RUN + 6>
__device__ __forceinline__ void load_window_dir(double* f, const double* __restrict__ P, int st,
                                                int wrap, int gl, int gr, double c, bool rev) {
  constexpr int NV = RUN + 6;
#pragma unroll
  for (int q = Q0; q < Q1; ++q) {
    // physical window position of upwind position q: q or NV - 1 - q; only the three
    // positions at each end can be ghosts
    const bool endl = (q < 3), endr = (q >= NV - 3);
    int idx = (rev ? NV - 1 - q : q) * st;
    bool ghost = false;
    if (endl || endr) {
      const int pq = rev ? NV - 1 - q : q;
      const bool lg = pq < gl, rg = pq >= NV - gr;
      ghost = lg || rg;
      if (ZERO) {
        if (ghost) idx = 3 * st;
      } else {
        if (lg) idx += wrap;
        if (rg) idx -= wrap;
      }
    }
    const double v = c * P[idx];
    f[q] = (ZERO && ghost) ? 0.0 : v;
  }
}

// N reconstructions side by side (recon_roles step by step over k < N): N independent
// dependency chains in flight.  A single reconstruction is a chain ~14 DP
// operations deep of ~32, and a DFMA result takes ~8 cycles (tools/probe/dfma_ilp.cu), so
// one chain at a time leaves the DP pipe half idle at four warps per scheduler.
template <int N, bool LINEAR>
__device__ __forceinline__ void recon_rolesN(const double* fc, const double* A, const double* B,
                                             const double* C, const double* KA, const double* KB,
                                             const double* KC, const double* a, const double* b,
                                             double* F) {
  double g0[N], c0[N], c1[N], c2[N];
#pragma unroll
  for (int k = 0; k < N; ++k) g0[k] = fma(2.0, a[k], A[k]);
#pragma unroll
  for (int k = 0; k < N; ++k) c0[k] = fma(2.0, g0[k], -a[k]);
#pragma unroll
  for (int k = 0; k < N; ++k) c1[k] = fma(3.0, b[k], -B[k]);
#pragma unroll
  for (int k = 0; k < N; ++k) c2[k] = fma(3.0, b[k], -C[k]);
  if (LINEAR) {
#pragma unroll
    for (int k = 0; k < N; ++k)
      F[k] = fc[k] + kSixth * fma(0.1, c0[k], fma(0.6, c1[k], 0.3 * c2[k]));
    return;
  }
  double g1[N], g2[N], e0[N], e1[N], e2[N], q0[N], q1[N], q2[N], w0[N], w1[N], w2[N], num[N], den[N];
#pragma unroll
  for (int k = 0; k < N; ++k) g1[k] = a[k] + b[k];
#pragma unroll
  for (int k = 0; k < N; ++k) g2[k] = fma(-2.0, b[k], C[k]);
#pragma unroll
  for (int k = 0; k < N; ++k) e0[k] = fma(g0[k], g0[k], KA[k]);
#pragma unroll
  for (int k = 0; k < N; ++k) e1[k] = fma(g1[k], g1[k], KB[k]);
#pragma unroll
  for (int k = 0; k < N; ++k) e2[k] = fma(g2[k], g2[k], KC[k]);
#pragma unroll
  for (int k = 0; k < N; ++k) q0[k] = e0[k] * e0[k];
#pragma unroll
  for (int k = 0; k < N; ++k) q1[k] = e1[k] * e1[k];
#pragma unroll
  for (int k = 0; k < N; ++k) q2[k] = e2[k] * e2[k];
#pragma unroll
  for (int k = 0; k < N; ++k) w0[k] = q1[k] * q2[k];
#pragma unroll
  for (int k = 0; k < N; ++k) w1[k] = (6.0 * q0[k]) * q2[k];
#pragma unroll
  for (int k = 0; k < N; ++k) w2[k] = (3.0 * q0[k]) * q1[k];
#pragma unroll
  for (int k = 0; k < N; ++k) num[k] = fma(w0[k], c0[k], fma(w1[k], c1[k], w2[k] * c2[k]));
#pragma unroll
  for (int k = 0; k < N; ++k) den[k] = 6.0 * (w0[k] + w1[k] + w2[k]);
  double r[N];
#pragma unroll
  for (int k = 0; k < N; ++k) asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r[k]) : "d"(den[k]));
  // one third-order step from the ~2^-20 seed: r (1 + e + e^2), e = 1 - den r (fast_rcp)
  double e[N];
#pragma unroll
  for (int k = 0; k < N; ++k) e[k] = fma(-den[k], r[k], 1.0);
#pragma unroll
  for (int k = 0; k < N; ++k) e[k] = fma(e[k], e[k], e[k]);
#pragma unroll
  for (int k = 0; k < N; ++k) r[k] = fma(r[k], e[k], r[k]);
#pragma unroll
  for (int k = 0; k < N; ++k) F[k] = fc[k] + num[k] * r[k];
}

// interfaces T0 .. T0 + NLEFT - 1 in groups of GS side by side
#ifndef SGWG_P4_GS
#define SGWG_P4_GS 3
#endif

template <int T0, int NLEFT, int GS, bool LINEAR, class DQ, class KQ>
__device__ __forceinline__ void recon_groups(const double* f, DQ Dq, KQ Kq, double* F) {
  if constexpr (NLEFT > 0) {
    constexpr int N = NLEFT < GS ? NLEFT : GS;
    double fc[N], A[N], B[N], C[N], KA[N], KB[N], KC[N], a[N], b[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int i = T0 + k + 2;
      fc[k] = f[i];
      A[k] = Dq(i - 1);
      B[k] = Dq(i);
      C[k] = Dq(i + 1);
      KA[k] = Kq(i - 1);
      KB[k] = Kq(i);
      KC[k] = Kq(i + 1);
      a[k] = f[i] - f[i - 1];
      b[k] = f[i + 1] - f[i];
    }
    recon_rolesN<N, LINEAR>(fc, A, B, C, KA, KB, KC, a, b, F + T0);
    recon_groups<T0 + N, NLEFT - N, GS, LINEAR>(f, Dq, Kq, F);
  }
}

template <int RUN, bool ZERO, bool LINEAR>
__device__ __noinline__ void adv_run_masked(const double* __restrict__ P, int st, int wrap, int gl,
                                            int gr, double c, double eps, double inv_h,
                                            double* __restrict__ out, int ost) {
  constexpr int NV = RUN + 6;
  const bool rev = c < 0.0;
  double f[NV];
  const double eps4 = 4.0 * eps;
  // second difference as the difference of the first differences (shared with a, b)
  auto Dq = [&](int q) { return (f[q + 1] - f[q]) - (f[q] - f[q - 1]); };
  auto Kq = [&](int q) {
    const double d = Dq(q);
    return fma(13.0 / 3.0 * d, d, eps4);
  };
  // interface t (left point i = t + 2 of the upwind-ordered window) -> F[t]; the upwind
  // reconstructions of interfaces 0 .. RUN read window positions 0 .. RUN + 4 only
  double F[RUN + 1];
  int ex = 0;  // max exponent field of the outputs (overflow guard)
  const double sh = rev ? -inv_h : inv_h;
  // reversed: interface t is the flux left of point RUN - t, so du(RUN - t) = (F[t-1] - F[t]) / h
  {
    load_window_dir<RUN, ZERO, 0, RUN + 5>(f, P, st, wrap, gl, gr, c, rev);
    recon_groups<0, RUN + 1, SGWG_P4_GS, LINEAR>(f, Dq, Kq, F);
#pragma unroll
    for (int t = 1; t <= RUN; ++t) {
      const double du = (F[t] - F[t - 1]) * sh;
      ex = max(ex, __double2hiint(du) & 0x7ff00000);
      out[(rev ? RUN - t : t - 1) * ost] = du;
    }
  }
  if (ex == 0x7ff00000)
    adv_run_ref_masked<RUN, ZERO, LINEAR>(P, st, wrap, gl, gr, c, eps, inv_h, out, ost);
}

// run r of a line with m full runs (r == m: the zero-ghost tail point)
template <bool ZERO, bool LINEAR>
__device__ __forceinline__ void run_masked(int r, int m, const double* P, int st, int wrap,
                                           double c, double eps, double inv_h, double* out) {
  if (ZERO && r == m) {
    adv_run_masked<1, true, LINEAR>(P, st, 0, 0, 3, c, eps, inv_h, out, st);
    return;
  }
  const int gl = (r == 0) ? 3 : 0;
  const int gr = (r == m - 1) ? (ZERO ? 2 : 3) : 0;
  adv_run_masked<8, ZERO, LINEAR>(P, st, wrap, gl, gr, c, eps, inv_h, out, st);
}

// K-output form of a periodic full run (the persistent x pass's second sweep):
// instead of du into shared memory, K = (0 - d1) - du (models.hpp:187-197
// order) straight to global memory: d1 = the first sweep's derivative at the
// run's points (shared memory, stride ost), gout / gst = K at the run's points.
template <bool LINEAR>
__device__ __noinline__ void adv_run_kout_ref(const double* __restrict__ P, int st, int wrap, int gl,
                                              int gr, double c, double eps, double inv_h,
                                              const double* __restrict__ d1, int ost,
                                              double* __restrict__ gout, long long gst) {
  constexpr int RUN = 8, NV = RUN + 6;
  double f[NV];
  load_window_masked<RUN, false>(f, P, st, wrap, gl, gr, c);
  const bool rev = c < 0.0;
  double Fp = 0.0;
#pragma unroll
  for (int t = 0; t <= RUN; ++t) {
    const int i = t + 2, m = t + 3;
    const double F = rev ? recon_ref(f[m + 2], f[m + 1], f[m], f[m - 1], f[m - 2], eps, LINEAR)
                         : recon_ref(f[i - 2], f[i - 1], f[i], f[i + 1], f[i + 2], eps, LINEAR);
    if (t > 0) gout[(t - 1) * gst] = (0.0 - d1[(t - 1) * ost]) - (F - Fp) * inv_h;
    Fp = F;
  }
}

template <bool LINEAR>
__device__ __noinline__ void adv_run_kout(const double* __restrict__ P, int st, int wrap, int gl,
                                          int gr, double c, double eps, double inv_h,
                                          const double* __restrict__ d1, int ost,
                                          double* __restrict__ gout, long long gst) {
  constexpr int RUN = 8, NV = RUN + 6;
  const bool rev = c < 0.0;
  double f[NV];
  load_window_dir<RUN, false, 0, RUN + 5>(f, P, st, wrap, gl, gr, c, rev);
  const double eps4 = 4.0 * eps;
  auto Dq = [&](int q) { return (f[q + 1] - f[q]) - (f[q] - f[q - 1]); };
  auto Kq = [&](int q) {
    const double d = Dq(q);
    return fma(13.0 / 3.0 * d, d, eps4);
  };
  double F[RUN + 1];
  recon_groups<0, RUN + 1, SGWG_P4_GS, LINEAR>(f, Dq, Kq, F);
  // du of point k of the run (adv_run_masked: reversed, interface t is left of point RUN - t)
  double du[RUN];
  const double sh = rev ? -inv_h : inv_h;
  int ex = 0;
#pragma unroll
  for (int t = 1; t <= RUN; ++t) {
    const double v = (F[t] - F[t - 1]) * sh;
    ex = max(ex, __double2hiint(v) & 0x7ff00000);
    du[t - 1] = v;
  }
  if (ex == 0x7ff00000) {
    adv_run_kout_ref<LINEAR>(P, st, wrap, gl, gr, c, eps, inv_h, d1, ost, gout, gst);
    return;
  }
  // du[t - 1] belongs to point rev ? RUN - t : t - 1
#pragma unroll
  for (int t = 0; t < RUN; ++t) {
    const int k = rev ? RUN - 1 - t : t;
    gout[k * gst] = (0.0 - d1[k * ost]) - du[t];
  }
}

// ---------------------------------------------------------------------------
// Warp tasks.  The work items of a sweep are its (line, full run of 8 points)
// pairs, numbered run-major (item = r * nlines + l) and packed 32 to a warp
// task, so every lane of every task but a sweep's last has a run whatever the
// line count (a velocity plane of 9 x 257 points has 9 rows: with a task = 32
// lines of one run, 9 lanes of 32 worked).  A lane's run position -- first /
// middle / last of its line -- is a runtime value: the masked run body selects
// the ghosts per lane.  The tail points of zero-ghost lines of 8m + 1 points
// are separate, cheap tasks (32 lines each) dealt last.  Tasks are decoded
// arithmetically by every warp (no table, no serial set-up) and dealt round
// robin: full runs of sweep 0, of sweep 1, then the tails.
// ---------------------------------------------------------------------------
struct P4Sweeps {
  // per sweep s = 0, 1 as scalars (a runtime-indexed array would live in local memory)
  int nl0, nl1, m0, m1, nf0, nf1, nt0, nt1;
  float inl0, inl1;
  __device__ void set(int s, int nlines_, int m_, bool zero) {
    const int nf = (nlines_ * m_ + 31) >> 5, nt = zero ? (nlines_ + 31) >> 5 : 0;
    if (s == 0) {
      nl0 = nlines_, m0 = m_, nf0 = nf, nt0 = nt, inl0 = 1.0f / (float)nlines_;
    } else {
      nl1 = nlines_, m1 = m_, nf1 = nf, nt1 = nt, inl1 = 1.0f / (float)nlines_;
    }
  }
  __device__ __forceinline__ int ntask() const { return nf0 + nf1 + nt0 + nt1; }
  // task t, lane -> sweep, line l, run r (r == m: the tail point), m; false: no item
  __device__ __forceinline__ bool decode(int t, int lane, int& sw, int& l, int& r, int& m) const {
    int u = t;
    bool tail = false;
    if (u < nf0) {
      sw = 0;
    } else if ((u -= nf0) < nf1) {
      sw = 1;
    } else if ((u -= nf1) < nt0) {
      sw = 0, tail = true;
    } else {
      u -= nt0;
      sw = 1, tail = true;
    }
    const int nl = sw ? nl1 : nl0;
    m = sw ? m1 : m0;
    const int idx = (u << 5) + lane;
    if (tail) {
      l = idx;
      r = m;
      return idx < nl;
    }
    r = qdiv(idx, sw ? inl1 : inl0);
    l = idx - r * nl;
    return r < m;
  }
};

// ---------------------------------------------------------------------------
// x pass: dims (0, 1) of C velocity points over the whole periodic x-plane
// ---------------------------------------------------------------------------
template <bool LINEAR>
__global__ void __launch_bounds__(kP4Threads, SGWG_P4_MINB) xpass4d_kernel(const Plane4Params p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  P4MARK(0, 0);
  const int4 tk = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  const int v0 = tk.y, nc = tk.z, cs = tk.w, C = 1 << cs;
  const int n1 = M->ext[0], n2 = M->ext[1], n4 = M->ext[3];
  const int V = M->ext[2] * n4;
  const int NT = (n1 * n2) << cs;
  extern __shared__ __align__(16) double sm[];
  double* U = sm;
  double* D1 = sm + NT;  // d/dx1
  double* D2 = D1 + NT;  // d/dx2
  SGWG_DCHECK(v0 + nc <= V && nc <= C && C <= kP4MaxC, "xpass tile velocity range");
  __shared__ double ca[kP4MaxC], cb[kP4MaxC];
  const int tid = threadIdx.x;
  {
    const double* src = p.uin + M->offset + v0;
    const int cm = nc - 1;
    for (int e = tid; e < NT; e += kP4Threads) {
      const int c = e & (C - 1);
      cp_async8(U + e, src + (e >> cs) * V + min(c, cm), c < nc);
    }
    cp_async_commit();
  }
  if (tid < C) {  // x_j lines at velocity point vl: coefficient v_j (models.hpp:341-344)
    const int vl = v0 + min(tid, nc - 1);
    const int i3 = vl / n4;
    ca[tid] = line_coef(p.flux_a, M, 0, p.space_dim, i3, p.c_a, p.efield);
    cb[tid] = line_coef(p.flux_b, M, 1, p.space_dim, vl - i3 * n4, p.c_b, p.efield);
  }
  // sweep 0: x1 lines (x2, c) = l, stride n2 C, n1 points; sweep 1: x2 lines
  // (x1, c), stride C, n2 points
  P4Sweeps T;
  T.set(0, n2 << cs, n1 >> 3, false);
  T.set(1, n1 << cs, n2 >> 3, false);
  P4MARK(0, 1);
  cp_async_wait<0>();
  __syncthreads();
  P4MARK(0, 2);
  const int lane = tid & 31, warp = tid >> 5;
  const int st0 = n2 << cs, wrap0 = n1 * st0, wrap1 = n2 << cs;
  const double ih1 = M->inv_h[0], ih2 = M->inv_h[1], eps = p.eps;
  const int ntask = T.ntask();
  for (int t = (p.dbg & 1) ? ntask : warp; t < ntask; t += kP4Threads / 32) {
    int sw, l, r, m;
    if (!T.decode(t, lane, sw, l, r, m)) continue;
    const int c = l & (C - 1);
    if (sw == 0) {
      run_masked<false, LINEAR>(r, m, U + l + (8 * r - 3) * st0, st0, wrap0, ca[c], eps, ih1,
                                D1 + l + 8 * r * st0);
    } else {
      const int base = (l >> cs) * wrap1 + c;
      run_masked<false, LINEAR>(r, m, U + base + (8 * r - 3) * C, C, wrap1, cb[c], eps, ih2,
                                D2 + base + 8 * r * C);
    }
  }
  P4MARK(0, 3);
  __syncthreads();
  P4MARK(0, 4);
  // K = (0 - dx1) - dx2 (models.hpp:187-197 order)
  double* kb = p.kbuf + M->offset + v0;
  for (int e = tid; e < NT; e += kP4Threads) {
    const int c = e & (C - 1);
    if (c < nc) kb[(e >> cs) * V + c] = (0.0 - D1[e]) - D2[e];
  }
  P4MARK(0, 5);
}

// ---------------------------------------------------------------------------
// v pass: dims (2, 3) of G whole velocity planes + RK stage + charge density
// ---------------------------------------------------------------------------
template <int STAGE, bool MOMENT>
__device__ __forceinline__ void vpass_epilogue(int NT, const double* U, const double* Kt,
                                               const double* UNt, double* DV1, const double* DV2,
                                               double* out, double dt, int& ex) {
  for (int e = threadIdx.x; e < NT; e += kP4Threads) {
    const double kv = (Kt[e] - DV1[e]) - DV2[e];
    ex = max(ex, __double2hiint(kv) & 0x7ff00000);
    double o;
    if (STAGE == 0)
      o = kv;
    else if (STAGE == 1)
      o = fma(dt, kv, U[e]);
    else if (STAGE == 2)
      o = fma(0.75, UNt[e], 0.25 * fma(dt, kv, U[e]));
    else
      o = fma(1.0 / 3.0, UNt[e], (2.0 / 3.0) * fma(dt, kv, U[e]));
    out[e] = o;
    if (MOMENT) DV1[e] = o;
  }
}

template <bool LINEAR>
__global__ void __launch_bounds__(kP4Threads, SGWG_P4_MINB) vpass4d_kernel(const Plane4Params p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  P4MARK(1, 0);
  const int4 tk = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  const int x0 = tk.y, G = tk.z;
  const int n3 = M->ext[2], n4 = M->ext[3];
  const int V = n3 * n4;
  const int NT = G * V;
  extern __shared__ __align__(16) double sm[];
  __shared__ unsigned long long bar[2];
  __shared__ double ce1[kP4MaxG], ce2[kP4MaxG];
  const int tid = threadIdx.x;
  const int stage = p.stage;
  const long long gs = M->offset + (long long)x0 * V;  // tile start (doubles)
  const long long ga = gs & ~1LL;                         // 16-byte aligned start
  const int shift = (int)(gs - ga);
  const unsigned nbytes = (unsigned)((((gs + NT + 1) & ~1LL) - ga) * 8);
  const int pitch = (NT + 3) & ~1;
  // [u^(s) | K | u^n | dv1 | dv2], the first three staged by bulk copies with
  // the tile's alignment shift
  double* U = sm + shift;
  double* Kt = sm + pitch + shift;
  double* UNt = sm + 2 * pitch + shift;
  double* DV1 = sm + 3 * pitch;
  double* DV2 = sm + 4 * pitch;
  if (tid == 0) {  // the CTA barrier below publishes the initialised mbarriers
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    bulk_g2s(sm, p.uin + ga, nbytes, &bar[0]);
    if (p.dbg & 4) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[1])) : "memory");
    } else if (stage > 1) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[1])),
                   "r"(2 * nbytes)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + pitch)),
          "l"(p.kbuf + ga), "r"(nbytes), "r"(smem_u32(&bar[1]))
          : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + 2 * pitch)),
          "l"(p.un + ga), "r"(nbytes), "r"(smem_u32(&bar[1]))
          : "memory");
    } else {
      bulk_g2s(sm + pitch, p.kbuf + ga, nbytes, &bar[1]);
    }
  }
  // sweep 0: v2 lines (rows rho = g n3 + i3), unit stride, n4 points;
  // sweep 1: v1 lines (columns kappa = g n4 + i4), stride n4, n3 points
  P4Sweeps T;
  T.set(0, G * n3, n4 >> 3, true);
  T.set(1, G * n4, n3 >> 3, true);
  if (tid < G) {  // v_j lines at x point x0+tid: -E_j(x) (VP) or the advection speed
    ce1[tid] = line_coef(p.flux_a, M, 2, p.space_dim, x0 + tid, p.c_a, p.efield);
    ce2[tid] = line_coef(p.flux_b, M, 3, p.space_dim, x0 + tid, p.c_b, p.efield);
  }
  __syncthreads();
  P4MARK(1, 1);
  mbar_wait(&bar[0], 0);
  P4MARK(1, 2);
  const int lane = tid & 31, warp = tid >> 5;
  {
    const float i3f = 1.0f / (float)n3, i4f = 1.0f / (float)n4;
    const double ih3 = M->inv_h[2], ih4 = M->inv_h[3], eps = p.eps;
    const int ntask = T.ntask();
    for (int t = (p.dbg & 1) ? ntask : warp; t < ntask; t += kP4Threads / 32) {
      int sw, l, r, m;
      if (!T.decode(t, lane, sw, l, r, m)) continue;
      if (sw == 0) {
        const int base = l * n4;
        run_masked<true, LINEAR>(r, m, U + base + 8 * r - 3, 1, 0, ce2[qdiv(l, i3f)], eps, ih4,
                                 DV2 + base + 8 * r);
      } else {
        const int gx = qdiv(l, i4f);
        const int base = gx * V + (l - gx * n4);
        run_masked<true, LINEAR>(r, m, U + base + (8 * r - 3) * n4, n4, 0, ce1[gx], eps, ih3,
                                 DV1 + base + 8 * r * n4);
      }
    }
  }
  P4MARK(1, 3);
  mbar_wait(&bar[1], 0);
  __syncthreads();
  P4MARK(1, 4);
  // epilogue: k = (K - dv1) - dv2, RK stage (timestep.hpp:86-104), output
  const double dt = (ctl != nullptr) ? ctl->dt : 0.0;
  const bool moment = (p.rho_parts != nullptr) && (stage > 0);
  double* out = p.out + gs;
  int ex = 0;
  if (p.dbg & 2) return;
  if (moment) {
    if (stage == 1)
      vpass_epilogue<1, true>(NT, U, Kt, UNt, DV1, DV2, out, dt, ex);
    else if (stage == 2)
      vpass_epilogue<2, true>(NT, U, Kt, UNt, DV1, DV2, out, dt, ex);
    else
      vpass_epilogue<3, true>(NT, U, Kt, UNt, DV1, DV2, out, dt, ex);
  } else {
    if (stage == 0)
      vpass_epilogue<0, false>(NT, U, Kt, UNt, DV1, DV2, out, dt, ex);
    else if (stage == 1)
      vpass_epilogue<1, false>(NT, U, Kt, UNt, DV1, DV2, out, dt, ex);
    else if (stage == 2)
      vpass_epilogue<2, false>(NT, U, Kt, UNt, DV1, DV2, out, dt, ex);
    else
      vpass_epilogue<3, false>(NT, U, Kt, UNt, DV1, DV2, out, dt, ex);
  }
  P4MARK(1, 6);
  if (stage > 0 && ex == 0x7ff00000) {  // non-finite tendency (tendency_finite, timestep.hpp:71-75)
    const unsigned long long code =
        (unsigned long long)ctl->cur_step * 4ull + (unsigned long long)stage;
    atomicMin(p.fail + tk.x, code);
  }
  if (moment) {
    // charge density of the stage output per x point (moment_density,
    // models.hpp:294-306) with the trapezoid weights (models.hpp:64-71,240-257)
    // h3 h4 f(a) f(b), f = 1/2 at the zero-ghost ends: the plane sum minus half
    // the edge rows / columns plus a quarter of the corners.  One warp per x point.
    __syncthreads();
    const double hh = M->h[2] * M->h[3];
    for (int gx = warp; gx < G; gx += kP4Threads / 32) {
      const double* w = DV1 + gx * V;
      double all = 0.0, edge = 0.0;
      for (int e = lane; e < V; e += 32) all += w[e];
      for (int e = lane; e < n4; e += 32) edge += w[e] + w[(n3 - 1) * n4 + e];
      for (int e = lane; e < n3; e += 32) edge += w[e * n4] + w[e * n4 + n4 - 1];
      double corner = (lane == 0) ? (w[0] + w[n4 - 1]) + (w[(n3 - 1) * n4] + w[V - 1]) : 0.0;
      double acc = fma(-0.5, edge, fma(0.25, corner, all));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) p.rho_parts[(M->xoff + x0 + gx) * kRhoParts] = hh * acc;
    }
  }
  P4MARK(1, 5);
  if (p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

// ---------------------------------------------------------------------------
// Persistent, software-pipelined v pass (default).  A phase trace of the
// one-tile-per-CTA form (tools/trace_p4.py) put ~45 % of a CTA's time outside
// the sweeps: a chain of dependent global loads before the first barrier
// (tile -> member -> E field, ~4.7 K cycles), the epilogue (~2 K) and the
// charge-density reduction (~3.5 K).  Here CTAs (two per SM) loop over the
// tile list and everything a tile needs is fetched one tile ahead: its
// descriptor (thread 0, stored to a 3-slot ring in shared memory), its u^(s)
// (bulk copy into the other U slot during the current sweeps), its K / u^n
// (bulk copies after the current epilogue) and its E-field line coefficients
// (loaded after the current epilogue).  The epilogue stores w_3 w_4 f of the
// stage output (trapezoid weights, models.hpp:64-71,240-257) so the charge
// density is a plain per-plane sum (4 accumulators per lane).
// smem: [U0 | U1 | K | u^n | dv1 | dv2], each p.vpitch doubles.
// ---------------------------------------------------------------------------
using VInfo = P4VTile;

// thread 0: the descriptor of tile t into a ring slot, async (16-byte pieces)
__device__ __forceinline__ void vp_fetch_info(const Plane4Params& p, int t, VInfo* dst) {
  const char* src = (const char*)(p.vtiles + t);
  for (int q = 0; q < (int)sizeof(VInfo); q += 16) {
    const unsigned sd = (unsigned)__cvta_generic_to_shared((char*)dst + q);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sd), "l"(src + q) : "memory");
  }
}

// threads tid < G: the line coefficients of the tile's x points into ce1 / ce2 -- for
// Vlasov-Poisson the raw E_j(x) by async copies (the sweeps apply the sign,
// models.hpp:346-349), else line_coef (no memory dependence)
__device__ __forceinline__ void vp_fetch_coefs(const Plane4Params& p, const VInfo* v, double* ce1,
                                               double* ce2) {
  const int tid = threadIdx.x;
  if (tid >= v->G) return;
  if (p.flux_a == kFluxKinVP) {
    const double* E = p.efield + v->xoff * p.space_dim + v->x0 + tid;
    cp_async8(ce1 + tid, E, true);
    cp_async8(ce2 + tid, E + v->nx, true);
  } else {
    const MemberDesc* M = p.mem + v->mi;
    ce1[tid] = line_coef(p.flux_a, M, 2, p.space_dim, v->x0 + tid, p.c_a, p.efield);
    ce2[tid] = line_coef(p.flux_b, M, 3, p.space_dim, v->x0 + tid, p.c_b, p.efield);
  }
}


__device__ __forceinline__ void bulk_g2s_noexpect(void* dst, const void* src, unsigned bytes,
                                                  unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// thread 0: K (and u^n for stages 2, 3) of tile v into the K / u^n slots
__device__ __forceinline__ void vp_issue_ku(const Plane4Params& p, const VInfo& v, double* Ks,
                                            double* UNs, unsigned long long* bar) {
  const bool un = p.stage > 1;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(un ? 2 * v.nbytes : v.nbytes)
               : "memory");
  bulk_g2s_noexpect(Ks, p.kbuf + v.ga, v.nbytes, bar);
  if (un) bulk_g2s_noexpect(UNs, p.un + v.ga, v.nbytes, bar);
}

// the sweeps of one tile (both directions, all warps); U = the tile's u^(s)
template <bool LINEAR>
__device__ __noinline__ void vp_tile_sweeps(const VInfo* vi, double eps, const double* U,
                                            double* DV1, double* DV2, const double* ce1,
                                            const double* ce2, double csign) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = vi->G, n3 = vi->n3, n4 = vi->n4, V = vi->V;
  P4Sweeps T;
  T.set(0, G * n3, n4 >> 3, true);
  T.set(1, G * n4, n3 >> 3, true);
  const float i3f = 1.0f / (float)n3, i4f = 1.0f / (float)n4;
  const double ih3 = vi->ih3, ih4 = vi->ih4;
  const int ntask = T.ntask();
  for (int q = warp; q < ntask; q += kP4Threads / 32) {
    int sw, l, r, m;
    if (!T.decode(q, lane, sw, l, r, m)) continue;
    if (sw == 0) {
      const int base = l * n4;
      SGWG_DCHECK(qdiv(l, i3f) == l / n3 && l < G * n3 && base + 8 * r < G * V, "vpass row run");
      run_masked<true, LINEAR>(r, m, U + base + 8 * r - 3, 1, 0, csign * ce2[qdiv(l, i3f)], eps,
                               ih4, DV2 + base + 8 * r);
    } else {
      const int gx = qdiv(l, i4f);
      const int base = gx * V + (l - gx * n4);
      SGWG_DCHECK(gx == l / n4 && gx < G && base + 8 * r * n4 < G * V, "vpass column run");
      run_masked<true, LINEAR>(r, m, U + base + (8 * r - 3) * n4, n4, 0, csign * ce1[gx], eps, ih3,
                               DV1 + base + 8 * r * n4);
    }
  }
}

// k = (K - dv1) - dv2, RK stage (timestep.hpp:86-104), output; MOMENT: DV1[e] = w3 w4 f
template <int STAGE, bool MOMENT>
__device__ __forceinline__ int vp_epilogue(const VInfo* vi, const double* U, const double* Kt,
                                           const double* UNt, double* DV1, const double* DV2,
                                           double* out, double dt) {
  const int NT = vi->NT, V = vi->V, n3 = vi->n3, n4 = vi->n4;
  const float iVf = 1.0f / (float)V, i4f = 1.0f / (float)n4;
  int ex = 0;
#pragma unroll 4
  for (int e = threadIdx.x; e < NT; e += kP4Threads) {
    const double kv = (Kt[e] - DV1[e]) - DV2[e];
    ex = max(ex, __double2hiint(kv) & 0x7ff00000);
    double o;
    if (STAGE == 0)
      o = kv;
    else if (STAGE == 1)
      o = fma(dt, kv, U[e]);
    else if (STAGE == 2)
      o = fma(0.75, UNt[e], 0.25 * fma(dt, kv, U[e]));
    else
      o = fma(1.0 / 3.0, UNt[e], (2.0 / 3.0) * fma(dt, kv, U[e]));
    out[e] = o;
    if (MOMENT) {
      const int g = qdiv(e, iVf), rem = e - g * V, i3 = qdiv(rem, i4f), i4 = rem - i3 * n4;
      const double w3 = (i3 == 0 || i3 == n3 - 1) ? 0.5 : 1.0;
      const double w4 = (i4 == 0 || i4 == n4 - 1) ? 0.5 : 1.0;
      DV1[e] = (w3 * w4) * o;
    }
  }
  return ex;
}

template <bool LINEAR>
__global__ void __launch_bounds__(kP4Threads, 2) vpass4d_persist_kernel(const Plane4Params p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ unsigned long long bar[3];  // U0, U1, K/u^n
  __shared__ double ce1[2][kP4MaxG], ce2[2][kP4MaxG];
  // tiles in a 4-slot ring: tile `it` of this CTA is tix[it % 4] with descriptor
  // info[it % 4] (async-filled two tiles ahead).  Tiles after the first two come
  // from a global counter (dynamic scheduling: a static round robin left the
  // slowest CTA ~17 % behind the median); the counter's value for tile it + 3
  // is requested at tile it, so its latency is never waited for.
  __shared__ VInfo info[4];
  __shared__ int tix[4];
  const double csign = (p.flux_a == kFluxKinVP) ? -1.0 : 1.0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pitch = p.vpitch;
  double* Ks = sm + 2 * pitch;
  double* UNs = sm + 3 * pitch;
  double* DV1 = sm + 4 * pitch;
  double* DV2 = sm + 5 * pitch;
  const int G0 = gridDim.x, nt = p.ntiles;
  if ((int)blockIdx.x >= nt) return;
  // static tile data before the dependency wait (overlaps the previous kernel under PDL)
  if (tid == 0) {
    tix[0] = blockIdx.x;
    tix[1] = blockIdx.x + G0;
    vp_fetch_info(p, tix[0], &info[0]);
    if (tix[1] < nt) vp_fetch_info(p, tix[1], &info[1]);
  }
  cp_async_commit();
  cp_async_wait<0>();
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  if (tid == 0) tix[2] = (tix[1] < nt) ? 2 * G0 + (int)atomicAdd(p.sched, 1u) : nt;
  const int stage = p.stage;
  const bool moment = (p.rho_parts != nullptr) && (stage > 0);
  __syncthreads();
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    bulk_g2s(sm, p.uin + info[0].ga, info[0].nbytes, &bar[0]);
    vp_issue_ku(p, info[0], Ks, UNs, &bar[2]);
  }
  vp_fetch_coefs(p, &info[0], ce1[0], ce2[0]);
  cp_async_commit();
  cp_async_wait<0>();
  const double dt = (ctl != nullptr) ? ctl->dt : 0.0;
#ifdef SGWG_TRACE
  long long ph[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long tc = clock64(), tn_;
#define P4PH(k)                 \
  do {                          \
    tn_ = clock64();            \
    ph[k] += tn_ - tc;          \
    tc = tn_;                   \
  } while (0)
#else
#define P4PH(k) \
  do {          \
  } while (0)
#endif
  for (int it = 0;; ++it) {
    // it: local tile counter -- U slot it & 1 (parity (it >> 1) & 1), K/u^n parity it & 1
    const int b = it & 1;
    // [A]: ce / info / tix of this tile published (and, at it = 0, the mbarriers);
    // the previous tile is completely done with the other U slot and dv1
    __syncthreads();
    P4PH(0);
    const int t = tix[it & 3];
    if (t >= nt) break;
    const int t1 = tix[(it + 1) & 3];
    const VInfo* vi = &info[it & 3];
    if (tid == 0) {
      if (t1 < nt) {
        const VInfo* v1 = &info[(it + 1) & 3];
        bulk_g2s(sm + (b ^ 1) * pitch, p.uin + v1->ga, v1->nbytes, &bar[b ^ 1]);
      }
      // the descriptor of the tile after next (its index came from the counter
      // during the previous tile's epilogue) into its ring slot
      const int t2 = tix[(it + 2) & 3];
      if (t2 < nt) vp_fetch_info(p, t2, &info[(it + 2) & 3]);
    }
    P4PH(9);
    // the next tile's line coefficients (its descriptor is in slot it + 1)
    if (t1 < nt) vp_fetch_coefs(p, &info[(it + 1) & 3], ce1[b ^ 1], ce2[b ^ 1]);
    cp_async_commit();
    const double* U = sm + b * pitch + vi->shift;
    SGWG_DCHECK(vi->shift + vi->NT <= pitch && (long long)vi->nbytes <= 8LL * pitch,
                "vpass tile exceeds its shared-memory slot");
    SGWG_DCHECK(vi->gs + vi->NT <= p.mem[vi->mi].offset + p.mem[vi->mi].npts,
                "vpass tile exceeds its member");
    SGWG_DCHECK(vi->G <= kP4MaxG && p.vtiles[t].gs == vi->gs, "vpass tile descriptor");
    P4PH(8);
    mbar_wait(&bar[b], (it >> 1) & 1);
    P4PH(1);
    vp_tile_sweeps<LINEAR>(vi, p.eps, U, DV1, DV2, ce1[b], ce2[b], csign);
    P4PH(2);
    cp_async_wait<0>();  // this thread's async copies (descriptor, coefficients) landed
    mbar_wait(&bar[2], it & 1);
    P4PH(3);
    // [B]: dv1 / dv2 complete, K / u^n landed
    __syncthreads();
    P4PH(4);
    // the counter's tile for three iterations ahead: requested now, stored after
    // the epilogue (the atomic's round trip hidden behind it)
    const bool more = (tid == 0) && tix[(it + 2) & 3] < nt;
    unsigned int got = 0u;
    if (more) got = atomicAdd(p.sched, 1u);
    double* out = p.out + vi->gs;
    const double* Kt = Ks + vi->shift;
    const double* UNt = UNs + vi->shift;
    int ex;
    if (moment) {
      ex = (stage == 1)   ? vp_epilogue<1, true>(vi, U, Kt, UNt, DV1, DV2, out, dt)
           : (stage == 2) ? vp_epilogue<2, true>(vi, U, Kt, UNt, DV1, DV2, out, dt)
                          : vp_epilogue<3, true>(vi, U, Kt, UNt, DV1, DV2, out, dt);
    } else {
      ex = (stage == 0)   ? vp_epilogue<0, false>(vi, U, Kt, UNt, DV1, DV2, out, dt)
           : (stage == 1) ? vp_epilogue<1, false>(vi, U, Kt, UNt, DV1, DV2, out, dt)
           : (stage == 2) ? vp_epilogue<2, false>(vi, U, Kt, UNt, DV1, DV2, out, dt)
                          : vp_epilogue<3, false>(vi, U, Kt, UNt, DV1, DV2, out, dt);
    }
    if (stage > 0 && ex == 0x7ff00000) {  // non-finite tendency (tendency_finite, timestep.hpp:71-75)
      const unsigned long long code =
          (unsigned long long)ctl->cur_step * 4ull + (unsigned long long)stage;
      atomicMin(p.fail + vi->mi, code);
    }
    if (tid == 0) tix[(it + 3) & 3] = more ? 2 * G0 + (int)got : nt;  // tile it - 1's slot
    P4PH(5);
    // [C]: K / u^n slots free, w f of the stage output in dv1
    __syncthreads();
    P4PH(6);
    if (tid == 0 && t1 < nt) vp_issue_ku(p, info[(it + 1) & 3], Ks, UNs, &bar[2]);
    if (moment) {
      // charge density of the stage output per x point (moment_density, models.hpp:294-306)
      const int V = vi->V;
      for (int gx = warp; gx < vi->G; gx += kP4Threads / 32) {
        const double* w = DV1 + gx * V;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int e = lane;
        for (; e + 96 < V; e += 128) {
          a0 += w[e];
          a1 += w[e + 32];
          a2 += w[e + 64];
          a3 += w[e + 96];
        }
        if (e < V) a0 += w[e];
        if (e + 32 < V) a1 += w[e + 32];
        if (e + 64 < V) a2 += w[e + 64];
        double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) p.rho_parts[(vi->xoff + vi->x0 + gx) * kRhoParts] = vi->hh * acc;
      }
    }
    P4PH(7);
  }
#ifdef SGWG_TRACE
  if (tid == 0 && blockIdx.x < kP4TraceCtas)
    for (int k = 0; k < 10; ++k) sgwg_p4trace[1][blockIdx.x][k] = ph[k];
#endif
  // the last CTA out resets the tile counter for the next launch
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(p.sched + 1, 1u) == (unsigned)min(G0, nt) - 1) {
      p.sched[0] = 0u;
      p.sched[1] = 0u;
      __threadfence();
    }
  }
  if (p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

// ---------------------------------------------------------------------------
// Persistent x pass (default; SGWG_P4_PERSIST=0 keeps xpass4d_kernel).  The
// phase trace of the one-tile-per-CTA form: issue of the strided gather +
// descriptor chain ~21 % of a CTA's time, the K store loop ~14 %.  Here CTAs
// (two per SM) loop over the tiles; the gather of tile i+1 (cp.async into the
// other U slot) is issued right after tile i's first barrier and lands during
// tile i's sweeps; the x1 sweep writes d/dx1 to shared memory, and the x2
// sweep, after a barrier, stores K = (0 - d/dx1) - d/dx2 straight to global
// memory (no d/dx2 array, no separate store phase).
// smem: [U0 | U1 | d/dx1], each p.xpitch doubles.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void xp_fetch_info(const Plane4Params& p, int t, P4XTile* dst) {
  const char* src = (const char*)(p.xtiles + t);
  for (int q = 0; q < (int)sizeof(P4XTile); q += 16) {
    const unsigned sd = (unsigned)__cvta_generic_to_shared((char*)dst + q);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(sd), "l"(src + q) : "memory");
  }
}

// every thread: its share of the strided gather of tile x (X x-points x C velocity points)
__device__ __forceinline__ void xp_issue_gather(const Plane4Params& p, const P4XTile* x, double* Ub) {
  const int cs = x->cs, C = 1 << cs, V = x->V, cm = x->nc - 1;
  const int NT = (x->n1 * x->n2) << cs;
  const double* src = p.uin + x->src;
  for (int e = threadIdx.x; e < NT; e += kP4Threads) {
    const int c = e & (C - 1);
    cp_async8(Ub + e, src + (e >> cs) * V + min(c, cm), c < x->nc);
  }
}

// threads tid < C: x_j line coefficients at velocity point v0 + tid (models.hpp:341-344)
__device__ __forceinline__ void xp_coefs(const P4XTile* x, double* ca, double* cb) {
  const int tid = threadIdx.x;
  if (tid < (1 << x->cs)) {
    const int vl = x->v0 + min(tid, x->nc - 1);
    const int i3 = vl / x->n4;
    ca[tid] = x->ca0 + i3 * x->ca1;
    cb[tid] = x->cb0 + (vl - i3 * x->n4) * x->cb1;
  }
}

template <bool LINEAR>
__global__ void __launch_bounds__(kP4Threads, 2) xpass4d_persist_kernel(const Plane4Params p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double ca[2][kP4MaxC], cb[2][kP4MaxC];
  __shared__ P4XTile info[4];  // tile `it` of this CTA: tix[it % 4], info[it % 4]
  __shared__ int tix[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int pitch = p.xpitch;
  double* D1 = sm + 2 * pitch;
  const int G0 = gridDim.x, nt = p.ntiles;
  if ((int)blockIdx.x >= nt) return;
  if (tid == 0) {
    tix[0] = blockIdx.x;
    tix[1] = blockIdx.x + G0;
    xp_fetch_info(p, tix[0], &info[0]);
    if (tix[1] < nt) xp_fetch_info(p, tix[1], &info[1]);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  xp_coefs(&info[0], ca[0], cb[0]);  // static (x coordinates / advection speeds)
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  if (tid == 0) tix[2] = (tix[1] < nt) ? 2 * G0 + (int)atomicAdd(p.sched, 1u) : nt;
  xp_issue_gather(p, &info[0], sm);
  cp_async_commit();
  const double eps = p.eps;
#ifdef SGWG_TRACE
  long long xph[6] = {0, 0, 0, 0, 0, 0};
  long long xtc = clock64(), xtn;
#define XPH(k)             \
  do {                     \
    xtn = clock64();       \
    xph[k] += xtn - xtc;   \
    xtc = xtn;             \
  } while (0)
#else
#define XPH(k) \
  do {         \
  } while (0)
#endif
  for (int it = 0;; ++it) {
    const int b = it & 1;
    cp_async_wait<0>();
    XPH(0);
    // [A]: this tile's u (every thread's copies), coefficients, descriptors and
    // indices visible; the previous tile's x2 sweep is done with the other U slot
    __syncthreads();
    XPH(1);
    const int t = tix[it & 3];
    if (t >= nt) break;
    const int t1 = tix[(it + 1) & 3];
    const P4XTile* xi = &info[it & 3];
    if (t1 < nt) {
      const P4XTile* x1i = &info[(it + 1) & 3];
      xp_issue_gather(p, x1i, sm + (b ^ 1) * pitch);
      xp_coefs(x1i, ca[b ^ 1], cb[b ^ 1]);
    }
    unsigned int got = 0u;
    const bool more = (tid == 0) && tix[(it + 2) & 3] < nt;
    if (tid == 0 && tix[(it + 2) & 3] < nt) xp_fetch_info(p, tix[(it + 2) & 3], &info[(it + 2) & 3]);
    if (more) got = atomicAdd(p.sched, 1u);
    cp_async_commit();
    XPH(2);
    const int cs = xi->cs, C = 1 << cs, nc = xi->nc;
    const int n1 = xi->n1, n2 = xi->n2, V = xi->V;
    SGWG_DCHECK(t >= 0 && t < nt && p.xtiles[t].src == xi->src && p.xtiles[t].cs == cs &&
                    p.xtiles[t].nc == nc && p.xtiles[t].V == V,
                "xpass tile descriptor");
    SGWG_DCHECK(((n1 * n2) << cs) <= pitch, "xpass tile exceeds its slot");
    const double* U = sm + b * pitch;
    const double* cfa = ca[b];
    const double* cfb = cb[b];
    const int st0 = n2 << cs, wrap0 = n1 * st0, wrap1 = n2 << cs;
    // x1 sweep: lines (x2, c) = l, stride n2 C, n1 points -> d/dx1
    {
      const double ih1 = xi->ih1;
      const int nl = n2 << cs, m = n1 >> 3, nb = (nl + 31) >> 5, ntask = nb * m;
      const float inb = 1.0f / (float)nb;
      for (int q = warp; q < ntask; q += kP4Threads / 32) {
        const int r = qdiv(q, inb), l = ((q - r * nb) << 5) + lane;
        if (l >= nl) continue;
        run_masked<false, LINEAR>(r, m, U + l + (8 * r - 3) * st0, st0, wrap0, cfa[l & (C - 1)],
                                  eps, ih1, D1 + l + 8 * r * st0);
      }
    }
    XPH(3);
    if (tid == 0) tix[(it + 3) & 3] = more ? 2 * G0 + (int)got : nt;  // tile it - 1's slot
    // [B]: d/dx1 complete
    __syncthreads();
    XPH(4);
    // x2 sweep: lines (x1, c), stride C, n2 points -> K to global
    {
      const double ih2 = xi->ih2;
      const int nl = n1 << cs, m = n2 >> 3, nb = (nl + 31) >> 5, ntask = nb * m;
      const float inb = 1.0f / (float)nb;
      double* kb = p.kbuf + xi->src;
      for (int q = warp; q < ntask; q += kP4Threads / 32) {
        const int r = qdiv(q, inb), l = ((q - r * nb) << 5) + lane;
        if (l >= nl) continue;
        const int c = l & (C - 1), x1 = l >> cs;
        if (c >= nc) continue;  // padded velocity point of a partial tile
        const int base = x1 * wrap1 + c;
        const int gl = (r == 0) ? 3 : 0, gr = (r == m - 1) ? 3 : 0;
        adv_run_kout<LINEAR>(U + base + (8 * r - 3) * C, C, wrap1, gl, gr, cfb[c], eps, ih2,
                             D1 + base + 8 * r * C, C,
                             kb + ((long long)x1 * n2 + 8 * r) * V + c, V);
      }
    }
    XPH(5);
  }
  cp_async_wait<0>();
#ifdef SGWG_TRACE
  if (tid == 0 && blockIdx.x < kP4TraceCtas)
    for (int k = 0; k < 6; ++k) sgwg_p4trace[0][blockIdx.x][k] = xph[k];
#endif
  if (tid == 0) {  // the last CTA out resets the tile counter for the next launch
    __threadfence();
    if (atomicAdd(p.sched + 1, 1u) == (unsigned)min(G0, nt) - 1) {
      p.sched[0] = 0u;
      p.sched[1] = 0u;
      __threadfence();
    }
  }
}

cudaError_t launch_plane4(const Plane4Params& p, int pass, int nblocks, size_t smem,
                          cudaStream_t s) {
  if (nblocks <= 0) return cudaSuccess;
  if (pass == 0) {
    if (p.xpitch > 0)
      return p.linear
                 ? launch_k(xpass4d_persist_kernel<true>, dim3(nblocks), dim3(kP4Threads), smem, s, p)
                 : launch_k(xpass4d_persist_kernel<false>, dim3(nblocks), dim3(kP4Threads), smem, s,
                            p);
    return p.linear ? launch_k(xpass4d_kernel<true>, dim3(nblocks), dim3(kP4Threads), smem, s, p)
                    : launch_k(xpass4d_kernel<false>, dim3(nblocks), dim3(kP4Threads), smem, s, p);
  }
  if (p.vpitch > 0) {  // persistent form: nblocks = min(tiles, 2 x SMs) CTAs
    return p.linear
               ? launch_k(vpass4d_persist_kernel<true>, dim3(nblocks), dim3(kP4Threads), smem, s, p)
               : launch_k(vpass4d_persist_kernel<false>, dim3(nblocks), dim3(kP4Threads), smem, s,
                          p);
  }
  return p.linear ? launch_k(vpass4d_kernel<true>, dim3(nblocks), dim3(kP4Threads), smem, s, p)
                  : launch_k(vpass4d_kernel<false>, dim3(nblocks), dim3(kP4Threads), smem, s, p);
}

cudaError_t configure_plane4() {
  const int maxs = 200 * 1024;
  cudaError_t e;
  cudaFuncSetAttribute(xpass4d_persist_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       maxs);
  cudaFuncSetAttribute(xpass4d_persist_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       maxs);
  cudaFuncSetAttribute(xpass4d_persist_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       100);
  cudaFuncSetAttribute(xpass4d_persist_kernel<false>,
                       cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  // two ~113 KB CTAs per SM need the full shared-memory carveout
  cudaFuncSetAttribute(vpass4d_persist_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       100);
  cudaFuncSetAttribute(vpass4d_persist_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       100);
  if ((e = cudaFuncSetAttribute(xpass4d_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                maxs)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(xpass4d_kernel<false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, maxs)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(vpass4d_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                maxs)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(vpass4d_persist_kernel<true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, maxs)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(vpass4d_persist_kernel<false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, maxs)) != cudaSuccess)
    return e;
  return cudaFuncSetAttribute(vpass4d_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              maxs);
}
