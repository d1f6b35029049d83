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

constexpr int kP4Threads = 256;
constexpr int kP4MaxC = 64;   // velocity points per x-pass tile

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

// Reference-form fallback of adv_run (recon_ref: weno5_flux_positive /
// _negative, weno.hpp:60-80): taken only when the fast form overflowed
// (|u| >~ 1e36 makes the common-denominator weights infinite, the reference's
// separate divides do not).
template <int RUN, int GL, int GR, bool ZERO, bool ACC>
__device__ __noinline__ void adv_run_ref(const double* __restrict__ P, int st, int wrap, double c,
                                         double eps, int linear, double inv_h,
                                         double* __restrict__ out, int ost) {
  constexpr int NV = RUN + 6;
  double f[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    if (q < GL)
      f[q] = ZERO ? 0.0 : c * P[q * st + wrap];
    else if (q >= NV - GR)
      f[q] = ZERO ? 0.0 : c * P[q * st - wrap];
    else
      f[q] = c * P[q * st];
  }
  const bool rev = c < 0.0;
  double Fp = 0.0;
#pragma unroll
  for (int t = 0; t <= RUN; ++t) {
    const int i = t + 2, m = t + 3;
    const double F = rev ? recon_ref(f[m + 2], f[m + 1], f[m], f[m - 1], f[m - 2], eps, linear)
                         : recon_ref(f[i - 2], f[i - 1], f[i], f[i + 1], f[i + 2], eps, linear);
    if (t > 0) {
      const double du = (F - Fp) * inv_h;
      if (ACC)
        out[(t - 1) * ost] += du;
      else
        out[(t - 1) * ost] = du;
    }
    Fp = F;
  }
}

// du/dx of c*u (upwind WENO5-JS, advect_derivative_line weno.hpp:160-192) for
// RUN consecutive points of one line.  P: the window's first value (physical
// point 8r - 3 of the line), st: smem stride along the line.  GL / GR values at
// the window ends are ghosts: zeros (ZERO) or the periodic image at -/+ wrap.
// Writes out[k*ost] = du (ACC: out[k*ost] += du).  Downwind lines (c < 0) use
// the mirrored reconstruction on the same physically ordered window.
template <int RUN, int GL, int GR, bool ZERO, bool LINEAR, bool ACC>
__device__ __noinline__ void adv_run(const double* __restrict__ P, int st, int wrap, double c,
                                     double eps, double inv_h, double* __restrict__ out,
                                     int ost) {
  constexpr int NV = RUN + 6;
  double f[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    if (q < GL)
      f[q] = ZERO ? 0.0 : c * P[q * st + wrap];
    else if (q >= NV - GR)
      f[q] = ZERO ? 0.0 : c * P[q * st - wrap];
    else
      f[q] = c * P[q * st];
  }
  const double eps4 = 4.0 * eps;
  double D[NV], K[NV], dd[NV];
#pragma unroll
  for (int q = 1; q < NV - 1; ++q) {
    D[q] = fma(-2.0, f[q], f[q - 1] + f[q + 1]);
    K[q] = fma(13.0 / 3.0 * D[q], D[q], eps4);
  }
#pragma unroll
  for (int q = 1; q < NV; ++q) dd[q] = f[q] - f[q - 1];
  double du[RUN];
  double Fp = 0.0;
  if (!(c < 0.0)) {
#pragma unroll
    for (int t = 0; t <= RUN; ++t) {
      const int i = t + 2;
      const double F = recon_roles<LINEAR>(f[i], D[i - 1], D[i], D[i + 1], K[i - 1], K[i],
                                           K[i + 1], dd[i], dd[i + 1]);
      if (t > 0) du[t - 1] = (F - Fp) * inv_h;
      Fp = F;
    }
  } else {
#pragma unroll
    for (int t = 0; t <= RUN; ++t) {
      const int m = t + 3;
      const double F = recon_roles<LINEAR>(f[m], D[m + 1], D[m], D[m - 1], K[m + 1], K[m],
                                           K[m - 1], -dd[m + 1], -dd[m]);
      if (t > 0) du[t - 1] = (F - Fp) * inv_h;
      Fp = F;
    }
  }
  // overflow guard on the integer pipe: a non-finite du (all exponent bits
  // set) sends the run through the reference form
  int ex = 0;
#pragma unroll
  for (int k = 0; k < RUN; ++k) ex = max(ex, __double2hiint(du[k]) & 0x7ff00000);
  if (ex == 0x7ff00000) {
    adv_run_ref<RUN, GL, GR, ZERO, ACC>(P, st, wrap, c, eps, LINEAR, inv_h, out, ost);
    return;
  }
#pragma unroll
  for (int k = 0; k < RUN; ++k) {
    if (ACC)
      out[k * ost] += du[k];
    else
      out[k * ost] = du[k];
  }
}

// A sweep over `nlines` lines of n points, as warp tasks of 32 lines sharing
// one run-position class.  Periodic lines have n = 8m; zero-ghost lines
// n = 8m + 1 (8m points in runs + a one-point tail).
struct SweepGeom {
  int nlines, m;
  int zero;      // zero ghosts (else periodic)
  float inv_nl;  // 1 / nlines (qdiv)
};

// class c of a sweep -> (first run, number of runs); classes:
// 0 first run, 1 middle runs, 2 last run, 3 tail (zero) / unused; m == 1:
// class 0 is the single run (both ends), class 2 unused.
__device__ __forceinline__ void class_runs(const SweepGeom& g, int c, int& r0, int& nr) {
  if (c == 0) {
    r0 = 0;
    nr = 1;
  } else if (c == 1) {
    r0 = 1;
    nr = max(0, g.m - 2);
  } else if (c == 2) {
    r0 = g.m - 1;
    nr = (g.m >= 2) ? 1 : 0;
  } else {
    r0 = g.m;
    nr = g.zero ? 1 : 0;
  }
}

template <bool ZERO, bool LINEAR, bool ACC>
__device__ __forceinline__ void run_dispatch(int cls, int m, const double* P, int st, int wrap,
                                             double c, double eps, double inv_h, double* out) {
  if constexpr (ZERO) {
    if (cls == 3)
      adv_run<1, 0, 3, true, LINEAR, ACC>(P, st, 0, c, eps, inv_h, out, st);
    else if (cls == 1)
      adv_run<8, 0, 0, true, LINEAR, ACC>(P, st, 0, c, eps, inv_h, out, st);
    else if (cls == 0 && m == 1)
      adv_run<8, 3, 2, true, LINEAR, ACC>(P, st, 0, c, eps, inv_h, out, st);
    else if (cls == 0)
      adv_run<8, 3, 0, true, LINEAR, ACC>(P, st, 0, c, eps, inv_h, out, st);
    else
      adv_run<8, 0, 2, true, LINEAR, ACC>(P, st, 0, c, eps, inv_h, out, st);
  } else {
    if (cls == 1)
      adv_run<8, 0, 0, true, LINEAR, ACC>(P, st, 0, c, eps, inv_h, out, st);
    else if (cls == 0 && m == 1)
      adv_run<8, 3, 3, false, LINEAR, ACC>(P, st, wrap, c, eps, inv_h, out, st);
    else if (cls == 0)
      adv_run<8, 3, 0, false, LINEAR, ACC>(P, st, wrap, c, eps, inv_h, out, st);
    else
      adv_run<8, 0, 3, false, LINEAR, ACC>(P, st, wrap, c, eps, inv_h, out, st);
  }
}

// warp tasks of one or two sweeps: task t -> (sweep s, class c, chunk)
struct TaskMap {
  int cum[9];  // cumulative warp tasks over (sweep, class)
  int r0[8], nr[8];
};

__device__ __forceinline__ void make_taskmap(TaskMap& tm, const SweepGeom* g, int nsweeps) {
  tm.cum[0] = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int s = k >> 2;
    int r0 = 0, nr = 0;
    if (s < nsweeps) class_runs(g[s], k & 3, r0, nr);
    tm.r0[k] = r0;
    tm.nr[k] = nr;
    tm.cum[k + 1] = tm.cum[k] + ((s < nsweeps) ? (nr * g[s].nlines + 31) >> 5 : 0);
  }
}

// ---------------------------------------------------------------------------
// x pass: dims (0, 1) of C velocity points over the whole periodic x-plane
// ---------------------------------------------------------------------------
template <bool LINEAR>
__global__ void __launch_bounds__(kP4Threads, 2) xpass4d_kernel(const Plane4Params p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  const int4 tk = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  const int v0 = tk.y, nc = tk.z, cs = tk.w, C = 1 << cs;
  const int n1 = M->ext[0], n2 = M->ext[1], n4 = M->ext[3];
  const int V = M->ext[2] * n4;
  const int NT = (n1 * n2) << cs;
  extern __shared__ __align__(16) double sm[];
  double* U = sm;
  double* D = sm + NT;
  __shared__ double ca[kP4MaxC], cb[kP4MaxC];
  const int tid = threadIdx.x;
  const double* src = p.uin + M->offset + v0;
  for (int e = tid; e < NT; e += kP4Threads) {
    const int pp = e >> cs, c = e & (C - 1);
    cp_async8(U + e, src + pp * V + min(c, nc - 1), c < nc);
  }
  cp_async_commit();
  if (tid < C) {  // x_j lines at velocity point vl: coefficient v_j (models.hpp:341-344)
    const int vl = v0 + min(tid, nc - 1);
    const int i3 = vl / n4;
    ca[tid] = line_coef(p.flux_a, M, 0, p.space_dim, i3, p.c_a, p.efield);
    cb[tid] = line_coef(p.flux_b, M, 1, p.space_dim, vl - i3 * n4, p.c_b, p.efield);
  }
  cp_async_wait<0>();
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  // phase A: x2 lines (x1, c), stride C, n2 points; phase B: x1 lines (x2, c) = l,
  // stride n2 C, n1 points, accumulated
  for (int ph = 0; ph < 2; ++ph) {
    SweepGeom g;
    g.nlines = (ph == 0 ? n1 : n2) << cs;
    g.m = (ph == 0 ? n2 : n1) >> 3;
    g.zero = 0;
    g.inv_nl = 1.0f / (float)g.nlines;
    __shared__ TaskMap tm;
    if (tid == 0) make_taskmap(tm, &g, 1);
    __syncthreads();
    const int st = (ph == 0) ? C : (n2 << cs);
    const int wrap = (ph == 0 ? n2 : n1) * st;
    const double inv_h = M->inv_h[ph == 0 ? 1 : 0];
    for (int t = warp; t < tm.cum[4]; t += kP4Threads / 32) {
      int k = 0;
      while (t >= tm.cum[k + 1]) ++k;
      const int i = ((t - tm.cum[k]) << 5) + lane;
      if (i >= tm.nr[k] * g.nlines) continue;
      const int q = qdiv(i, g.inv_nl);
      const int l = i - q * g.nlines, r = tm.r0[k] + q;
      const int c = l & (C - 1);
      const int base = (ph == 0) ? (l >> cs) * (n2 << cs) + c : l;
      const double* P = U + base + (8 * r - 3) * st;
      double* o = D + base + 8 * r * st;
      if (ph == 0)
        run_dispatch<false, LINEAR, false>(k, g.m, P, st, wrap, cb[c], p.eps, inv_h, o);
      else
        run_dispatch<false, LINEAR, true>(k, g.m, P, st, wrap, ca[c], p.eps, inv_h, o);
    }
    __syncthreads();
  }
  // K = (0 - dx1) - dx2 (in the order dx2 + dx1 of the sweeps; fast build)
  double* kb = p.kbuf + M->offset + v0;
  for (int e = tid; e < NT; e += kP4Threads) {
    const int pp = e >> cs, c = e & (C - 1);
    if (c < nc) kb[pp * V + c] = 0.0 - D[e];
  }
}

// ---------------------------------------------------------------------------
// v pass: dims (2, 3) of G whole velocity planes + RK stage + charge density
// ---------------------------------------------------------------------------
template <bool LINEAR>
__global__ void __launch_bounds__(kP4Threads, 2) vpass4d_kernel(const Plane4Params p) {
  pdl_wait();
  const StepCtl* ctl = p.ctl;
  if (ctl != nullptr && !ctl->active) return;
  const int4 tk = p.tiles[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  const int x0 = tk.y, G = tk.z;
  const int n3 = M->ext[2], n4 = M->ext[3];
  const int V = n3 * n4;
  const int NT = G * V;
  extern __shared__ __align__(16) double sm[];
  __shared__ unsigned long long bar;
  __shared__ double ce1[kP4MaxG], ce2[kP4MaxG];
  const int tid = threadIdx.x;
  const long long gs = M->offset + (long long)x0 * V;  // tile start (doubles)
  const long long ga = gs & ~1LL;                         // 16-byte aligned start
  const int shift = (int)(gs - ga);
  const unsigned nbytes = (unsigned)((((gs + NT + 1) & ~1LL) - ga) * 8);
  const int pitch = (NT + 3) & ~1;
  double* U = sm + shift;
  double* DV1 = sm + pitch;
  double* DV2 = DV1 + pitch;
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (tid == 0) bulk_g2s(sm, p.uin + ga, nbytes, &bar);
  if (tid < G) {  // v_j lines at x point x0+tid: -E_j(x) (VP) or the advection speed
    ce1[tid] = line_coef(p.flux_a, M, 2, p.space_dim, x0 + tid, p.c_a, p.efield);
    ce2[tid] = line_coef(p.flux_b, M, 3, p.space_dim, x0 + tid, p.c_b, p.efield);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  const int lane = tid & 31, warp = tid >> 5;
  {
    // sweep 0: v2 lines (rows rho = g n3 + i3), unit stride, n4 points;
    // sweep 1: v1 lines (columns kappa = g n4 + i4), stride n4, n3 points
    SweepGeom g[2];
    g[0].nlines = G * n3;
    g[0].m = n4 >> 3;
    g[1].nlines = G * n4;
    g[1].m = n3 >> 3;
    g[0].zero = g[1].zero = 1;
    g[0].inv_nl = 1.0f / (float)g[0].nlines;
    g[1].inv_nl = 1.0f / (float)g[1].nlines;
    __shared__ TaskMap tm;
    if (tid == 0) make_taskmap(tm, g, 2);
    __syncthreads();
    const float i3f = 1.0f / (float)n3, i4f = 1.0f / (float)n4;
    const double ih3 = M->inv_h[2], ih4 = M->inv_h[3];
    for (int t = warp; t < tm.cum[8]; t += kP4Threads / 32) {
      int k = 0;
      while (t >= tm.cum[k + 1]) ++k;
      const int s = k >> 2, cls = k & 3;
      const int i = ((t - tm.cum[k]) << 5) + lane;
      if (i >= tm.nr[k] * g[s].nlines) continue;
      const int q = qdiv(i, g[s].inv_nl);
      const int l = i - q * g[s].nlines, r = tm.r0[k] + q;
      if (s == 0) {
        const int gx = qdiv(l, i3f);
        const int base = l * n4 + 8 * r;
        run_dispatch<true, LINEAR, false>(cls, g[0].m, U + base - 3, 1, 0, ce2[gx], p.eps, ih4,
                                          DV2 + base);
      } else {
        const int gx = qdiv(l, i4f);
        const int base = gx * V + (l - gx * n4) + 8 * r * n4;
        run_dispatch<true, LINEAR, false>(cls, g[1].m, U + base - 3 * n4, n4, 0, ce1[gx], p.eps,
                                          ih3, DV1 + base);
      }
    }
  }
  __syncthreads();
  // epilogue: k = (K - dv1) - dv2, RK stage (timestep.hpp:86-104), non-finite
  // check, output; trapezoid-weighted stage output for the charge density
  const double* kb = p.kbuf + gs;
  const double* un = p.un + gs;
  double* out = p.out + gs;
  const double dt = (ctl != nullptr) ? ctl->dt : 0.0;
  const bool moment = (p.rho_parts != nullptr) && (p.stage > 0);
  const float iVf = 1.0f / (float)V, i4f = 1.0f / (float)n4;
  const double h3 = M->h[2], h4 = M->h[3];
  bool bad = false;
  for (int e0 = tid; e0 < NT; e0 += 4 * kP4Threads) {
    double kin[4], unv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = e0 + j * kP4Threads;
      kin[j] = (e < NT) ? __ldg(kb + e) : 0.0;
      unv[j] = (e < NT && p.stage > 1) ? __ldg(un + e) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = e0 + j * kP4Threads;
      if (e >= NT) break;
      const double kv = (kin[j] - DV1[e]) - DV2[e];
      double o;
      if (p.stage == 0) {
        o = kv;
      } else {
        bad |= !isfinite(kv);
        const double ui = U[e];
        if (p.stage == 1)
          o = fma(dt, kv, ui);
        else if (p.stage == 2)
          o = fma(0.75, unv[j], 0.25 * fma(dt, kv, ui));
        else
          o = fma(1.0 / 3.0, unv[j], (2.0 / 3.0) * fma(dt, kv, ui));
      }
      out[e] = o;
      if (moment) {  // trapezoid weights of the velocity block (models.hpp:64-71,240-257)
        const int gx = qdiv(e, iVf), rr = e - gx * V;
        const int a = qdiv(rr, i4f), b = rr - a * n4;
        const double wa = (a == 0 || a == n3 - 1) ? 0.5 * h3 : h3;
        const double wb = (b == 0 || b == n4 - 1) ? 0.5 * h4 : h4;
        DV1[e] = (wa * wb) * o;
      }
    }
  }
  if (bad) {
    const unsigned long long code =
        (unsigned long long)ctl->cur_step * 4ull + (unsigned long long)p.stage;
    atomicMin(p.fail + tk.x, code);
  }
  if (moment) {  // one warp per x point, fixed order
    __syncthreads();
    for (int gx = warp; gx < G; gx += kP4Threads / 32) {
      const double* w = DV1 + gx * V;
      double acc = 0.0;
      for (int e = lane; e < V; e += 32) acc += w[e];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) p.rho_parts[(M->xoff + x0 + gx) * kRhoParts] = acc;
    }
  }
  if (p.dtp != nullptr) fused_step_dt(p.dtp, p.counter);
}

cudaError_t launch_plane4(const Plane4Params& p, int pass, int nblocks, size_t smem,
                          cudaStream_t s) {
  if (nblocks <= 0) return cudaSuccess;
  if (pass == 0)
    return p.linear ? launch_k(xpass4d_kernel<true>, dim3(nblocks), dim3(kP4Threads), smem, s, p)
                    : launch_k(xpass4d_kernel<false>, dim3(nblocks), dim3(kP4Threads), smem, s, p);
  return p.linear ? launch_k(vpass4d_kernel<true>, dim3(nblocks), dim3(kP4Threads), smem, s, p)
                  : launch_k(vpass4d_kernel<false>, dim3(nblocks), dim3(kP4Threads), smem, s, p);
}

cudaError_t configure_plane4() {
  const int maxs = 200 * 1024;
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(xpass4d_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                maxs)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(xpass4d_kernel<false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, maxs)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(vpass4d_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                maxs)) != cudaSuccess)
    return e;
  return cudaFuncSetAttribute(vpass4d_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              maxs);
}
