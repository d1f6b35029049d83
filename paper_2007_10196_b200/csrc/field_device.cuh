// field_device.cuh -- Vlasov-Poisson field device code (BASELINE C4/C5), shared
// by the field kernels (k_field.cu) and the persistent 2D kernel (kernels.cuh).
//
// NEW PHYSICS: the reference has no Poisson solver.  This
// follows the kinetic template of vb_rhs_into (models.hpp:334-363): the
// charge density uses the reference's trapezoid weights over the contiguous
// velocity block (moment_density models.hpp:294-306, block_weights 240-257,
// trapezoid_weights_1d 64-71), rho(x) = 1 - sum_v w_v f(x, v); the field solves
// -lap(phi) = rho, E = -grad(phi) spectrally on the member's own periodic
// x-grid (mean and Nyquist modes dropped), as the oracle restatement
// oracle/sgw_oracle.c:spectral_poisson does with a direct DFT.
//
// COH = true: loads of data written by other CTAs of the same (persistent)
// launch go through L2 (ld.global.cg).
#pragma once
#include <math.h>

#include "sgwg_internal.h"

namespace sgwg {

#ifndef SGWG_FIELD_THREADS
#define SGWG_FIELD_THREADS 512
#endif
constexpr int kFieldThreads = SGWG_FIELD_THREADS;
constexpr int kFieldMaxX = 2048;
constexpr int kFieldSmemDoubles = 6 * kFieldMaxX + 2 * kFieldMaxX;  // + 2 x 2H twiddles

template <bool COH>
__device__ __forceinline__ double fld_ld(const double* p) {
  return COH ? __ldcg(p) : __ldg(p);
}

__device__ __forceinline__ int bitrev(int x, int bits) {
  return (int)(__brev((unsigned)x) >> (32 - bits));
}

// radix-2 FFTs of all lines along `axis` (1 = x2, contiguous) of NA complex
// n1 x n2 arrays (re[k], im[k]) at once; n1 = 2^b1, n2 = 2^b2.  DIF (forward,
// sign -1): natural order in, bit-reversed order out; DIT (inverse, sign +1,
// unnormalised): bit-reversed in, natural out -- so no bit-reversal pass is
// needed, and the spectral step works in bit-reversed order.  Twiddles from the
// stage-major table T[half + pos] = e^{i pi pos/half} (consecutive lanes read
// consecutive entries: no shared-memory bank conflicts).
// Two consecutive radix-2 stages are done per barrier: a thread loads the four
// elements the two stages couple, applies both stages in registers and stores
// them back -- the same floating-point operations in the same order as two
// separate stages (bitwise identical), half the barriers and shared-memory
// round trips; an odd stage count leaves one single stage.
template <int NA, bool DIF>
__device__ inline void fft_lines(double* const* re, double* const* im, int b1, int b2, int axis,
                                 const double* tc, const double* ts) {
  const int bits = axis ? b2 : b1;
  if (bits == 0) return;
  const int len = 1 << bits;
  const int nx = 1 << (b1 + b2);
  const int stride = axis ? 1 : (1 << b2);
  const double sign = DIF ? -1.0 : 1.0;
  auto base_of = [&](int line) { return axis ? (line << b2) : line; };
  // lanes walk positions along contiguous lines (axis 1) and walk lines when
  // the lines are strided (axis 0), so shared-memory accesses stay conflict-free
  const int lbits = b1 + b2 - bits;  // log2(number of lines)
  // (a, b) -> (a + b, (a - b) w)   [DIF]   /   (a + b w, a - b w)   [DIT]
  auto bfly = [&](double& ar, double& ai, double& xr, double& xi, double c, double s) {
    if (DIF) {
      const double dr = ar - xr, di = ai - xi;
      ar = ar + xr;
      ai = ai + xi;
      xr = dr * c - di * s;
      xi = dr * s + di * c;
    } else {
      const double br = xr * c - xi * s, bi = xr * s + xi * c;
      xr = ar - br;
      xi = ai - bi;
      ar = ar + br;
      ai = ai + bi;
    }
  };
  int st = 0;
  for (; st + 1 < bits; st += 2) {  // stage pairs
    // DIF: halves h, h/2 (h = 2^(bits-1-st)); DIT: halves h, 2h (h = 2^st)
    const int lh = DIF ? bits - 1 - st : st;
    const int h = 1 << lh;
    const int qb = DIF ? lh - 1 : lh;  // log2(quads per group)
    for (int bf = threadIdx.x; bf < nx / 4; bf += blockDim.x) {
      const int line = axis ? bf >> (bits - 2) : bf & ((1 << lbits) - 1);
      const int q = axis ? bf & ((len >> 2) - 1) : bf >> lbits;
      const int grp = q >> qb, pos = q & ((1 << qb) - 1);
      int ia, ib, ic, id;  // element indices
      double c1, s1, c2, s2, c3, s3;
      if (DIF) {  // group of 2h: a = p, b = p + h/2, c = p + h, d = p + 3h/2
        ia = base_of(line) + ((grp << (lh + 1)) + pos) * stride;
        ib = ia + (h >> 1) * stride;
        ic = ia + h * stride;
        id = ib + h * stride;
        c1 = tc[h + pos], s1 = sign * ts[h + pos];                        // (a, c)
        c2 = tc[h + pos + (h >> 1)], s2 = sign * ts[h + pos + (h >> 1)];  // (b, d)
        c3 = tc[(h >> 1) + pos], s3 = sign * ts[(h >> 1) + pos];          // (a, b), (c, d)
      } else {    // group of 4h: a = p, b = p + h, c = p + 2h, d = p + 3h
        ia = base_of(line) + ((grp << (lh + 2)) + pos) * stride;
        ib = ia + h * stride;
        ic = ib + h * stride;
        id = ic + h * stride;
        c1 = tc[h + pos], s1 = sign * ts[h + pos];                        // (a, b), (c, d)
        c2 = tc[2 * h + pos], s2 = sign * ts[2 * h + pos];                // (a, c)
        c3 = tc[2 * h + pos + h], s3 = sign * ts[2 * h + pos + h];        // (b, d)
      }
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        double ar = re[k][ia], ai = im[k][ia], br = re[k][ib], bi = im[k][ib];
        double cr = re[k][ic], ci = im[k][ic], dr = re[k][id], di = im[k][id];
        if (DIF) {
          bfly(ar, ai, cr, ci, c1, s1);
          bfly(br, bi, dr, di, c2, s2);
          bfly(ar, ai, br, bi, c3, s3);
          bfly(cr, ci, dr, di, c3, s3);
        } else {
          bfly(ar, ai, br, bi, c1, s1);
          bfly(cr, ci, dr, di, c1, s1);
          bfly(ar, ai, cr, ci, c2, s2);
          bfly(br, bi, dr, di, c3, s3);
        }
        re[k][ia] = ar, im[k][ia] = ai, re[k][ib] = br, im[k][ib] = bi;
        re[k][ic] = cr, im[k][ic] = ci, re[k][id] = dr, im[k][id] = di;
      }
    }
    __syncthreads();
  }
  if (st < bits) {  // last single stage
    const int lh = DIF ? bits - 1 - st : st;
    const int half = 1 << lh;
    for (int bf = threadIdx.x; bf < nx / 2; bf += blockDim.x) {
      const int line = axis ? bf >> (bits - 1) : bf & ((1 << lbits) - 1);
      const int q = axis ? bf & ((len >> 1) - 1) : bf >> lbits;
      const int grp = q >> lh, pos = q & (half - 1);
      const int i0 = base_of(line) + ((grp << (lh + 1)) + pos) * stride;
      const int i1 = i0 + half * stride;
      const double c = tc[half + pos], s = sign * ts[half + pos];  // e^{sign i pi pos/half}
#pragma unroll
      for (int k = 0; k < NA; ++k) {
        double ar = re[k][i0], ai = im[k][i0], xr = re[k][i1], xi = im[k][i1];
        bfly(ar, ai, xr, xi, c, s);
        re[k][i0] = ar, im[k][i0] = ai, re[k][i1] = xr, im[k][i1] = xi;
      }
    }
    __syncthreads();
  }
}

// Partial charge-density sum of one x point over velocity chunk `part` of
// M->rparts equal chunks: sum_v w_v f(x_i, v) (rho = 1 - sum of the partials),
// computed by one warp (lanes stride the contiguous chunk, 4 loads in flight,
// fixed reduction order).  Trapezoid weights of the velocity block
// (moment_density models.hpp:294-306, block_weights 240-257).
template <bool COH>
__device__ inline void moment_part(const FieldParams& p, const MemberDesc* M, int xi, int part) {
  const int dx = p.space_dim;
  const int lane = threadIdx.x & 31;
  const int vn = M->vn;
  const int chunk = (vn + M->rparts - 1) / M->rparts;
  const int v0 = part * chunk, v1 = min(vn, v0 + chunk);
  const int ev0 = M->ext[dx], ev1 = (dx == 2) ? M->ext[dx + 1] : 1;
  const double hv0 = M->h[dx], hv1 = (dx == 2) ? M->h[dx + 1] : 1.0;
  const int zb0 = M->bc[dx], zb1 = (dx == 2) ? M->bc[dx + 1] : 0;
  const double* block = p.f + M->offset + (long long)xi * vn;
  const float inv_ev1 = 1.0f / (float)ev1;
  auto weight = [&](int vi) {
    const int i0 = (int)(((float)vi + 0.5f) * inv_ev1), i1 = vi - i0 * ev1;
    double w0 = hv0, w1 = hv1;
    if (zb0 == 1 && (i0 == 0 || i0 == ev0 - 1)) w0 *= 0.5;
    if (dx == 2 && zb1 == 1 && (i1 == 0 || i1 == ev1 - 1)) w1 *= 0.5;
    return (dx == 2) ? w0 * w1 : w0;
  };
  double acc = 0.0;
  for (int vb = v0 + lane; vb < v1; vb += 4 * 32) {
    double v[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) v[b] = (vb + 32 * b < v1) ? fld_ld<COH>(block + vb + 32 * b) : 0.0;
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (vb + 32 * b < v1) acc = fma(weight(vb + 32 * b), v[b], acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) p.rho_parts[(M->xoff + xi) * kRhoParts + part] = acc;
}

// E of member mi from its rho partials (whole block; sh >= kFieldSmemDoubles
// doubles; red >= 2 * blockDim/32 doubles); also p.rho and
// p.emax[mi*dx + comp] = max|E_comp|.  Both field components are transformed
// back together.
#ifdef SGWG_TRACE
__device__ long long sgwg_ftrace[128][8];  // per member: phase clocks of the last field launch
#define SGWG_FMARK(mi, ph) \
  if (threadIdx.x == 0 && (mi) < 128) sgwg_ftrace[mi][ph] = clock64()
#else
#define SGWG_FMARK(mi, ph)
#endif

template <bool COH>
__device__ inline void field_member(const FieldParams& p, int mi, double* sh, double* red) {
  SGWG_FMARK(mi, 0);
  const MemberDesc* M = p.mem + mi;
  const int dx = p.space_dim;
  const int n1 = M->xext[0], n2 = M->xext[1];
  const int b1 = __ffs(n1) - 1, b2 = __ffs(n2) - 1;
  const int nx = M->nx;
  double* rr = sh;
  double* ri = sh + nx;
  double* er[2] = {sh + 2 * nx, sh + 4 * nx};
  double* ei[2] = {sh + 3 * nx, sh + 5 * nx};
  const int H = max(1, max(n1, n2) / 2);
  double* twc = sh + 6 * nx;  // stage-major twiddles, 2H each
  double* tws = twc + 2 * H;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // the phase's loads (charge-density partials of two x points, two twiddle
  // entries per thread and round) all in flight before any use
  // twiddles: T[half + pos] = e^{i pi pos/half} = family table entry
  // e^{i pi q/hmax}, q = pos hmax/half (half = 1 .. H; hmax a power of two)
  const int lhmax = 31 - __clz(p.hmax);
  const int span = 2 * blockDim.x;
  for (int r0 = 0; r0 < max(nx, 2 * H); r0 += span) {
    double v[2][kRhoParts], c[2], sn[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = r0 + threadIdx.x + u * blockDim.x;
      const bool okt = e > 0 && e < 2 * H;
      const int k = 31 - __clz(max(e, 1));
      const int q = (e - (1 << k)) << (lhmax - k);
      c[u] = okt ? fld_ld<COH>(p.twid + q) : 0.0;
      sn[u] = okt ? fld_ld<COH>(p.twid + p.hmax + q) : 0.0;
      const double* pt = p.rho_parts + (M->xoff + e) * kRhoParts;
#pragma unroll
      for (int t = 0; t < kRhoParts; ++t)
        v[u][t] = (e < nx && t < M->rparts) ? fld_ld<COH>(pt + t) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = r0 + threadIdx.x + u * blockDim.x;
      if (e > 0 && e < 2 * H) {
        twc[e] = c[u];
        tws[e] = sn[u];
      }
      if (e < nx) {
        double acc = v[u][0];
#pragma unroll
        for (int t = 1; t < kRhoParts; ++t)
          if (t < M->rparts) acc += v[u][t];
        const double r = 1.0 - acc;
        p.rho[M->xoff + e] = r;
        rr[e] = r;
        ri[e] = 0.0;
      }
    }
  }
  __syncthreads();
  SGWG_FMARK(mi, 1);
  {  // forward, output in bit-reversed order along both axes
    double* R[1] = {rr};
    double* I[1] = {ri};
    fft_lines<1, true>(R, I, b1, b2, 1, twc, tws);
    fft_lines<1, true>(R, I, b1, b2, 0, twc, tws);
  }
  SGWG_FMARK(mi, 2);
  const double two_pi = 6.283185307179586476925286766559;
  for (int id = threadIdx.x; id < nx; id += blockDim.x) {  // bit-reversed storage order
    const int k1 = (b1 > 0) ? bitrev(id >> b2, b1) : 0;
    const int k2 = (b2 > 0) ? bitrev(id & (n2 - 1), b2) : 0;
    const int s1 = (k1 <= n1 / 2) ? k1 : k1 - n1;
    const int s2 = (k2 <= n2 / 2) ? k2 : k2 - n2;
    const bool nyq = ((n1 % 2 == 0) && k1 == n1 / 2 && n1 > 1) ||
                     ((n2 % 2 == 0) && k2 == n2 / 2 && n2 > 1);
    const double kap1 = two_pi * (double)s1 / p.L[0];
    const double kap2 = (dx == 2) ? two_pi * (double)s2 / p.L[1] : 0.0;
    const bool drop = (s1 == 0 && s2 == 0) || nyq;
    const double inv = drop ? 0.0 : 1.0 / (kap1 * kap1 + kap2 * kap2);
    for (int comp = 0; comp < dx; ++comp) {
      const double kc = (comp == 0) ? kap1 : kap2;
      er[comp][id] = drop ? 0.0 : kc * ri[id] * inv;  // -i kc rhat / |k|^2
      ei[comp][id] = drop ? 0.0 : -kc * rr[id] * inv;
    }
  }
  __syncthreads();
  SGWG_FMARK(mi, 3);
  if (dx == 2) {  // inverse, bit-reversed in, natural out
    fft_lines<2, false>(er, ei, b1, b2, 0, twc, tws);
    fft_lines<2, false>(er, ei, b1, b2, 1, twc, tws);
  } else {
    fft_lines<1, false>(er, ei, b1, b2, 0, twc, tws);
    fft_lines<1, false>(er, ei, b1, b2, 1, twc, tws);
  }
  SGWG_FMARK(mi, 4);
  double lmax[2] = {0.0, 0.0};
  const double inv_n = 1.0 / (double)nx;
  for (int comp = 0; comp < dx; ++comp) {
    double* E = p.efield + M->xoff * dx + (long long)comp * nx;
    // the ring copy of the step-start field (batched energy record)
    double* E2 = (p.ering != nullptr)
                     ? p.ering + (p.ctl->step % p.ering_slots) * p.ering_stride + M->xoff * dx +
                           (long long)comp * nx
                     : nullptr;
    for (int id = threadIdx.x; id < nx; id += blockDim.x) {
      const double e = er[comp][id] * inv_n;
      E[id] = e;
      if (E2 != nullptr) E2[id] = e;
      lmax[comp] = fmax(lmax[comp], fabs(e));
    }
  }
#pragma unroll
  for (int comp = 0; comp < 2; ++comp) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
      lmax[comp] = fmax(lmax[comp], __shfl_xor_sync(0xffffffffu, lmax[comp], o));
    if (lane == 0) red[comp * nwarps + warp] = lmax[comp];
  }
  __syncthreads();
  if (threadIdx.x < dx) {
    double m = 0.0;
    for (int q = 0; q < nwarps; ++q) m = fmax(m, red[threadIdx.x * nwarps + q]);
    p.emax[mi * dx + threadIdx.x] = m;
  }
  SGWG_FMARK(mi, 5);
}

// degree-4 Lagrange weights in the reference's cell form (interp.hpp:36-53
// with OffsetTable::cell_weights, interp.hpp:119-122) for fine index j of a
// periodic line refined by 2^m: 5 source indices i-2..i+2 and weights.
__device__ __forceinline__ void lagrange5(int j, int m, int n_src, int* idx, double* w) {
  const int f = 1 << m, r = j & (f - 1), i = j >> m;
  const double t = (double)r / f;
  for (int q = 0; q < 5; ++q) idx[q] = ((i - 2 + q) % n_src + n_src) % n_src;
  if (r == 0) {
    for (int q = 0; q < 5; ++q) w[q] = (q == 2) ? 1.0 : 0.0;
    return;
  }
  const double c0 = (t - 1.0) * (t - 2.0) / 12.0, c1 = (4.0 - t * t) / 6.0,
               c2 = (t + 2.0) * (t + 1.0) / 12.0;
  // sum_k c_k p_k(t) expanded into point weights (substencil_values, interp.hpp:45-53)
  const double a0 = 0.5 * (t + 1.0) * t, a1 = -(t + 2.0) * t, a2 = 0.5 * (t + 2.0) * (t + 1.0);
  const double b1 = 0.5 * t * (t - 1.0), b2 = -(t + 1.0) * (t - 1.0), b3 = 0.5 * (t + 1.0) * t;
  const double e2 = 0.5 * (t - 1.0) * (t - 2.0), e3 = -t * (t - 2.0), e4 = 0.5 * t * (t - 1.0);
  w[0] = c0 * a0;
  w[1] = c0 * a1 + c1 * b1;
  w[2] = c0 * a2 + c1 * b2 + c2 * e2;
  w[3] = c1 * b3 + c2 * e3;
  w[4] = c2 * e4;
}

// Members that share an x-grid are combined on that grid before interpolating
// (interpolation is linear): per group g, Eg_c = sum_{m in g} c_m E_m,c in
// member order (one thread per group x point).
template <bool COH>
__device__ inline void group_point(const FieldParams& p, const double* coef, int X) {
  int g = 0;
  while (g + 1 < p.negrp && p.egrp[g + 1].w <= X) ++g;
  const int4 G = p.egrp[g];
  const int nxg = G.x * G.y, xi = X - G.w;
  const int dx = p.space_dim;
  const int2 mr = p.egrp_m[g];
  for (int c = 0; c < dx; ++c) {
    double acc = 0.0;
    for (int k = 0; k < mr.y; ++k) {
      const int mi = p.egrp_mem[mr.x + k];
      const MemberDesc* M = p.mem + mi;
      acc = fma(coef[mi], fld_ld<COH>(p.efield + M->xoff * dx + (long long)c * M->nx + xi), acc);
    }
    p.egrid[G.z + c * nxg + xi] = acc;
  }
}

// h-weighted |E_c|^2 contribution of finest x point q, computed by one thread
// (WARP = false: consecutive threads take consecutive points, so the loads of
// one group coalesce) or by one warp (WARP: lanes over the members, warp-reduced
// in a fixed order, every lane returns the value; small families):
// E_c = sum_g I_g(Eg), I_g separable degree-4 Lagrange
// interpolation from group g's x-grid (or, without groups, E_c =
// sum_m c_m I_m(E_m) member by member).
template <bool COH, bool WARP>
__device__ inline double energy_point(const FieldParams& p, int q, int fine0, int fine1) {
  const int dx = p.space_dim;
  const int lane = WARP ? (threadIdx.x & 31) : 0;
  const int lstep = WARP ? 32 : 1;
  const int i = q / fine1, j = q - (q / fine1) * fine1;
  double ec[2] = {0.0, 0.0};
  const bool direct = (p.negrp == 0);  // small families: every member, no group pass
  const int ng = direct ? p.nmembers : p.negrp;
  for (int g = lane; g < ng; g += lstep) {
    const MemberDesc* M = p.mem + g;
    const int4 G = direct ? make_int4(M->xext[0], M->xext[1], 0, 0) : p.egrp[g];
    const int n0 = G.x, n1 = G.y;
    int ia[5], ja[5];
    double wa[5], wb[5];
    lagrange5(i, __ffs(fine0 / n0) - 1, n0, ia, wa);
    if (dx == 2) {
      lagrange5(j, __ffs(fine1 / n1) - 1, n1, ja, wb);
    } else {
      for (int b = 0; b < 5; ++b) ja[b] = 0, wb[b] = (b == 2) ? 1.0 : 0.0;
    }
    for (int c = 0; c < dx; ++c) {
      const double* E = direct ? p.efield + M->xoff * dx + (long long)c * M->nx
                               : p.egrid + G.z + c * n0 * n1;
      double v = 0.0;
      for (int a = 0; a < 5; ++a) {
        double s = 0.0;
        for (int b = 0; b < 5; ++b) s = fma(wb[b], fld_ld<COH>(E + ia[a] * n1 + ja[b]), s);
        v = fma(wa[a], s, v);
      }
      if (direct)
        ec[c] = fma(p.ecoef[g], v, ec[c]);
      else
        ec[c] += v;
    }
  }
  if (WARP) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ec[0] += __shfl_xor_sync(0xffffffffu, ec[0], o);
      ec[1] += __shfl_xor_sync(0xffffffffu, ec[1], o);
    }
  }
  double acc = 0.0;
  for (int c = 0; c < dx; ++c) acc = fma(ec[c], ec[c], acc);
  return acc;
}

}  // namespace sgwg
