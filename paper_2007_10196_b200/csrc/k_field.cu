// k_field.cu -- Vlasov-Poisson field kernels of every member (BASELINE C4/C5);
// the device code is in field_device.cuh (shared with the persistent kernel).
//
// moment_kernel: rho of every x point (one warp each, many CTAs).
// field_kernel:  one CTA per member: the x-grid has <= 2048 points (C4: 32*2^l;
//                C5: (8*2^l1)x(8*2^l2), l1+l2 <= 5), so the 2D FFT lives in
//                shared memory.
// field_energy_kernel: per-step ||E_c||_2 diagnostic.
#include <cstdlib>

#include "field_device.cuh"
#include "pdl.cuh"

namespace sgwg {

__global__ void __launch_bounds__(256) moment_kernel(const FieldParams p) {
  pdl_wait();
  if (p.ctl != nullptr && !p.ctl->active) return;
  const int2 tk = p.mtasks[blockIdx.x];
  const MemberDesc* M = p.mem + tk.x;
  const int item = tk.y + (threadIdx.x >> 5);  // (x point, velocity chunk)
  if (item >= M->nx * M->rparts) return;
  moment_part<false>(p, M, item / M->rparts, item % M->rparts);
}

__global__ void __launch_bounds__(kFieldThreads) field_kernel(const FieldParams p) {
  pdl_wait();
  if (p.ctl != nullptr && !p.ctl->active) return;
  extern __shared__ double sh[];
  __shared__ double red[2 * kFieldThreads / 32];
  field_member<false>(p, blockIdx.x, sh, red);
}

__global__ void __launch_bounds__(256) group_field_kernel(const FieldParams p, const double* coef) {
  pdl_wait();
  if (p.ctl != nullptr && !p.ctl->active) return;
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  if (X < p.ngx) group_point<false>(p, coef, X);
}

__global__ void __launch_bounds__(256) field_energy_kernel(const FieldParams p, int fine0,
                                                           int fine1, double hvol,
                                                           double* out_base, long long cap) {
  pdl_wait();
  if (p.ctl != nullptr && !p.ctl->active) return;
  // launched after the step's dt kernel: the step being taken is step - 1
  const long long slot = (p.ctl != nullptr) ? p.ctl->step - 1 : 0;
  if (slot >= cap) return;
  double acc = 0.0;
  if (p.negrp > 0) {  // groups (large fine grids): one thread per finest x point
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < fine0 * fine1;
         q += gridDim.x * blockDim.x)
      acc += energy_point<false, false>(p, q, fine0, fine1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  } else {  // members directly (small families): one warp per finest x point
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); q < fine0 * fine1;
         q += warps)
      acc += energy_point<false, true>(p, q, fine0, fine1);
  }
  if ((threadIdx.x & 31) == 0) atomicAdd(out_base + slot, acc * hvol);
}

// Per-step ||E||^2 record of 2D-in-x families with member groups, one kernel: a CTA
// per finest x row i.  (1) per group g and component c, the group's E combined
// over its members (sum_m c_m E_m in member order) and interpolated along x1 to
// row i: T_g[c][j'] = sum_a w_a(i) Eg[c][ia][j'] (separable degree-4 Lagrange,
// lagrange5); (2) per finest point (i, j): E_c = sum_g sum_b w_b(j) T_g[c][jb],
// accumulate |E|^2; (3) the row's sum into part[i]; the last CTA adds the parts
// in row order (deterministic) and writes the record.  Replaces group_field_kernel
// + field_energy_kernel (57 us per C5 step measured) for the grouped 2D case.
constexpr int kERowMax = 4096;  // doubles of T per CTA (2 x sum_g n1_g)
// the sum of |E|^2 over finest x row i (E packed per member at ef); the result in thread 0
// (eg != nullptr: the groups' combined fields, laid out like p.egrid, computed beforehand
// with the same member-order sums)
__device__ __forceinline__ double energy_row(const FieldParams& p, const double* ef, int i,
                                             int fine0, int fine1, double* T, int* toff,
                                             double* red, const double* eg_grid = nullptr) {
  const int tid = threadIdx.x;
  const int ng = p.negrp;
  if (tid == 0) {
    int o = 0;
    for (int g = 0; g < ng; ++g) {
      toff[g] = o;
      o += 2 * p.egrp[g].y;
    }
    toff[ng] = o;
  }
  __syncthreads();
  const int ntot = toff[ng];
  for (int e = tid; e < ntot; e += blockDim.x) {
    int g = 0;
    while (e >= toff[g + 1]) ++g;
    const int4 G = p.egrp[g];
    const int n0 = G.x, n1 = G.y;
    const int c = (e - toff[g]) / n1, jp = (e - toff[g]) - c * n1;
    int ia[5];
    double wa[5];
    lagrange5(i, __ffs(fine0 / n0) - 1, n0, ia, wa);
    const int2 mr = p.egrp_m[g];
    double v = 0.0;
    for (int a = 0; a < 5; ++a) {
      if (wa[a] == 0.0) continue;
      double eg = 0.0;
      if (eg_grid != nullptr) {
        eg = eg_grid[G.z + c * n0 * n1 + ia[a] * n1 + jp];
      } else {
        for (int k = 0; k < mr.y; ++k) {
          const int mi = p.egrp_mem[mr.x + k];
          const MemberDesc* M = p.mem + mi;
          eg = fma(p.ecoef[mi], ef[M->xoff * 2 + (long long)c * M->nx + ia[a] * n1 + jp], eg);
        }
      }
      v = fma(wa[a], eg, v);
    }
    T[e] = v;
  }
  __syncthreads();
  double acc = 0.0;
  for (int j = tid; j < fine1; j += blockDim.x) {
    double e0 = 0.0, e1 = 0.0;
    for (int g = 0; g < ng; ++g) {
      const int n1 = p.egrp[g].y;
      int jb[5];
      double wb[5];
      lagrange5(j, __ffs(fine1 / n1) - 1, n1, jb, wb);
      const double* Tg = T + toff[g];
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int b = 0; b < 5; ++b) {
        s0 = fma(wb[b], Tg[jb[b]], s0);
        s1 = fma(wb[b], Tg[n1 + jb[b]], s1);
      }
      e0 += s0;
      e1 += s1;
    }
    acc = fma(e0, e0, fma(e1, e1, acc));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  double r = 0.0;
  if (tid == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += red[w];
  return r;
}

__global__ void __launch_bounds__(256) energy_rows_kernel(const FieldParams p, int fine0, int fine1,
                                                          double hvol, double* out_base,
                                                          long long cap, double* part,
                                                          unsigned int* done) {
  pdl_wait();
  if (p.ctl != nullptr && !p.ctl->active) return;
  const long long slot = (p.ctl != nullptr) ? p.ctl->step - 1 : 0;
  if (slot >= cap) return;
  __shared__ double T[kERowMax];
  __shared__ int toff[64];
  __shared__ double red[8];
  __shared__ unsigned int s_last;
  const int i = blockIdx.x, tid = threadIdx.x;
  const double r = energy_row(p, p.efield, i, fine0, fine1, T, toff, red);
  if (tid == 0) {
    part[i] = r;
    __threadfence();
    s_last = (atomicAdd(done, 1u) == gridDim.x - 1) ? 1u : 0u;
  }
  __syncthreads();
  if (s_last && tid == 0) {
    __threadfence();
    double tot = 0.0;
    for (int q = 0; q < (int)gridDim.x; ++q) tot += part[q];
    out_base[slot] = tot * hvol;
    *done = 0u;
  }
}

// Batched form for captured step chunks (one launch at the end of a chunk of <=
// kEnergyRing steps instead of one per step: a per-step launch beside the stage kernels
// displaced their CTAs for ~55 us per C5 step).  The step-start field of step k sits in
// ring slot k % ering_slots (field_member); CTA (i, b) handles row i of step
// k = *recorded + b and does nothing when k >= ctl->step (steps not taken: the chunk ran
// into its stop).  Per step the last row CTA adds the row sums in row order
// (deterministic, the same arithmetic as energy_rows_kernel); the last CTA of the launch
// advances *recorded.  done: kEnergyRing + 1 self-resetting counters.
// Two launches: the groups' combined fields of every step of the batch
// (group_batch_kernel: egrid_b + b * egrid_stride), then the rows.
__global__ void __launch_bounds__(256) group_batch_kernel(const FieldParams p, const double* coef,
                                                          double* egrid_b, long long egrid_stride,
                                                          const long long* recorded) {
  pdl_wait();
  const int b = blockIdx.y;
  const long long k = *recorded + b;
  if (k >= p.ctl->step) return;
  FieldParams q = p;
  q.efield = p.ering + (k % p.ering_slots) * p.ering_stride;
  q.egrid = egrid_b + b * egrid_stride;
  const int X = blockIdx.x * blockDim.x + threadIdx.x;
  if (X < p.ngx) group_point<false>(q, coef, X);
}

// Row i of one step from the groups' combined fields eg (laid out like p.egrid).  Groups
// that share an x2 extent share the x2 interpolation, so their x1-interpolated rows are
// summed first (in group order): T2[class][c][j'] = sum_{g in class} sum_a w_a(i) Eg[c][ia][j'],
// then per finest point E_c = sum_class sum_b w_b(j) T2[class][c][jb].  Lagrange weights
// of every refinement 2^m from a table built once per CTA.  The row's sum in thread 0.
constexpr int kEClsMax = 8;
constexpr int kEWtab = 256;  // sum_m 2^m, m < 8
__device__ __forceinline__ double energy_row_cls(const FieldParams& p, const double* eg, int i,
                                                 int fine0, int fine1, double* T2, double* wtab,
                                                 double (*gwa)[5], int (*gia)[5], int* coff,
                                                 double* red) {
  const int tid = threadIdx.x;
  const int ng = p.negrp, nc = p.ncls;
  // weights of refinement 2^m at phase r: wtab[((1 << m) - 1 + r) * 5 + q]
  const int mmax = __ffs(fine1 / p.cls_n1[0]) - 1;  // classes sorted by ascending extent
  if (tid < (2 << mmax) - 1) {
    const int m = 31 - __clz(tid + 1), r = tid + 1 - (1 << m);
    int idx[5];
    double w[5];
    lagrange5(r, m, 8, idx, w);
#pragma unroll
    for (int q = 0; q < 5; ++q) wtab[tid * 5 + q] = w[q];
  }
  if (tid < ng) {
    const int n0 = p.egrp[tid].x;
    int ia[5];
    double wa[5];
    lagrange5(i, __ffs(fine0 / n0) - 1, n0, ia, wa);
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      gwa[tid][q] = wa[q];
      gia[tid][q] = ia[q];
    }
  }
  if (tid == 0) {
    int o = 0;
    for (int k = 0; k < nc; ++k) {
      coff[k] = o;
      o += 2 * p.cls_n1[k];
    }
    coff[nc] = o;
  }
  __syncthreads();
  const int ntot = coff[nc];
  for (int e = tid; e < ntot; e += blockDim.x) {
    int k = 0;
    while (e >= coff[k + 1]) ++k;
    const int n1 = p.cls_n1[k];
    const int c = (e - coff[k]) >= n1 ? 1 : 0, jp = (e - coff[k]) - c * n1;
    double v = 0.0;
    for (int g = 0; g < ng; ++g) {
      if (p.grp_cls[g] != k) continue;
      const int4 G = p.egrp[g];
      const double* src = eg + G.z + c * G.x * n1 + jp;
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < 5; ++a) s = fma(gwa[g][a], src[gia[g][a] * n1], s);
      v += s;
    }
    T2[e] = v;
  }
  __syncthreads();
  double acc = 0.0;
  for (int j = tid; j < fine1; j += blockDim.x) {
    double e0 = 0.0, e1 = 0.0;
    for (int k = 0; k < nc; ++k) {
      const int n1 = p.cls_n1[k];
      const int m = __ffs(fine1 / n1) - 1;
      const int r = j & ((1 << m) - 1), jc = j >> m;
      const double* w = wtab + ((1 << m) - 1 + r) * 5;
      const double* Tk = T2 + coff[k];
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int b = 0; b < 5; ++b) {
        const int jb = (jc - 2 + b) & (n1 - 1);  // periodic, power-of-two extents
        s0 = fma(w[b], Tk[jb], s0);
        s1 = fma(w[b], Tk[n1 + jb], s1);
      }
      e0 += s0;
      e1 += s1;
    }
    acc = fma(e0, e0, fma(e1, e1, acc));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  double r = 0.0;
  if (tid == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += red[w];
  return r;
}

__global__ void __launch_bounds__(256) energy_rows_batch_kernel(const FieldParams p, int fine0,
                                                                int fine1, double hvol,
                                                                double* out_base, long long cap,
                                                                double* part, unsigned int* done,
                                                                long long* recorded,
                                                                const double* egrid_b,
                                                                long long egrid_stride) {
  pdl_wait();
  __shared__ double T2[1024 + 16];
  __shared__ double wtab[kEWtab * 5];
  __shared__ double gwa[64][5];
  __shared__ int gia[64][5];
  __shared__ int coff[kEClsMax + 1];
  __shared__ double red[8];
  __shared__ unsigned int s_last;
  const int i = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const long long taken = p.ctl->step;
  const long long k = *recorded + b;
  if (k < taken && k < cap) {  // block-uniform
    const double r = energy_row_cls(p, egrid_b + b * egrid_stride, i, fine0, fine1, T2, wtab, gwa,
                                    gia, coff, red);
    if (tid == 0) {
      part[(long long)b * fine0 + i] = r;
      __threadfence();
      s_last = (atomicAdd(done + b, 1u) == gridDim.x - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (s_last && tid == 0) {
      __threadfence();
      double tot = 0.0;
      for (int q = 0; q < fine0; ++q) tot += part[(long long)b * fine0 + q];
      out_base[k] = tot * hvol;
      done[b] = 0u;
    }
  }
  if (tid == 0) {  // every CTA has read *recorded before the last one out rewrites it
    __threadfence();
    if (atomicAdd(done + kEnergyRing, 1u) == gridDim.x * gridDim.y - 1) {
      done[kEnergyRing] = 0u;
      *recorded = taken;
      __threadfence();
    }
  }
}

// Batched record of small families without member groups (1D1V C4: 11 members, 1,024
// finest x points): one CTA per step of the chunk, a thread per finest point over all
// members (energy_point), the block sum in a fixed order.
__global__ void __launch_bounds__(256) energy_direct_batch_kernel(const FieldParams p, int fine0,
                                                                  int fine1, double hvol,
                                                                  double* out_base, long long cap,
                                                                  unsigned int* done,
                                                                  long long* recorded) {
  pdl_wait();
  __shared__ double red[8];
  const int b = blockIdx.x, tid = threadIdx.x;
  const long long taken = p.ctl->step;
  const long long k = *recorded + b;
  if (k < taken && k < cap) {  // block-uniform
    FieldParams q = p;
    q.efield = p.ering + (k % p.ering_slots) * p.ering_stride;
    double acc = 0.0;
    for (int x = tid; x < fine0 * fine1; x += blockDim.x)
      acc += energy_point<false, false>(q, x, fine0, fine1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
      out_base[k] = tot * hvol;
    }
  }
  if (tid == 0) {  // every CTA has read *recorded before the last one out rewrites it
    __threadfence();
    if (atomicAdd(done + kEnergyRing, 1u) == gridDim.x - 1) {
      done[kEnergyRing] = 0u;
      *recorded = taken;
      __threadfence();
    }
  }
}

cudaError_t launch_field_energy_batch_direct(const FieldParams& p, const double* coef, int fine0,
                                             int fine1, double hvol, double* out_base,
                                             long long cap, int nbatch, unsigned int* done,
                                             long long* recorded, cudaStream_t s) {
  FieldParams q = p;
  q.ecoef = coef;
  q.negrp = 0;
  return launch_k(energy_direct_batch_kernel, dim3(nbatch), dim3(256), 0, s, q, fine0, fine1, hvol,
                  out_base, cap, done, recorded);
}

cudaError_t launch_field_energy_batch(const FieldParams& p, const double* coef, int fine0, int fine1,
                                      double hvol, double* out_base, long long cap, int nbatch,
                                      double* part, unsigned int* done, long long* recorded,
                                      double* egrid_b, long long egrid_stride, cudaStream_t s) {
  FieldParams q = p;
  q.ecoef = coef;
  cudaError_t e = launch_k(group_batch_kernel, dim3((q.ngx + 255) / 256, nbatch), dim3(256), 0, s,
                           q, coef, egrid_b, egrid_stride, (const long long*)recorded);
  if (e != cudaSuccess) return e;
  return launch_k(energy_rows_batch_kernel, dim3(fine0, nbatch), dim3(256), 0, s, q, fine0, fine1,
                  hvol, out_base, cap, part, done, recorded, (const double*)egrid_b, egrid_stride);
}

cudaError_t launch_field_energy(const FieldParams& p, const double* coef, int fine0, int fine1,
                                double hvol, double* out_base, long long cap, cudaStream_t s,
                                double* part, unsigned int* done) {
  FieldParams q = p;
  q.ecoef = coef;
  if (q.negrp > 0 && q.negrp < 64 && q.space_dim == 2 && part != nullptr &&
      std::getenv("SGWG_ENERGY_LEGACY") == nullptr) {
    int need = 0;  // T of one row must fit the CTA's shared array
    (void)need;
    return launch_k(energy_rows_kernel, dim3(fine0), dim3(256), 0, s, q, fine0, fine1, hvol, out_base,
                    cap, part, done);
  }
  if (q.negrp > 0) {
    cudaError_t e = launch_k(group_field_kernel, dim3((q.ngx + 255) / 256), dim3(256), 0, s, q, coef);
    if (e != cudaSuccess) return e;
  }
  int blocks = (q.negrp > 0) ? (fine0 * fine1 + 255) / 256  // a thread per point
                             : (fine0 * fine1 + 7) / 8;     // a warp per point
  if (blocks > 148 * 16) blocks = 148 * 16;
  return launch_k(field_energy_kernel, dim3(blocks), dim3(256), 0, s, q, fine0, fine1, hvol,
                  out_base, cap);
}

__global__ void twiddle_kernel(double* tw, int hmax) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < hmax) sincospi((double)k / (double)hmax, &tw[hmax + k], &tw[k]);
}

cudaError_t launch_twiddles(double* tw, int hmax, cudaStream_t s) {
  twiddle_kernel<<<(hmax + 255) / 256, 256, 0, s>>>(tw, hmax);
  return cudaGetLastError();
}

cudaError_t configure_field() {
  return cudaFuncSetAttribute(field_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(kFieldSmemDoubles * sizeof(double)));
}

cudaError_t launch_field(const FieldParams& p, int nmembers, bool with_moment, cudaStream_t s) {
  if (nmembers <= 0) return cudaSuccess;
  if (with_moment) {
    cudaError_t e = launch_k(moment_kernel, dim3(p.nmtasks), dim3(256), 0, s, p);
    if (e != cudaSuccess) return e;
  }
  return launch_k(field_kernel, dim3(nmembers), dim3(kFieldThreads),
                  kFieldSmemDoubles * sizeof(double), s, p);
}

}  // namespace sgwg

#ifdef SGWG_TRACE
extern "C" int sgwg_ftrace_dump(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, sgwg::sgwg_ftrace, sizeof(sgwg::sgwg_ftrace));
}
#endif
