// k_field.cu -- Vlasov-Poisson field kernels of every member (BASELINE C4/C5);
// the device code is in field_device.cuh (shared with the persistent kernel).
//
// moment_kernel: rho of every x point (one warp each, many CTAs).
// field_kernel:  one CTA per member: the x-grid has <= 2048 points (C4: 32*2^l;
//                C5: (8*2^l1)x(8*2^l2), l1+l2 <= 5), so the 2D FFT lives in
//                shared memory.
// field_energy_kernel: per-step ||E_c||_2 diagnostic.
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

cudaError_t launch_field_energy(const FieldParams& p, const double* coef, int fine0, int fine1,
                                double hvol, double* out_base, long long cap, cudaStream_t s) {
  FieldParams q = p;
  q.ecoef = coef;
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
