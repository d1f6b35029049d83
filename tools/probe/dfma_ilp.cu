// DFMA issue model of one SM sub-partition (B200): cycles per DFMA of a warp as a
// function of the independent chains per thread (ILP) and the warps per sub-partition.
// One CTA per SM, 32 * 4 * W threads.  Build: nvcc -arch=sm_100a -O3 dfma_ilp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void k(double* out, long long* cyc, int iters) {
  double a[ILP];
  const double x = 1.0 + 1e-9 * threadIdx.x, y = 1e-9;
#pragma unroll
  for (int q = 0; q < ILP; ++q) a[q] = q * 1e-3;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < ILP; ++q) a[q] = fma(a[q], x, y);
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < ILP; ++q) s += a[q];
  if (s == 123.456) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int ILP>
void run(int warps_per_smsp, double* out, long long* cyc) {
  const int iters = 4096;
  k<ILP><<<148, 128 * warps_per_smsp>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double per = (double)c / ((double)iters * ILP);
  printf("warps/SMSP %d  ILP %d  cycles per DFMA per warp %.2f  pipe busy %.0f %%\n", warps_per_smsp,
         ILP, per, 100.0 * 2.0 * warps_per_smsp / per);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  for (int w = 1; w <= 4; ++w) {
    run<1>(w, out, cyc);
    run<2>(w, out, cyc);
    run<4>(w, out, cyc);
    run<8>(w, out, cyc);
  }
  return 0;
}
