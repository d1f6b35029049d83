// Sweep microbenchmark: the production masked line sweep (plane4d.cuh
// adv_run_masked) run repeatedly on shared-memory data with no loads, stores
// to global or barriers -- the ceiling of the sweep code itself at a given
// occupancy.  Prints achieved DP instruction throughput vs the DFMA peak.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include \
//        tools/probe/sweep_probe.cu -o tools/probe/sweep_probe
#define SGWG_NS fast
#define SGWG_FAST 1
#include "../../paper_2007_10196_b200/csrc/kernels.cuh"
#include <cstdio>

using namespace sgwg::fast;

template <int MINB, bool ZERO>
__global__ void __launch_bounds__(256, MINB) sweep_probe(double* sink, int reps, int n, int st) {
  extern __shared__ double sm[];
  const int NT = 2400;
  for (int e = threadIdx.x; e < 2 * NT; e += blockDim.x) sm[e] = sin(0.001 * (e + blockIdx.x));
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int m = n >> 3;
  // lines: lane -> line (stride st between line starts), runs along the line with unit stride
  for (int rep = 0; rep < reps; ++rep) {
    for (int q = warp; q < 32; q += 8) {
      const int r = q % m;
      const int l = lane;
      const double* P = sm + l * st + 8 * r - 3 + 3;
      double* out = sm + NT + l * st + 8 * r;
      run_masked<ZERO, false>(r, m, P, 1, n, 1.0, 1e-6, 1.0, out);
    }
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = sm[NT + 5];
}

template <int MINB, bool ZERO>
void run(int blocks_per_sm, const char* name) {
  double* sink;
  cudaMalloc(&sink, 8 * 148 * 8);
  const int smem = 2 * 2400 * 8;
  cudaFuncSetAttribute(sweep_probe<MINB, ZERO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 200, blocks = 148 * blocks_per_sm;
  sweep_probe<MINB, ZERO><<<blocks, 256, smem>>>(sink, 2, 65, 73);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  sweep_probe<MINB, ZERO><<<blocks, 256, smem>>>(sink, reps, 65, 73);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  // per run: 8 points; count DP instructions as ~39 per point (SASS of adv_run_masked<8>)
  const double runs = (double)blocks * reps * 32 /*tasks*/ * 32 /*lanes*/;
  const double pts = runs * 8;
  printf("%s minb=%d blocks/SM=%d: %.3f ms, %.3e pt-dir/s, %.2f ns per run-lane, err=%s\n", name, MINB,
         blocks_per_sm, ms, pts / (ms * 1e-3), ms * 1e6 / runs * 148 * 4, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<2, true>(2, "zero");
  run<2, false>(2, "periodic");
  run<1, true>(1, "zero");
  return 0;
}
