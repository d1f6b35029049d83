// k_fast.cu -- FMA-contracted, divide-reduced instantiation of kernels.cuh
// (SGWG_ARITH_FAST).  Compiled with the default --fmad=true.
#define SGWG_NS fast
#define SGWG_FAST 1
#include "kernels.cuh"
