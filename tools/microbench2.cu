// Micro-benchmarks for the operator's execution model on B200 (one CTA of 8 warps per SM):
//  (1) DFMA dependent-chain latency (one warp),
//  (2) DFMA issue rate of 8 warps / SM at ILP 1, 2, 4, 8,
//  (3) instruction-fetch cost: the same number of independent FP64 instructions executed as a
//      short loop vs. as one long unrolled straight-line body (code size >> L1.5 I-cache).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench2 microbench2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3;
  const double b = 0.999999, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 32; ++u) a = fma(a, b, c);
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
__global__ void k_ilp(double* out, long long* cyc, int iters) {
  double a[ILP];
#pragma unroll
  for (int q = 0; q < ILP; ++q) a[q] = threadIdx.x * 1e-3 + q;
  const double b = 0.999999, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 32 / ILP; ++u)
#pragma unroll
      for (int q = 0; q < ILP; ++q) a[q] = fma(a[q], b, c);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int q = 0; q < ILP; ++q) s += a[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

// straight-line body of N x 8 independent DFMAs (unrolled) vs the same work as a loop
template <int N>
__global__ void k_long(double* out, long long* cyc, int reps) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int u = 0; u < N; ++u) {
      const double b = 1.0 - 1e-9 * u;   // distinct immediates defeat loop re-rolling
      a0 = fma(a0, b, 1e-7); a1 = fma(a1, b, 2e-7); a2 = fma(a2, b, 3e-7); a3 = fma(a3, b, 4e-7);
      a4 = fma(a4, b, 5e-7); a5 = fma(a5, b, 6e-7); a6 = fma(a6, b, 7e-7); a7 = fma(a7, b, 8e-7);
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long *cyc, h;
  cudaMalloc(&out, sizeof(double) * (1 << 22));
  cudaMalloc(&cyc, sizeof(long long));
  const int iters = 4000;
  k_lat<<<1, 32>>>(out, cyc, 10);
  k_lat<<<1, 32>>>(out, cyc, iters);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (iters * 32.0));
#define ILPRUN(I)                                                                               \
  k_ilp<I><<<nsm, 256>>>(out, cyc, 10);                                                         \
  k_ilp<I><<<nsm, 256>>>(out, cyc, iters);                                                      \
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                                               \
  printf("8 warps/SM, ILP %d: %.3f warp-DFMA/clk/SM (%.1f FMA/clk/SM)\n", I,                    \
         8.0 * iters * 32 / h, 8.0 * iters * 32 * 32 / h);
  ILPRUN(1) ILPRUN(2) ILPRUN(4) ILPRUN(8)
  // code size: N*8 DFMA per rep; 16 B per instruction
#define LONGRUN(N, R)                                                                           \
  k_long<N><<<nsm, 256>>>(out, cyc, 2);                                                         \
  k_long<N><<<nsm, 256>>>(out, cyc, R);                                                         \
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);                                               \
  printf("straight-line body %6d instr (%5d KB): %.3f warp-instr/clk/SM over 8 warps\n", N * 8, \
         N * 8 * 16 / 1024, 8.0 * N * 8 * R / h);
  LONGRUN(16, 4000) LONGRUN(128, 500) LONGRUN(512, 125) LONGRUN(2048, 32) LONGRUN(4096, 16)
  return 0;
}
