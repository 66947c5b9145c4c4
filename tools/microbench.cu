// Micro-benchmarks of the per-SM pipes that bound the condensed-operator kernel on B200:
// DFMA throughput (FP64 peak), SHFL.64 throughput, LDS.64 (broadcast / distinct) throughput.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_shfl(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, 2);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 4);
      a2 += __shfl_xor_sync(0xffffffffu, a2, 2);
      a3 += __shfl_xor_sync(0xffffffffu, a3, 4);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}

template <int MODE>
__global__ void k_lds(double* out, int iters) {
  __shared__ double s[4096];
  for (int t = threadIdx.x; t < 4096; t += blockDim.x) s[t] = t;
  __syncthreads();
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  int lane = threadIdx.x & 31;
  int base = MODE == 0 ? (lane / 8) : lane;   // 0: 4 distinct addresses per warp (broadcast), 1: 32 distinct
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      int o = (u * 64 + i * 8) & 2047;
      acc0 += s[base + o];
      acc1 += s[base + o + 512];
      acc2 += s[base + o + 1024];
      acc3 += s[base + o + 1536];
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * 1 << 24);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = nsm * 8, threads = 256, iters = 2000;
  float ms;
  // DFMA (best of 10 launches)
  k_dfma<<<blocks, threads>>>(out, 10);
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  ms = best;
  double nfma = (double)blocks * threads * iters * 16 * 8;
  printf("DFMA: %.2f TFLOP/s fp64 (%.1f FMA/clk/SM at %.0f MHz nominal)\n", 2 * nfma / ms / 1e9,
         nfma / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1e3);
  // SHFL (64-bit = 2 SHFL.32)
  k_shfl<<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  k_shfl<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double nsh = (double)blocks * threads / 32 * iters * 16 * 4;   // warp-level 64-bit shuffles
  printf("SHFL.64: %.3f warp-shuffles/clk/SM\n", nsh / (ms * 1e-3) / nsm / (clk * 1e3));
  // LDS
  k_lds<0><<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  k_lds<0><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double nld = (double)blocks * threads / 32 * iters * 16 * 4;
  printf("LDS.64 (4 distinct addr/warp): %.3f warp-loads/clk/SM\n", nld / (ms * 1e-3) / nsm / (clk * 1e3));
  k_lds<1><<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  k_lds<1><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("LDS.64 (32 distinct addr/warp): %.3f warp-loads/clk/SM\n", nld / (ms * 1e-3) / nsm / (clk * 1e3));
  return 0;
}
