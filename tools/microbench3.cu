// Store-path micro-benchmark for the operator's finalize pattern: each CTA (one per SM, 256
// threads) writes S doubles per "step" from shared memory to a fresh global range, as rows of
// R doubles handled one warp per row (8-byte stores, 4-wide batches), vs. one TMA bulk store
// (cp.async.bulk.global.shared::cta) per row issued by one lane.  Cycles per step (clock64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench3 microbench3.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int S = 6144, R = 384, NR = S / R;

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_store(double* out, long long* cyc, int steps) {
  __shared__ __align__(128) double sm[S];
  for (int t = threadIdx.x; t < S; t += 256) sm[t] = t;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  for (int st = 0; st < steps; ++st) {
    double* dst = out + ((long long)blockIdx.x * steps + st) * S;
    if (MODE == 0) {
      for (int r = warp; r < NR; r += 8) {
        const double* s = sm + r * R;
        double* d = dst + r * R;
        int t = lane;
        for (; t + 96 < R; t += 128) {
          const double v0 = s[t], v1 = s[t + 32], v2 = s[t + 64], v3 = s[t + 96];
          d[t] = v0; d[t + 32] = v1; d[t + 64] = v2; d[t + 96] = v3;
        }
        for (; t < R; t += 32) d[t] = s[t];
      }
    } else {
      if (warp == 0 && lane < NR) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                     ::"l"(dst + lane * R), "r"((unsigned)__cvta_generic_to_shared(sm + lane * R)), "r"(R * 8)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
    __syncthreads();
  }
  if (MODE == 1 && warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int steps = 200;
  double* out;
  long long *cyc, h;
  cudaMalloc(&out, sizeof(double) * (size_t)nsm * steps * S);
  cudaMalloc(&cyc, 8);
  for (int grid : {32, nsm}) {
    k_store<0><<<grid, 256>>>(out, cyc, steps);
    k_store<0><<<grid, 256>>>(out, cyc, steps);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("grid %3d  8-byte stores: %.0f cycles/step (%.1f B/clk/SM)\n", grid, (double)h / steps,
           8.0 * S * steps / h);
    k_store<1><<<grid, 256>>>(out, cyc, steps);
    k_store<1><<<grid, 256>>>(out, cyc, steps);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("grid %3d  TMA bulk stores: %.0f cycles/step (%.1f B/clk/SM)\n", grid, (double)h / steps,
           8.0 * S * steps / h);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
