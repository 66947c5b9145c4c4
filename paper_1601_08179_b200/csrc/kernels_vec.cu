// PCG vector kernels and deterministic fp64 reductions (rows a9, a10 of SURVEY §8(a)).
//
// Solver BT: CG (Hestenes-Stiefel) with the diagonal
// preconditioner z = Pinv .* r in the transformed system.  All scalars (alpha, beta,
// r.z, r.r, done flag, iteration count) live in device memory; every kernel returns
// immediately once `done` is set, so the host may enqueue iterations ahead of the
// convergence test without changing the result.
//
// Reductions are two-stage and deterministic: a fixed grid of SC_RED_BLOCKS blocks writes
// one partial per block (warp shuffle + shared memory, fixed order), and a single block
// sums the partials in a fixed order.
#include <cuda_runtime.h>
#include "sc_internal.h"

namespace sc {

#define VEC_THREADS 256

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum of NV values; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV]) {
  __shared__ double red[NV][VEC_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = warp_sum(v[q]);
    if (lane == 0) red[q][wid] = s;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double s = lane < VEC_THREADS / 32 ? red[q][lane] : 0.0;
      v[q] = warp_sum(s);
    }
  }
}

__device__ __forceinline__ bool owned(long long i, const OwnMask& m) {
  for (int q = 0; q < m.n; ++q)
    if (i >= m.lo[q] && i < m.hi[q]) return false;
  return true;
}

__global__ void k_dot_partial(const double* __restrict__ a, const double* __restrict__ b, long long n,
                              OwnMask m, double* __restrict__ partials, const double* __restrict__ done) {
  if (done != nullptr && *done != 0.0) return;
  double v[1] = {0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (owned(i, m)) v[0] += a[i] * b[i];
  block_sum<1>(v);
  if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
}

// r = b (free entries), x = 0, p = Pinv r; partials: [r.z | r.r]
__global__ void k_pcg_init(const double* __restrict__ b, const double* __restrict__ pinv, double* __restrict__ x,
                           double* __restrict__ r, double* __restrict__ p, long long n, OwnMask m,
                           double* __restrict__ partials) {
  double v[2] = {0.0, 0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double pi = pinv[i];
    double ri = pi != 0.0 ? b[i] : 0.0;
    double zi = pi * ri;
    r[i] = ri; x[i] = 0.0; p[i] = zi;
    if (owned(i, m)) { v[0] += ri * zi; v[1] += ri * ri; }
  }
  block_sum<2>(v);
  if (threadIdx.x == 0) { partials[blockIdx.x] = v[0]; partials[SC_RED_BLOCKS + blockIdx.x] = v[1]; }
}

// r -= alpha q ; z = Pinv r ; partials [r.z | r.r]   (4 streams: r, q, Pinv read; r written)
__global__ void k_pcg_update(double* __restrict__ r, const double* __restrict__ q, const double* __restrict__ pinv,
                             long long n, OwnMask m, const double* __restrict__ scal, double* __restrict__ partials) {
  if (scal[SCAL_DONE] != 0.0) return;
  const double alpha = scal[SCAL_ALPHA];
  double v[2] = {0.0, 0.0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double ri = r[i] - alpha * q[i];
    r[i] = ri;
    double zi = pinv[i] * ri;
    if (owned(i, m)) { v[0] += ri * zi; v[1] += ri * ri; }
  }
  block_sum<2>(v);
  if (threadIdx.x == 0) { partials[blockIdx.x] = v[0]; partials[SC_RED_BLOCKS + blockIdx.x] = v[1]; }
}

// x += alpha p (the x update of this iteration, moved here from the update kernel so that p is
// streamed once) ; p = Pinv r + beta p unless converged   (6 streams: x, p, r, Pinv read; x, p
// written).  The kernel acts only if this iteration's alpha kernel ran (device flag SCAL_RAN),
// so iterations enqueued after convergence change nothing and the iteration has no host-side
// arguments (graph-capturable).
__global__ void k_pcg_direction(double* __restrict__ x, double* __restrict__ p, const double* __restrict__ r,
                                const double* __restrict__ pinv, long long n, const double* __restrict__ scal, int) {
  if (scal[SCAL_RAN] == 0.0 || scal[SCAL_BREAK] != 0.0) return;
  const double alpha = scal[SCAL_ALPHA], beta = scal[SCAL_BETA];
  const bool dir = scal[SCAL_DONE] == 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double pi = p[i];
    x[i] += alpha * pi;
    if (dir) p[i] = pinv[i] * r[i] + beta * pi;
  }
}

// Table-Pinv variants (uniform geometry): entries are visited class by class (faces x/y/z, edges
// x/y/z, vertices), each thread keeping its index inside the entity incrementally (the grid
// stride S is fixed), so Pinv costs a cached table load instead of an 8-byte stream per entry.
// r -= alpha q ; z = Pinv r ; partials [r.z | r.r]   (3 streams: r, q read; r written)
__global__ void k_pcg_update_tab(double* __restrict__ r, const double* __restrict__ q, PinvTab T, OwnMask m,
                                 const double* __restrict__ scal, double* __restrict__ partials) {
  if (scal[SCAL_DONE] != 0.0) return;
  const double alpha = scal[SCAL_ALPHA];
  const long long S = (long long)gridDim.x * blockDim.x, g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double v[2] = {0.0, 0.0};
  for (int c = 0; c < 7; ++c) {
    const int nc = T.n[c], step = (int)(S % nc);
    const double* tb = T.tab + T.base[c];
    int loc = (int)(g % nc);
    const long long end = T.off[c] + T.len[c];
    for (long long i = T.off[c] + g; i < end; i += S) {
      const double ri = r[i] - alpha * q[i];
      r[i] = ri;
      const double zi = __ldg(tb + loc) * ri;
      if (owned(i, m)) { v[0] += ri * zi; v[1] += ri * ri; }
      loc += step;
      if (loc >= nc) loc -= nc;
    }
  }
  block_sum<2>(v);
  if (threadIdx.x == 0) { partials[blockIdx.x] = v[0]; partials[SC_RED_BLOCKS + blockIdx.x] = v[1]; }
}

// x += alpha p ; p = Pinv r + beta p unless converged   (5 streams: x, p, r read; x, p written)
__global__ void k_pcg_direction_tab(double* __restrict__ x, double* __restrict__ p, const double* __restrict__ r,
                                    PinvTab T, const double* __restrict__ scal) {
  if (scal[SCAL_RAN] == 0.0 || scal[SCAL_BREAK] != 0.0) return;
  const double alpha = scal[SCAL_ALPHA], beta = scal[SCAL_BETA];
  const bool dir = scal[SCAL_DONE] == 0.0;
  const long long S = (long long)gridDim.x * blockDim.x, g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (int c = 0; c < 7; ++c) {
    const int nc = T.n[c], step = (int)(S % nc);
    const double* tb = T.tab + T.base[c];
    int loc = (int)(g % nc);
    const long long end = T.off[c] + T.len[c];
    for (long long i = T.off[c] + g; i < end; i += S) {
      const double pi = p[i];
      x[i] += alpha * pi;
      if (dir) p[i] = __ldg(tb + loc) * r[i] + beta * pi;
      loc += step;
      if (loc >= nc) loc -= nc;
    }
  }
}

// Fixed-order second stage: scal[slot0 + v] = sum_b partials[v * SC_RED_BLOCKS + b].
__global__ void k_reduce2(const double* __restrict__ partials, double* __restrict__ scal, int slot0, int nvals,
                          const double* __restrict__ done) {
  if (done != nullptr && *done != 0.0) return;
  for (int q = 0; q < nvals; ++q) {
    double v[1] = {0.0};
    for (int b = threadIdx.x; b < SC_RED_BLOCKS; b += blockDim.x) v[0] += partials[q * SC_RED_BLOCKS + b];
    block_sum<1>(v);
    if (threadIdx.x == 0) scal[slot0 + q] = v[0];
    __syncthreads();
  }
}

// Fixed-order sum of n values (one block): thread t sums v[t], v[t + nt], ... in order, then a
// fixed-shape block reduction.  Used for the per-tile x . y partials of the operator.
__global__ void k_sum_ordered(const double* __restrict__ v, int n, double* __restrict__ scal, int slot,
                              const double* __restrict__ done) {
  if (done != nullptr && *done != 0.0) return;
  double a[1] = {0.0};
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[0] += v[i];
  block_sum<1>(a);
  if (threadIdx.x == 0) scal[slot] = a[0];
}

__global__ void k_pcg_init_finalize(double* scal, double tol2, int maxit) {
  double rz = scal[SCAL_RED0], rr = scal[SCAL_RED1];
  scal[SCAL_RZ] = rz;
  scal[SCAL_RR] = rr;
  scal[SCAL_RR0] = rr;
  scal[SCAL_ITERS] = 0.0;
  scal[SCAL_BREAK] = 0.0;
  scal[SCAL_TOL2] = tol2;
  scal[SCAL_MAXIT] = (double)maxit;
  scal[SCAL_DONE] = (rr == 0.0 || maxit <= 0) ? 1.0 : 0.0;
}

__global__ void k_pcg_alpha(double* scal) {
  scal[SCAL_RAN] = 0.0;
  if (scal[SCAL_DONE] != 0.0) return;
  double pq = scal[SCAL_RED0];
  if (!(pq > 0.0)) { scal[SCAL_BREAK] = 1.0; scal[SCAL_DONE] = 1.0; return; }
  scal[SCAL_PQ] = pq;
  scal[SCAL_ALPHA] = scal[SCAL_RZ] / pq;
  scal[SCAL_ITERS] += 1.0;
  scal[SCAL_RAN] = 1.0;
}

__global__ void k_pcg_beta(double* scal) {
  if (scal[SCAL_DONE] != 0.0) return;
  double rznew = scal[SCAL_RED0], rr = scal[SCAL_RED1];
  scal[SCAL_RR] = rr;
  if (rr <= scal[SCAL_TOL2] * scal[SCAL_RR0] || scal[SCAL_ITERS] >= scal[SCAL_MAXIT]) {
    scal[SCAL_DONE] = 1.0;
    return;
  }
  scal[SCAL_BETA] = rznew / scal[SCAL_RZ];
  scal[SCAL_RZ] = rznew;
}

int launch_dot_partial(const double* a, const double* b, long long n, OwnMask m, double* partials,
                       const double* done, void* stream, int* nl) {
  k_dot_partial<<<SC_RED_BLOCKS, VEC_THREADS, 0, (cudaStream_t)stream>>>(a, b, n, m, partials, done);
  (*nl)++;
  return cudaGetLastError();
}

int launch_reduce2(const double* partials, double* scal, int slot0, int nvals, const double* done, void* stream,
                   int* nl) {
  k_reduce2<<<1, VEC_THREADS, 0, (cudaStream_t)stream>>>(partials, scal, slot0, nvals, done);
  (*nl)++;
  return cudaGetLastError();
}

int launch_sum_ordered(const double* v, int n, double* scal, int slot, const double* done, void* stream, int* nl) {
  k_sum_ordered<<<1, VEC_THREADS, 0, (cudaStream_t)stream>>>(v, n, scal, slot, done);
  (*nl)++;
  return cudaGetLastError();
}

int launch_pcg_init(const double* b, const double* pinv, double* x, double* r, double* p, long long n, OwnMask m,
                    double* partials, void* stream, int* nl) {
  k_pcg_init<<<SC_RED_BLOCKS, VEC_THREADS, 0, (cudaStream_t)stream>>>(b, pinv, x, r, p, n, m, partials);
  (*nl)++;
  return cudaGetLastError();
}

int launch_pcg_init_finalize(double* scal, const double* partials, double tol2, int maxit, void* stream, int* nl) {
  (void)partials;
  k_pcg_init_finalize<<<1, 1, 0, (cudaStream_t)stream>>>(scal, tol2, maxit);
  (*nl)++;
  return cudaGetLastError();
}

int launch_pcg_alpha(double* scal, void* stream, int* nl) {
  k_pcg_alpha<<<1, 1, 0, (cudaStream_t)stream>>>(scal);
  (*nl)++;
  return cudaGetLastError();
}

int launch_pcg_update(double* r, const double* q, const double* pinv, long long n, OwnMask m, const double* scal,
                      double* partials, void* stream, int* nl) {
  k_pcg_update<<<SC_RED_BLOCKS, VEC_THREADS, 0, (cudaStream_t)stream>>>(r, q, pinv, n, m, scal, partials);
  (*nl)++;
  return cudaGetLastError();
}

int launch_pcg_beta(double* scal, void* stream, int* nl) {
  k_pcg_beta<<<1, 1, 0, (cudaStream_t)stream>>>(scal);
  (*nl)++;
  return cudaGetLastError();
}

int launch_pcg_direction(double* x, double* p, const double* r, const double* pinv, long long n, const double* scal,
                         void* stream, int* nl) {
  k_pcg_direction<<<SC_RED_BLOCKS, VEC_THREADS, 0, (cudaStream_t)stream>>>(x, p, r, pinv, n, scal, 0);
  (*nl)++;
  return cudaGetLastError();
}

int launch_pcg_update_tab(double* r, const double* q, const PinvTab& T, OwnMask m, const double* scal,
                          double* partials, void* stream, int* nl) {
  k_pcg_update_tab<<<SC_RED_BLOCKS, VEC_THREADS, 0, (cudaStream_t)stream>>>(r, q, T, m, scal, partials);
  (*nl)++;
  return cudaGetLastError();
}

int launch_pcg_direction_tab(double* x, double* p, const double* r, const PinvTab& T, const double* scal,
                             void* stream, int* nl) {
  k_pcg_direction_tab<<<SC_RED_BLOCKS, VEC_THREADS, 0, (cudaStream_t)stream>>>(x, p, r, T, scal);
  (*nl)++;
  return cudaGetLastError();
}

int launch_reduce_partials(const double* partials, int nparts, double* out, const double* done, void* stream,
                           int* nl) {
  (void)nparts;
  return launch_reduce2(partials, out, 0, 1, done, stream, nl);
}

}  // namespace sc

namespace sc {

// y[seg] += add[seg] for up to 4 segments packed back to back in `add` (interface-plane halo sum).
struct Segs { long long off[4], len[4]; int n; };

__global__ void k_add_segments(double* __restrict__ y, const double* __restrict__ add, Segs s) {
  long long base = 0;
  for (int q = 0; q < s.n; ++q) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < s.len[q];
         i += (long long)gridDim.x * blockDim.x)
      y[s.off[q] + i] += add[base + i];
    base += s.len[q];
  }
}

int launch_add_segments(double* y, const double* add, const long long* off, const long long* len, int n,
                        void* stream, int* nl) {
  Segs s;
  s.n = n;
  for (int q = 0; q < 4; ++q) { s.off[q] = q < n ? off[q] : 0; s.len[q] = q < n ? len[q] : 0; }
  k_add_segments<<<592, VEC_THREADS, 0, (cudaStream_t)stream>>>(y, add, s);
  (*nl)++;
  return cudaGetLastError();
}

}  // namespace sc
