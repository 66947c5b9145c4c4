// Per-solve and helper kernels: basis/layout conversions, seeded random fill,
// Alg. 4 pre-processing (condense RHS) and post-processing (recover + back-transform).
// These are not on the timed PCG path ("their performance is not graded").
#include <cuda_runtime.h>
#include "sc_device.cuh"

namespace sc {

__device__ __forceinline__ long long lat_index(const Geom& g, int gx, int gy, int gz) {
  return gx + (long long)g.nx1 * (gy + (long long)g.ny1 * gz);
}

// lattice -> skeleton: out[q] = sum over the entity's nodes of A (x) A applied in-entity.
__global__ void k_to_skel(Geom g, const double* __restrict__ in, double* __restrict__ out, int mat) {
  const int p = g.p, ni = g.ni;
  const double* A = g.tab + TAB_MAT + mat * SC_NIMAX * SC_NIMAX;   // A[r*ni + c]
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.n_total;
       q += (long long)gridDim.x * blockDim.x) {
    int gx, gy, gz;
    bool dr;
    if (!decode_entry(g, q, &gx, &gy, &gz, &dr) || (dr && !g.nodir)) { out[q] = 0.0; continue; }
    int c[3] = {gx, gy, gz};
    int free_dirs[2], nf = 0;
    for (int d = 0; d < 3; ++d)
      if (c[d] % p != 0) free_dirs[nf++] = d;
    double v;
    if (nf == 0 || mat == MAT_I) {
      v = in[lat_index(g, gx, gy, gz)];
    } else if (nf == 1) {
      int d0 = free_dirs[0], a = c[d0] % p - 1, base = c[d0] - (a + 1);
      v = 0.0;
      for (int a2 = 0; a2 < ni; ++a2) {
        int cc[3] = {c[0], c[1], c[2]};
        cc[d0] = base + 1 + a2;
        v += A[a * ni + a2] * in[lat_index(g, cc[0], cc[1], cc[2])];
      }
    } else {
      int d0 = free_dirs[0], d1 = free_dirs[1];
      int a = c[d0] % p - 1, b = c[d1] % p - 1, ba = c[d0] - (a + 1), bb = c[d1] - (b + 1);
      v = 0.0;
      for (int b2 = 0; b2 < ni; ++b2) {
        double s = 0.0;
        for (int a2 = 0; a2 < ni; ++a2) {
          int cc[3] = {c[0], c[1], c[2]};
          cc[d0] = ba + 1 + a2;
          cc[d1] = bb + 1 + b2;
          s += A[a * ni + a2] * in[lat_index(g, cc[0], cc[1], cc[2])];
        }
        v += A[b * ni + b2] * s;
      }
    }
    out[q] = v;
  }
}

// Skeleton index of the entity node at local lattice coords (gx,gy,gz) (a skeleton node).
__device__ __forceinline__ long long skel_index(const Geom& g, int gx, int gy, int gz, bool* dr) {
  const int p = g.p, ni = g.ni, nx = g.nx, ny = g.ny;
  const long long n2 = (long long)ni * ni;
  bool bx = gx % p == 0, by = gy % p == 0, bz = gz % p == 0;
  int fx = gx / p, fy = gy / p, fz = gz / p;
  int ax = gx % p - 1, ay = gy % p - 1, az = gz % p - 1;
  int nb = (int)bx + (int)by + (int)bz;
  if (nb == 1) {
    if (bx) { *dr = (fx == 0 || fx == nx); return g.off_f[0] + (fx + (long long)(nx + 1) * (fy + (long long)ny * fz)) * n2 + ay + ni * az; }
    if (by) { *dr = (fy == 0 || fy == ny); return g.off_f[1] + (fx + (long long)nx * (fy + (long long)(ny + 1) * fz)) * n2 + ax + ni * az; }
    *dr = zdir(g, fz);
    return g.off_f[2] + (fx + (long long)nx * (fy + (long long)ny * fz)) * n2 + ax + ni * ay;
  }
  if (nb == 2) {
    if (!bx) { *dr = (fy == 0 || fy == ny) || zdir(g, fz); return g.off_e[0] + (fx + (long long)nx * (fy + (long long)(ny + 1) * fz)) * ni + ax; }
    if (!by) { *dr = (fx == 0 || fx == nx) || zdir(g, fz); return g.off_e[1] + (fx + (long long)(nx + 1) * (fy + (long long)ny * fz)) * ni + ay; }
    *dr = (fx == 0 || fx == nx) || (fy == 0 || fy == ny);
    return g.off_e[2] + (fx + (long long)(nx + 1) * (fy + (long long)(ny + 1) * fz)) * ni + az;
  }
  *dr = (fx == 0 || fx == nx) || (fy == 0 || fy == ny) || zdir(g, fz);
  return g.off_v + fx + (long long)(nx + 1) * (fy + (long long)(ny + 1) * fz);
}

// skeleton -> lattice (interior lattice nodes and Dirichlet nodes written as 0).
__global__ void k_from_skel(Geom g, const double* __restrict__ in, double* __restrict__ out, int mat) {
  const int p = g.p, ni = g.ni;
  const double* A = g.tab + TAB_MAT + mat * SC_NIMAX * SC_NIMAX;
  const long long nl = (long long)g.nx1 * g.ny1 * g.nz1;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nl;
       q += (long long)gridDim.x * blockDim.x) {
    int gx = (int)(q % g.nx1);
    long long t = q / g.nx1;
    int gy = (int)(t % g.ny1), gz = (int)(t / g.ny1);
    int c[3] = {gx, gy, gz};
    int free_dirs[3], nf = 0;
    for (int d = 0; d < 3; ++d)
      if (c[d] % p != 0) free_dirs[nf++] = d;
    if (nf == 3) { out[q] = 0.0; continue; }
    bool dr;
    long long si = skel_index(g, gx, gy, gz, &dr);
    if (dr && !g.nodir) { out[q] = 0.0; continue; }
    double v;
    if (nf == 0 || mat == MAT_I) {
      v = in[si];
    } else if (nf == 1) {
      int d0 = free_dirs[0], a = c[d0] % p - 1;
      long long base = si - a;
      v = 0.0;
      for (int a2 = 0; a2 < ni; ++a2) v += A[a * ni + a2] * in[base + a2];
    } else {
      int d0 = free_dirs[0], d1 = free_dirs[1];
      int a = c[d0] % p - 1, b = c[d1] % p - 1;
      long long base = si - a - (long long)ni * b;
      v = 0.0;
      for (int b2 = 0; b2 < ni; ++b2) {
        double s = 0.0;
        for (int a2 = 0; a2 < ni; ++a2) s += A[a * ni + a2] * in[base + a2 + (long long)ni * b2];
        v += A[b * ni + b2] * s;
      }
    }
    out[q] = v;
  }
}

__device__ __forceinline__ double splitmix_uniform(uint64_t seed, uint64_t gidx) {
  uint64_t z = seed * 0x9E3779B97F4A7C15ULL + gidx;
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27; z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
}

__global__ void k_fill_random(Geom g, uint64_t seed, double* __restrict__ v) {
  const long long nx1 = g.nx1, ny1 = g.ny1;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.n_total;
       q += (long long)gridDim.x * blockDim.x) {
    int gx, gy, gz;
    bool dr;
    if (!decode_entry(g, q, &gx, &gy, &gz, &dr) || dr) { v[q] = 0.0; continue; }
    long long gzg = gz + (long long)g.z_begin * g.p;
    uint64_t gi = (uint64_t)(gx + nx1 * (gy + ny1 * gzg));
    v[q] = splitmix_uniform(seed, gi);
  }
}

// out(.., c, ..) = sum_c' A[c-1][c'-1] in(.., c', ..) for interior c along `axis`, copy otherwise.
__device__ void transform_axis(const double* in, double* out, const double* A, int p, int ni, int axis) {
  const int n = p + 1, n3 = n * n * n;
  const int stride = axis == 0 ? 1 : (axis == 1 ? n : n * n);
  for (int t = threadIdx.x; t < n3; t += blockDim.x) {
    int c = (t / stride) % n;
    if (c == 0 || c == p) { out[t] = in[t]; continue; }
    int base = t - c * stride;
    double s = 0.0;
    for (int c2 = 1; c2 < p; ++c2) s += A[(c - 1) * ni + (c2 - 1)] * in[base + c2 * stride];
    out[t] = s;
  }
}

// F~_e = (S(x)S(x)S) (h1h2h3/8)(w(x)w(x)w) f  ->  buf2 (element-local, i fastest)
__device__ void element_ftilde(const Geom& g, const double* f, int ex, int ey, int ez, double* buf,
                               double* buf2) {
  const int p = g.p, ni = g.ni, n = p + 1, n3 = n * n * n;
  const double* w = g.tab + TAB_W;
  const double* S = g.tab + TAB_MAT + MAT_S * SC_NIMAX * SC_NIMAX;
  double J = g.hx[ex] * g.hy[ey] * g.hz[ez] * 0.125;
  for (int t = threadIdx.x; t < n3; t += blockDim.x) {
    int i = t % n, j = (t / n) % n, k = t / (n * n);
    buf[t] = J * w[i] * w[j] * w[k] * f[lat_index(g, ex * p + i, ey * p + j, ez * p + k)];
  }
  __syncthreads();
  transform_axis(buf, buf2, S, p, ni, 0);
  __syncthreads();
  transform_axis(buf2, buf, S, p, ni, 1);
  __syncthreads();
  transform_axis(buf, buf2, S, p, ni, 2);
  __syncthreads();
}

__global__ void k_condense(Geom g, const double* __restrict__ f, double* __restrict__ b, double* scratch) {
  const int p = g.p, ni = g.ni, n = p + 1, n3 = n * n * n, n2 = ni * ni, nsh = 6 * n2 + 12 * ni + 8;
  double* buf = scratch + (long long)blockIdx.x * 2 * n3;
  double* buf2 = buf + n3;
  const double* lam = g.tab + TAB_LAM;
  const double* a0 = g.tab + TAB_A0;
  const double* ap = g.tab + TAB_AP;
  const long long ne = (long long)g.nx * g.ny * g.nz;
  for (long long e = blockIdx.x; e < ne; e += gridDim.x) {
    int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
    double d[4];
    metric(g, ex, ey, ez, d);
    element_ftilde(g, f, ex, ey, ez, buf, buf2);
    // v = F~_I D^{-1} (interior, in buf)
    for (int t = threadIdx.x; t < n3; t += blockDim.x) {
      int i = t % n, j = (t / n) % n, k = t / (n * n);
      if (i == 0 || i == p || j == 0 || j == p || k == 0 || k == p) continue;
      buf[t] = buf2[t] / (d[0] + d[1] * lam[i - 1] + d[2] * lam[j - 1] + d[3] * lam[k - 1]);
    }
    __syncthreads();
    for (int s = threadIdx.x; s < nsh; s += blockDim.x) {
      int i, j, k, ent, loc;
      shell_node(p, ni, s, &i, &j, &k, &ent, &loc);
      bool dr;
      long long base = entity_base(g, ex, ey, ez, ent, &dr);
      if (dr) continue;
      double val = buf2[i + n * (j + n * k)];
      if (ent < 6) {   // b~ = F~_B - Htilde_BI D^{-1} F~_I  (faces only)
        int dir = ent >> 1;
        const double* a = (ent & 1) ? ap : a0;
        double acc = 0.0;
        for (int q = 1; q < p; ++q) {
          int cc[3] = {i, j, k};
          cc[dir] = q;
          acc += a[q - 1] * buf[cc[0] + n * (cc[1] + n * cc[2])];
        }
        val -= d[1 + dir] * acc;
      }
      atomicAdd(&b[base + loc], val);
    }
    __syncthreads();
  }
}

__global__ void k_recover(Geom g, const double* __restrict__ f, const double* __restrict__ x,
                          double* __restrict__ u, double* scratch) {
  const int p = g.p, ni = g.ni, n = p + 1, n3 = n * n * n, n2 = ni * ni, nsh = 6 * n2 + 12 * ni + 8;
  double* buf = scratch + (long long)blockIdx.x * 2 * n3;
  double* buf2 = buf + n3;
  const double* lam = g.tab + TAB_LAM;
  const double* a0 = g.tab + TAB_A0;
  const double* ap = g.tab + TAB_AP;
  const double* ST = g.tab + TAB_MAT + MAT_ST * SC_NIMAX * SC_NIMAX;
  const long long ne = (long long)g.nx * g.ny * g.nz;
  for (long long e = blockIdx.x; e < ne; e += gridDim.x) {
    int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
    double d[4];
    metric(g, ex, ey, ez, d);
    element_ftilde(g, f, ex, ey, ez, buf, buf2);   // F~ in buf2
    for (int s = threadIdx.x; s < nsh; s += blockDim.x) {
      int i, j, k, ent, loc;
      shell_node(p, ni, s, &i, &j, &k, &ent, &loc);
      bool dr;
      long long base = entity_base(g, ex, ey, ez, ent, &dr);
      buf[i + n * (j + n * k)] = (dr && !g.nodir) ? 0.0 : x[base + loc];
    }
    __syncthreads();
    // u~_I = D^{-1} (F~_I - Htilde_IB u~_B)   (Alg. 4)
    for (int t = threadIdx.x; t < n3; t += blockDim.x) {
      int i = t % n, j = (t / n) % n, k = t / (n * n);
      if (i == 0 || i == p || j == 0 || j == p || k == 0 || k == p) continue;
      double fin = d[1] * (a0[i - 1] * buf[0 + n * (j + n * k)] + ap[i - 1] * buf[p + n * (j + n * k)]) +
                   d[2] * (a0[j - 1] * buf[i + n * (0 + n * k)] + ap[j - 1] * buf[i + n * (p + n * k)]) +
                   d[3] * (a0[k - 1] * buf[i + n * (j + n * 0)] + ap[k - 1] * buf[i + n * (j + n * p)]);
      buf[t] = (buf2[t] - fin) / (d[0] + d[1] * lam[i - 1] + d[2] * lam[j - 1] + d[3] * lam[k - 1]);
    }
    __syncthreads();
    // u_e = (S(x)S(x)S)^T u~_e
    transform_axis(buf, buf2, ST, p, ni, 0);
    __syncthreads();
    transform_axis(buf2, buf, ST, p, ni, 1);
    __syncthreads();
    transform_axis(buf, buf2, ST, p, ni, 2);
    __syncthreads();
    for (int t = threadIdx.x; t < n3; t += blockDim.x) {
      int i = t % n, j = (t / n) % n, k = t / (n * n);
      u[lat_index(g, ex * p + i, ey * p + j, ez * p + k)] = buf2[t];
    }
    __syncthreads();
  }
}

// Free / Dirichlet split of skeleton vectors (inhomogeneous Dirichlet data, P:625 E3):
//   mode 0: a <- a on Dirichlet entries, 0 elsewhere (the lifting vector)
//   mode 1: a <- 0 on Dirichlet entries, a - b elsewhere (subtract the lifting's image)
//   mode 2: a <- b on Dirichlet entries, a elsewhere (complete a free solution with its data)
__global__ void k_dir_split(Geom g, double* __restrict__ a, const double* __restrict__ b, int mode) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.n_total;
       q += (long long)gridDim.x * blockDim.x) {
    int gx, gy, gz;
    bool dr;
    if (!decode_entry(g, q, &gx, &gy, &gz, &dr)) { a[q] = 0.0; continue; }
    if (mode == 0) a[q] = dr ? a[q] : 0.0;
    else if (mode == 1) a[q] = dr ? 0.0 : a[q] - b[q];
    else if (dr) a[q] = b[q];
  }
}

int launch_dir_split(const Geom& g, double* a, const double* b, int mode, void* stream, int* nl) {
  k_dir_split<<<1184, 256, 0, (cudaStream_t)stream>>>(g, a, b, mode);
  (*nl)++;
  return cudaGetLastError();
}

int launch_convert(const Geom& g, const double* in, double* out, int to_skel, int mat, void* stream, int* nl) {
  cudaStream_t st = (cudaStream_t)stream;
  if (to_skel) k_to_skel<<<1184, 256, 0, st>>>(g, in, out, mat);
  else k_from_skel<<<1184, 256, 0, st>>>(g, in, out, mat);
  (*nl)++;
  return cudaGetLastError();
}

int launch_fill_random(const Geom& g, uint64_t seed, double* v, void* stream, int* nl) {
  k_fill_random<<<1184, 256, 0, (cudaStream_t)stream>>>(g, seed, v);
  (*nl)++;
  return cudaGetLastError();
}

int launch_condense(const Geom& g, const double* f, double* b, double* scratch, long long scratch_elems,
                    void* stream, int* nl) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t err = cudaMemsetAsync(b, 0, sizeof(double) * g.n_total, st);
  if (err != cudaSuccess) return err;
  long long n3 = (long long)(g.p + 1) * (g.p + 1) * (g.p + 1);
  long long nblk = scratch_elems / (2 * n3);
  long long ne = (long long)g.nx * g.ny * g.nz;
  if (nblk > ne) nblk = ne;
  if (nblk < 1) return cudaErrorInvalidValue;
  k_condense<<<(unsigned)nblk, 256, 0, st>>>(g, f, b, scratch);
  (*nl)++;
  return cudaGetLastError();
}

int launch_recover(const Geom& g, const double* f, const double* x, double* u, double* scratch,
                   long long scratch_elems, void* stream, int* nl) {
  cudaStream_t st = (cudaStream_t)stream;
  long long n3 = (long long)(g.p + 1) * (g.p + 1) * (g.p + 1);
  long long nblk = scratch_elems / (2 * n3);
  long long ne = (long long)g.nx * g.ny * g.nz;
  if (nblk > ne) nblk = ne;
  if (nblk < 1) return cudaErrorInvalidValue;
  k_recover<<<(unsigned)nblk, 256, 0, st>>>(g, f, x, u, scratch);
  (*nl)++;
  return cudaGetLastError();
}

}  // namespace sc
