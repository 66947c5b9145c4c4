// Device helpers shared by the kernels: skeleton layout addressing.
#pragma once
#include <cuda_runtime.h>
#include "sc_internal.h"

namespace sc {

// Element-local shell numbering (26 entities):
//   faces 0..5  = w(i=0), e(i=p), s(j=0), n(j=p), b(k=0), t(k=p); face coords (a,b):
//                 w/e: (j,k), s/n: (i,k), b/t: (i,j); entry a + n_I b.
//   edges 6..17 = x-edges (along x, coord i) at (j,k) = bits (jb,kb): 6 + jb + 2kb
//                 y-edges (coord j) at (i,k): 10 + ib + 2kb;  z-edges (coord k) at (i,j): 14 + ib + 2jb
//   vertices 18..25 = 18 + ib + 2jb + 4kb.
// Global skeleton ids:
//   x-face (fx,ey,ez) = fx + (nx+1)(ey + ny ez)     y-face (ex,fy,ez) = ex + nx(fy + (ny+1) ez)
//   z-face (ex,ey,fz) = ex + nx(ey + ny fz)
//   x-edge (ex,fy,fz) = ex + nx(fy + (ny+1) fz)     y-edge (fx,ey,fz) = fx + (nx+1)(ey + ny fz)
//   z-edge (fx,fy,ez) = fx + (nx+1)(fy + (ny+1) ez)
//   vertex (fx,fy,fz) = fx + (nx+1)(fy + (ny+1) fz)

__device__ __forceinline__ bool zdir(const Geom& g, int fz) {
  return (fz == 0 && g.dir_bot) || (fz == g.nz && g.dir_top);
}

// Base address (entry index into the skeleton vector) of element-local entity `ent` of
// element (ex,ey,ez); *dir = entity lies on the Dirichlet boundary.
__device__ __forceinline__ long long entity_base(const Geom& g, int ex, int ey, int ez, int ent, bool* dir) {
  const long long n2 = (long long)g.ni * g.ni, n1 = g.ni;
  const int nx = g.nx, ny = g.ny;
  if (ent < 6) {
    int hi = ent & 1;
    if (ent < 2) {
      int fx = ex + hi;
      *dir = (fx == 0 || fx == nx);
      return g.off_f[0] + (fx + (long long)(nx + 1) * (ey + (long long)ny * ez)) * n2;
    } else if (ent < 4) {
      int fy = ey + hi;
      *dir = (fy == 0 || fy == ny);
      return g.off_f[1] + (ex + (long long)nx * (fy + (long long)(ny + 1) * ez)) * n2;
    } else {
      int fz = ez + hi;
      *dir = zdir(g, fz);
      return g.off_f[2] + (ex + (long long)nx * (ey + (long long)ny * fz)) * n2;
    }
  }
  if (ent < 18) {
    int e = ent - 6, grp = e >> 2, b0 = e & 1, b1 = (e >> 1) & 1;
    if (grp == 0) {          // x-edge at (fy, fz)
      int fy = ey + b0, fz = ez + b1;
      *dir = (fy == 0 || fy == ny) || zdir(g, fz);
      return g.off_e[0] + (ex + (long long)nx * (fy + (long long)(ny + 1) * fz)) * n1;
    } else if (grp == 1) {   // y-edge at (fx, fz)
      int fx = ex + b0, fz = ez + b1;
      *dir = (fx == 0 || fx == nx) || zdir(g, fz);
      return g.off_e[1] + (fx + (long long)(nx + 1) * (ey + (long long)ny * fz)) * n1;
    } else {                 // z-edge at (fx, fy)
      int fx = ex + b0, fy = ey + b1;
      *dir = (fx == 0 || fx == nx) || (fy == 0 || fy == ny);
      return g.off_e[2] + (fx + (long long)(nx + 1) * (fy + (long long)(ny + 1) * ez)) * n1;
    }
  }
  int v = ent - 18;
  int fx = ex + (v & 1), fy = ey + ((v >> 1) & 1), fz = ez + ((v >> 2) & 1);
  *dir = (fx == 0 || fx == nx) || (fy == 0 || fy == ny) || zdir(g, fz);
  return g.off_v + fx + (long long)(nx + 1) * (fy + (long long)(ny + 1) * fz);
}

// Decode skeleton entry q -> local lattice coordinates (gx, gy, gz); returns false for
// padding entries.  *dir = entry lies on the Dirichlet boundary.
__device__ __forceinline__ bool decode_entry(const Geom& g, long long q, int* gx, int* gy, int* gz, bool* dir) {
  const int p = g.p, ni = g.ni, nx = g.nx, ny = g.ny;
  const long long n2 = (long long)ni * ni;
  for (int d = 0; d < 3; ++d) {
    long long o = q - g.off_f[d];
    if (o >= 0 && o < g.n_f[d] * n2) {
      long long id = o / n2;
      int r = (int)(o - id * n2), a = r % ni, b = r / ni;
      if (d == 0) {
        int fx = (int)(id % (nx + 1)); long long t = id / (nx + 1);
        int ey = (int)(t % ny), ez = (int)(t / ny);
        *gx = fx * p; *gy = ey * p + 1 + a; *gz = ez * p + 1 + b;
        *dir = (fx == 0 || fx == nx);
      } else if (d == 1) {
        int ex = (int)(id % nx); long long t = id / nx;
        int fy = (int)(t % (ny + 1)), ez = (int)(t / (ny + 1));
        *gx = ex * p + 1 + a; *gy = fy * p; *gz = ez * p + 1 + b;
        *dir = (fy == 0 || fy == ny);
      } else {
        int ex = (int)(id % nx); long long t = id / nx;
        int ey = (int)(t % ny), fz = (int)(t / ny);
        *gx = ex * p + 1 + a; *gy = ey * p + 1 + b; *gz = fz * p;
        *dir = zdir(g, fz);
      }
      return true;
    }
  }
  for (int d = 0; d < 3; ++d) {
    long long o = q - g.off_e[d];
    if (o >= 0 && o < g.n_e[d] * ni) {
      long long id = o / ni;
      int c = (int)(o - id * ni) + 1;
      if (d == 0) {
        int ex = (int)(id % nx); long long t = id / nx;
        int fy = (int)(t % (ny + 1)), fz = (int)(t / (ny + 1));
        *gx = ex * p + c; *gy = fy * p; *gz = fz * p;
        *dir = (fy == 0 || fy == ny) || zdir(g, fz);
      } else if (d == 1) {
        int fx = (int)(id % (nx + 1)); long long t = id / (nx + 1);
        int ey = (int)(t % ny), fz = (int)(t / ny);
        *gx = fx * p; *gy = ey * p + c; *gz = fz * p;
        *dir = (fx == 0 || fx == nx) || zdir(g, fz);
      } else {
        int fx = (int)(id % (nx + 1)); long long t = id / (nx + 1);
        int fy = (int)(t % (ny + 1)), ez = (int)(t / (ny + 1));
        *gx = fx * p; *gy = fy * p; *gz = ez * p + c;
        *dir = (fx == 0 || fx == nx) || (fy == 0 || fy == ny);
      }
      return true;
    }
  }
  long long o = q - g.off_v;
  if (o >= 0 && o < g.n_v) {
    int fx = (int)(o % (nx + 1)); long long t = o / (nx + 1);
    int fy = (int)(t % (ny + 1)), fz = (int)(t / (ny + 1));
    *gx = fx * p; *gy = fy * p; *gz = fz * p;
    *dir = (fx == 0 || fx == nx) || (fy == 0 || fy == ny) || zdir(g, fz);
    return true;
  }
  return false;
}

// Element-local coordinates (i,j,k) of shell node s (faces, then edges, then vertices).
__device__ __forceinline__ void shell_node(int p, int ni, int s, int* i, int* j, int* k, int* ent, int* loc) {
  const int n2 = ni * ni;
  if (s < 6 * n2) {
    int f = s / n2, r = s - f * n2, a = r % ni + 1, b = r / ni + 1, hi = (f & 1) ? p : 0;
    *ent = f; *loc = r;
    if (f < 2) { *i = hi; *j = a; *k = b; }
    else if (f < 4) { *i = a; *j = hi; *k = b; }
    else { *i = a; *j = b; *k = hi; }
    return;
  }
  s -= 6 * n2;
  if (s < 12 * ni) {
    int e = s / ni, c = s - e * ni + 1, grp = e >> 2;
    int b0 = (e & 1) ? p : 0, b1 = (e & 2) ? p : 0;
    *ent = 6 + e; *loc = c - 1;
    if (grp == 0) { *i = c; *j = b0; *k = b1; }
    else if (grp == 1) { *i = b0; *j = c; *k = b1; }
    else { *i = b0; *j = b1; *k = c; }
    return;
  }
  s -= 12 * ni;
  *ent = 18 + s; *loc = 0;
  *i = (s & 1) ? p : 0; *j = (s & 2) ? p : 0; *k = (s & 4) ? p : 0;
}

// Offset of the shell value at element coords (i,j,k) (a shell node) in the element-local
// shell array [faces 6 n2 | edges 12 ni | vertices 8].
__device__ __forceinline__ int shell_index(int p, int ni, int i, int j, int k) {
  const int n2 = ni * ni;
  bool bi = (i == 0 || i == p), bj = (j == 0 || j == p), bk = (k == 0 || k == p);
  int nb = (int)bi + (int)bj + (int)bk;
  if (nb == 1) {
    if (bi) return (i ? 1 : 0) * n2 + (j - 1) + ni * (k - 1);
    if (bj) return (2 + (j ? 1 : 0)) * n2 + (i - 1) + ni * (k - 1);
    return (4 + (k ? 1 : 0)) * n2 + (i - 1) + ni * (j - 1);
  }
  if (nb == 2) {
    if (!bi) return 6 * n2 + (0 + (j ? 1 : 0) + 2 * (k ? 1 : 0)) * ni + i - 1;
    if (!bj) return 6 * n2 + (4 + (i ? 1 : 0) + 2 * (k ? 1 : 0)) * ni + j - 1;
    return 6 * n2 + (8 + (i ? 1 : 0) + 2 * (j ? 1 : 0)) * ni + k - 1;
  }
  return 6 * n2 + 12 * ni + (i ? 1 : 0) + 2 * (j ? 1 : 0) + 4 * (k ? 1 : 0);
}

// d_e = (h1h2h3/8)(lambda, 4/h1^2, 4/h2^2, 4/h3^2)  (Eq. eq:metriccoeffelement)
__device__ __forceinline__ void metric(const Geom& g, int ex, int ey, int ez, double d[4]) {
  double h1 = g.hx[ex], h2 = g.hy[ey], h3 = g.hz[ez];
  double s = h1 * h2 * h3 * 0.125;
  d[0] = s * g.lam_h;
  d[1] = s * 4.0 / (h1 * h1);
  d[2] = s * 4.0 / (h2 * h2);
  d[3] = s * 4.0 / (h3 * h3);
}

}  // namespace sc
