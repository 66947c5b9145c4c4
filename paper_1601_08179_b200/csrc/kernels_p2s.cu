// Condensed operator for p = 2 (n_I = 1) as an owner-computes stencil, uniform geometry, one rank
// (VERDICT r1 item 6).
//
// At p = 2 every skeleton entity holds one value, so the skeleton is the GLL lattice without the
// element centres.  On a uniform grid the assembled condensed operator R^ H~ R^T (Table 2 / Eq. 26,
// PAPER.md P:415-440, plus the condensed part -H_BI H_II^{-1} H_IB) is a constant-coefficient
// stencil per node class: the output at a free node G is the sum over the elements containing G of
// their element-matrix rows, and every such element lies inside the domain.  With lattice offsets:
//   vertex : itself and +-1, +-2 along each axis                                 (13 points)
//   edge   : itself, +-1 along the edge, +-1 and +-2 along both transverse axes   (11 points)
//   face   : itself, +-2 along the normal, +-1 along both in-plane axes, and the
//            (+-1 normal, +-1 in-plane) diagonals (the condensed face-face part)   (15 points)
// The coefficients come from the element matrix evaluated on the host (p2s_make_coef, which also
// checks that no coupling falls outside these lists).  A thread owns the lattice cell (fx, fy, fz):
// the vertex, the three edges and the three faces at its low corner (7 nodes), loads the stencil
// values it needs (each entity array is x-fastest, so a warp's loads of one neighbour are one
// coalesced row; the rows are shared by neighbouring warps through L1 / L2) and writes each of its
// outputs once: no colours, no memset, no read-modify-write of y, no atomics (the colour-scheduled
// kernel moved 5.2x the algorithmic bytes).
#include <cuda_runtime.h>
#include <string.h>
#include <string>
#include <utility>
#include <vector>
#include "sc_device.cuh"

namespace sc {

namespace p2s {

// node classes owned by a cell, by sub-position (a, b, c) in the 2 x 2 x 2 lattice cell
constexpr int kSub[7][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {0, 1, 1}, {1, 0, 1}, {1, 1, 0}};
constexpr int kN[7] = {13, 11, 11, 11, 15, 15, 15};
constexpr int kOff[7][15][3] = {
    // vertex
    {{0, 0, 0}, {-1, 0, 0}, {1, 0, 0}, {-2, 0, 0}, {2, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, -2, 0}, {0, 2, 0},
     {0, 0, -1}, {0, 0, 1}, {0, 0, -2}, {0, 0, 2}},
    // x-edge
    {{0, 0, 0}, {-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, -2, 0}, {0, 2, 0}, {0, 0, -1}, {0, 0, 1},
     {0, 0, -2}, {0, 0, 2}},
    // y-edge
    {{0, 0, 0}, {0, -1, 0}, {0, 1, 0}, {-1, 0, 0}, {1, 0, 0}, {-2, 0, 0}, {2, 0, 0}, {0, 0, -1}, {0, 0, 1},
     {0, 0, -2}, {0, 0, 2}},
    // z-edge
    {{0, 0, 0}, {0, 0, -1}, {0, 0, 1}, {-1, 0, 0}, {1, 0, 0}, {-2, 0, 0}, {2, 0, 0}, {0, -1, 0}, {0, 1, 0},
     {0, -2, 0}, {0, 2, 0}},
    // x-face
    {{0, 0, 0}, {-2, 0, 0}, {2, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}, {-1, -1, 0}, {-1, 1, 0},
     {1, -1, 0}, {1, 1, 0}, {-1, 0, -1}, {-1, 0, 1}, {1, 0, -1}, {1, 0, 1}},
    // y-face
    {{0, 0, 0}, {0, -2, 0}, {0, 2, 0}, {-1, 0, 0}, {1, 0, 0}, {0, 0, -1}, {0, 0, 1}, {-1, -1, 0}, {-1, 1, 0},
     {1, -1, 0}, {1, 1, 0}, {0, -1, -1}, {0, -1, 1}, {0, 1, -1}, {0, 1, 1}},
    // z-face
    {{0, 0, 0}, {0, 0, -2}, {0, 0, 2}, {-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {-1, 0, -1}, {-1, 0, 1},
     {1, 0, -1}, {1, 0, 1}, {0, -1, -1}, {0, -1, 1}, {0, 1, -1}, {0, 1, 1}},
};

struct Params {
  Geom g;
  const double* x;
  double* y;
  const double* done;
  long long off[7], rs[7], ps[7];   // per node class (sub-position order of kSub): array offset, y / z strides
  double coef[7][15];
};

// floor((a + d) / 2) and (a + d) mod 2 for a in {0, 1}, d in [-2, 2]
__host__ __device__ constexpr int cell_of(int v) { return v >= 0 ? v / 2 : -((1 - v) / 2); }
__host__ __device__ constexpr int sub_of(int v) { return v & 1; }
// node class of sub-position (sx, sy, sz), in kSub order
__host__ __device__ constexpr int cls_of(int sx, int sy, int sz) {
  return (sx == 0 && sy == 0 && sz == 0) ? 0 : (sx == 1 && sy == 0 && sz == 0) ? 1 : (sx == 0 && sy == 1 && sz == 0) ? 2
       : (sx == 0 && sy == 0 && sz == 1) ? 3 : (sx == 0 && sy == 1 && sz == 1) ? 4 : (sx == 1 && sy == 0 && sz == 1) ? 5 : 6;
}

// Per-thread state: the skeleton index of this cell's node of every class (cx = cy = cz = 0); a
// neighbour cell's node is base + cx + cy rs + cz ps.  CHECK: lattice coordinates of the cell for
// the free-node test (strictly inside the domain); interior warps skip it.
struct Cell {
  long long base[7];
  int fx, fy, fz;
};

template <bool CHECK, int C, int K>
__device__ __forceinline__ double term(const Params& P, const Cell& c) {
  constexpr int vx = kSub[C][0] + kOff[C][K][0], vy = kSub[C][1] + kOff[C][K][1], vz = kSub[C][2] + kOff[C][K][2];
  constexpr int CX = cell_of(vx), CY = cell_of(vy), CZ = cell_of(vz);
  constexpr int SX = sub_of(vx), SY = sub_of(vy), SZ = sub_of(vz);
  constexpr int N = cls_of(SX, SY, SZ);
  const long long i = c.base[N] + CX + CY * P.rs[N] + CZ * P.ps[N];
  if (!CHECK) return P.coef[C][K] * __ldg(P.x + i);
  const Geom& g = P.g;
  const int X = 2 * (c.fx + CX) + SX, Y = 2 * (c.fy + CY) + SY, Z = 2 * (c.fz + CZ) + SZ;
  const bool ok = X >= 1 && X <= 2 * g.nx - 1 && Y >= 1 && Y <= 2 * g.ny - 1 && Z >= 1 && Z <= 2 * g.nz - 1;
  const double v = __ldg(P.x + (ok ? i : 0));   // branch-free: a valid address, masked
  return P.coef[C][K] * (ok ? v : 0.0);
}

template <bool CHECK, int C, int... K>
__device__ __forceinline__ double stencil(const Params& P, const Cell& c, std::integer_sequence<int, K...>) {
  double s = 0.0;
  ((s += term<CHECK, C, K>(P, c)), ...);
  return s;
}

// Output of class C of the cell: written if the node exists (0 at Dirichlet nodes).
template <bool CHECK, int C>
__device__ __forceinline__ void out(const Params& P, const Cell& c) {
  const Geom& g = P.g;
  constexpr int a = kSub[C][0], b = kSub[C][1], cc = kSub[C][2];
  if (!CHECK) {
    P.y[c.base[C]] = stencil<false, C>(P, c, std::make_integer_sequence<int, kN[C]>{});
    return;
  }
  const int X = 2 * c.fx + a, Y = 2 * c.fy + b, Z = 2 * c.fz + cc;
  if (X > 2 * g.nx || Y > 2 * g.ny || Z > 2 * g.nz) return;   // entity does not exist
  const bool fr = X >= 1 && X <= 2 * g.nx - 1 && Y >= 1 && Y <= 2 * g.ny - 1 && Z >= 1 && Z <= 2 * g.nz - 1;
  const double v = fr ? stencil<true, C>(P, c, std::make_integer_sequence<int, kN[C]>{}) : 0.0;
  P.y[c.base[C]] = v;
}

template <bool CHECK>
__device__ __forceinline__ void all_out(const Params& P, const Cell& c) {
  out<CHECK, 0>(P, c); out<CHECK, 1>(P, c); out<CHECK, 2>(P, c); out<CHECK, 3>(P, c);
  out<CHECK, 4>(P, c); out<CHECK, 5>(P, c); out<CHECK, 6>(P, c);
}

#ifndef SC_P2S_MINB
#define SC_P2S_MINB 5
#endif
__global__ void __launch_bounds__(256, SC_P2S_MINB) k_apply_p2s(const __grid_constant__ Params P) {
  if (P.done != nullptr && *P.done != 0.0) return;
  const Geom& g = P.g;
  const int nchunk = (g.nx + 1 + 31) >> 5;
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nrow = (long long)(g.ny + 1) * (g.nz + 1);
  if (w >= nrow * nchunk) return;
  const int chunk = (int)(w % nchunk);
  const long long row = w / nchunk;
  Cell c;
  c.fy = (int)(row % (g.ny + 1));
  c.fz = (int)(row / (g.ny + 1));
  c.fx = chunk * 32 + (threadIdx.x & 31);
  if (c.fx > g.nx) return;
#pragma unroll
  for (int q = 0; q < 7; ++q) c.base[q] = P.off[q] + c.fx + c.fy * P.rs[q] + c.fz * P.ps[q];
  // warp-uniform: every cell of the warp (and every neighbour it reads) strictly inside the domain
  const int x0 = chunk * 32, x1 = min(x0 + 31, g.nx);
  const bool interior = x0 >= 2 && x1 <= g.nx - 2 && c.fy >= 2 && c.fy <= g.ny - 2 && c.fz >= 2 && c.fz <= g.nz - 2;
  if (interior) all_out<false>(P, c);
  else all_out<true>(P, c);
}

// padding entries of y (between the 256-byte aligned entity arrays) are written as 0
__global__ void k_p2s_padding(Geom g, double* __restrict__ y) {
  const long long ends[7] = {g.off_f[0] + g.n_f[0], g.off_f[1] + g.n_f[1], g.off_f[2] + g.n_f[2],
                             g.off_e[0] + g.n_e[0], g.off_e[1] + g.n_e[1], g.off_e[2] + g.n_e[2], g.off_v + g.n_v};
  const long long nexts[7] = {g.off_f[1], g.off_f[2], g.off_e[0], g.off_e[1], g.off_e[2], g.off_v, g.n_total};
  for (int q = 0; q < 7; ++q)
    for (long long i = ends[q] + threadIdx.x; i < nexts[q]; i += blockDim.x) y[i] = 0.0;
}

}  // namespace p2s

// Host: stencil coefficients from the p = 2 element matrix in the transformed basis (m = (w0, 1, w0),
// Ktilde rows (K00, a0, K0p), (a0, Lam, ap), (K0p, ap, K00); condensed part -H_sI H_Is' / D on face
// pairs), summed over the elements containing a node of each class.  Returns false (with a message)
// if a coupling falls outside the compiled offset lists.
bool p2s_make_coef(const double d[4], double lam, double a0, double ap, double K00, double K0p, double w0,
                   std::vector<double>& coef, std::string& err) {
  const double m[3] = {w0, 1.0, w0};
  const double Kt[3][3] = {{K00, a0, K0p}, {a0, lam, ap}, {K0p, ap, K00}};
  const double D = d[0] + (d[1] + d[2] + d[3]) * lam;
  auto face_dir = [](const int s[3]) {
    int nb = 0, dir = -1;
    for (int q = 0; q < 3; ++q)
      if (s[q] != 1) { ++nb; dir = q; }
    return nb == 1 ? dir : -1;
  };
  auto H = [&](const int s[3], const int t[3]) {
    double v = 0.0;
    if (s[0] == t[0] && s[1] == t[1] && s[2] == t[2]) v += d[0] * m[s[0]] * m[s[1]] * m[s[2]];
    for (int dir = 0; dir < 3; ++dir) {
      const int o1 = (dir + 1) % 3, o2 = (dir + 2) % 3;
      if (s[o1] != t[o1] || s[o2] != t[o2]) continue;
      const bool full = s[o1] != 1 || s[o2] != 1;
      if (!full && (s[dir] == 1 || t[dir] == 1)) continue;
      v += d[1 + dir] * m[s[o1]] * m[s[o2]] * Kt[s[dir]][t[dir]];
    }
    const int fs = face_dir(s), ft = face_dir(t);
    if (fs >= 0 && ft >= 0) {
      const double as = s[fs] == 0 ? a0 : ap, at = t[ft] == 0 ? a0 : ap;
      v -= d[1 + fs] * as * d[1 + ft] * at / D;
    }
    return v;
  };
  coef.assign(7 * 15, 0.0);
  for (int c = 0; c < 7; ++c) {
    // accumulated couplings of the node G = sub + (2, 2, 2) by offset (5 x 5 x 5 window)
    double acc[5][5][5] = {};
    bool hit[5][5][5] = {};
    const int G[3] = {p2s::kSub[c][0] + 2, p2s::kSub[c][1] + 2, p2s::kSub[c][2] + 2};
    for (int ox = 0; ox <= 4; ox += 2)
      for (int oy = 0; oy <= 4; oy += 2)
        for (int oz = 0; oz <= 4; oz += 2) {
          const int s[3] = {G[0] - ox, G[1] - oy, G[2] - oz};
          bool in = true;
          for (int q = 0; q < 3; ++q) in &= s[q] >= 0 && s[q] <= 2;
          if (!in || (s[0] == 1 && s[1] == 1 && s[2] == 1)) continue;
          for (int tx = 0; tx <= 2; ++tx)
            for (int ty = 0; ty <= 2; ++ty)
              for (int tz = 0; tz <= 2; ++tz) {
                if (tx == 1 && ty == 1 && tz == 1) continue;
                const int t[3] = {tx, ty, tz};
                const double h = H(s, t);
                const int dx = ox + tx - G[0], dy = oy + ty - G[1], dz = oz + tz - G[2];
                acc[dx + 2][dy + 2][dz + 2] += h;
                hit[dx + 2][dy + 2][dz + 2] |= (h != 0.0);
              }
        }
    bool used[5][5][5] = {};
    for (int k = 0; k < p2s::kN[c]; ++k) {
      const int* o = p2s::kOff[c][k];
      coef[c * 15 + k] = acc[o[0] + 2][o[1] + 2][o[2] + 2];
      used[o[0] + 2][o[1] + 2][o[2] + 2] = true;
    }
    for (int i = 0; i < 5; ++i)
      for (int j = 0; j < 5; ++j)
        for (int k = 0; k < 5; ++k)
          if (hit[i][j][k] && !used[i][j][k] && acc[i][j][k] != 0.0) {
            err = "p2s stencil: coupling outside the compiled offsets (class " + std::to_string(c) + ")";
            return false;
          }
  }
  return true;
}

int launch_apply_p2s(const Geom& g, const double* x, double* y, const double* done, const double* coef, void* stream,
                     int* nl, void* events) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  p2s::Params P;
  memset(&P, 0, sizeof(P));
  P.g = g; P.x = x; P.y = y; P.done = done;
  memcpy(P.coef, coef, sizeof(P.coef));
  {  // entity arrays in kSub order: vertex, x-edge, y-edge, z-edge, x-face, y-face, z-face
    const long long nx = g.nx, ny = g.ny, nx1 = nx + 1, ny1 = ny + 1;
    const long long off[7] = {g.off_v, g.off_e[0], g.off_e[1], g.off_e[2], g.off_f[0], g.off_f[1], g.off_f[2]};
    const long long xc[7] = {nx1, nx, nx1, nx1, nx1, nx, nx};     // entities per x-row
    const long long yc[7] = {ny1, ny1, ny, ny1, ny, ny1, ny};     // rows per z-plane
    for (int q = 0; q < 7; ++q) { P.off[q] = off[q]; P.rs[q] = xc[q]; P.ps[q] = xc[q] * yc[q]; }
  }
  const long long warps = (long long)((g.nx + 1 + 31) >> 5) * (g.ny + 1) * (g.nz + 1);
  const long long blocks = (warps + 7) / 8;
  if (ev) cudaEventRecord(ev[0], st);
  p2s::k_apply_p2s<<<(unsigned)blocks, 256, 0, st>>>(P);
  p2s::k_p2s_padding<<<1, 256, 0, st>>>(g, y);
  *nl += 2;
  if (ev) cudaEventRecord(ev[1], st);
  return cudaGetLastError();
}

}  // namespace sc
