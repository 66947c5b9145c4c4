// Condensed operator for p = 2 (n_I = 1), uniform geometry.
//
// At p = 2 an element has one interior point and 26 shell values (6 faces, 12 edges, 8 vertices
// of one value each), so the tile-column machinery's per-step cost dominates.  Here a warp takes
// 32 consecutive elements of one x-row and a lane one element, entirely in registers:
//  * every entity array is x-fastest, so each lane's loads / stores of its own entities
//    are coalesced across the warp;
//  * the entities an element shares with its x-neighbour (E face, the ib = 1 edges / vertices) are
//    the neighbour lane's ib = 0 entities: read by a shuffle down, and the contributions summed by
//    a shuffle up, so each is written once per warp;
//  * warps are colour-scheduled by (x-chunk parity, ey parity, ez parity): no two warps of one
//    launch share an entity, so the assembly is a plain read-modify-write of y (zeroed first).
// Arithmetic: Table 2 / Eq. 26 at n_I = 1 -- u = c1 (W + E) + c2 (S + N) +
// c3 (B + T), v = u / D, faces -= c_d v; primary part of faces, edges and vertices from the
// arrowhead rows of Ktilde (the same closed forms as kernels_big.cu with every line sum a0 * value).
#include <cuda_runtime.h>
#include <string.h>
#include "sc_device.cuh"

namespace sc {

struct P2Params {
  Geom g;
  const double* x;
  double* y;
  const double* done;
  BigCoef cf;
};

#ifndef SC_P2_MINB
#define SC_P2_MINB 2
#endif
#ifndef SC_P2_ITEMS
#define SC_P2_ITEMS 2
#endif
// Warp item wid of colour `colour`: 32 consecutive elements of one x-row (see the file comment).
__device__ __forceinline__ void p2_item(const P2Params& P, int colour, long long wid) {
  const Geom& g = P.g;
  const BigCoef& cf = P.cf;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int cp = colour & 1, ry = (colour >> 1) & 1, rz = colour >> 2;
  const int nch = (nx + 31) >> 5;
  const int cc = (nch - cp + 1) >> 1, cy = (ny - ry + 1) >> 1, cz = (nz - rz + 1) >> 1;
  if (wid >= (long long)cc * cy * cz) return;   // warp-uniform
  const int lane = threadIdx.x & 31;
  const int chunk = cp + 2 * (int)(wid % cc);
  const int ey = ry + 2 * (int)((wid / cc) % cy), ez = rz + 2 * (int)(wid / ((long long)cc * cy));
  const int ex = chunk * 32 + lane;
  const bool act = ex < nx;
  const bool last = act && (lane == 31 || ex == nx - 1);
  const long long nx1 = nx + 1, ny1 = ny + 1;
  // entity indices (n_I = 1: one value per entity) and Dirichlet flags
  auto xf = [&](int fx, int fy_, int fz_) { return g.off_f[0] + fx + nx1 * (fy_ + (long long)ny * fz_); };
  auto yf = [&](int ex_, int fy, int ez_) { return g.off_f[1] + ex_ + (long long)nx * (fy + ny1 * ez_); };
  auto zf = [&](int ex_, int ey_, int fz) { return g.off_f[2] + ex_ + (long long)nx * (ey_ + (long long)ny * fz); };
  auto xe = [&](int ex_, int fy, int fz) { return g.off_e[0] + ex_ + (long long)nx * (fy + ny1 * fz); };
  auto ye = [&](int fx, int ey_, int fz) { return g.off_e[1] + fx + nx1 * (ey_ + (long long)ny * fz); };
  auto ze = [&](int fx, int fy, int ez_) { return g.off_e[2] + fx + nx1 * (fy + ny1 * ez_); };
  auto vx = [&](int fx, int fy, int fz) { return g.off_v + fx + nx1 * (fy + ny1 * fz); };
  const bool dX0 = ex == 0, dX1 = ex + 1 == nx;                 // x-planes fx = ex, ex + 1
  const bool dY[2] = {ey == 0, ey + 1 == ny};                   // y-planes fy = ey + jb
  const bool dZ[2] = {zdir(g, ez), zdir(g, ez + 1)};            // z-planes fz = ez + kb
  const double* X = P.x;
  auto ld = [&](long long a, bool dir) { return (act && !dir) ? __ldg(X + a) : 0.0; };

  // ---- a3: own (ib = 0) entities; the ib = 1 ones are the next lane's
  const double W = ld(xf(ex, ey, ez), dX0);
  const double S = ld(yf(ex, ey, ez), dY[0]), N = ld(yf(ex, ey + 1, ez), dY[1]);
  const double Bf = ld(zf(ex, ey, ez), dZ[0]), T = ld(zf(ex, ey, ez + 1), dZ[1]);
  double Xe[2][2], Y0[2], Z0[2], V0[2][2];
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    Y0[b] = ld(ye(ex, ey, ez + b), dX0 || dZ[b]);
    Z0[b] = ld(ze(ex, ey + b, ez), dX0 || dY[b]);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      Xe[b][c] = ld(xe(ex, ey + b, ez + c), dY[b] || dZ[c]);
      V0[b][c] = ld(vx(ex, ey + b, ez + c), dX0 || dY[b] || dZ[c]);
    }
  }
  // the y lines this warp read-modify-writes at the end: prefetched into L2 now (lanes 0 / 16
  // cover the 256 bytes of the warp's 32 consecutive entries of each of the 17 entity rows)
  if ((lane & 15) == 0 && act) {
    const double* Yp = P.y;
    auto pf = [&](long long a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(Yp + a)); };
    pf(xf(ex, ey, ez)); pf(yf(ex, ey, ez)); pf(yf(ex, ey + 1, ez)); pf(zf(ex, ey, ez)); pf(zf(ex, ey, ez + 1));
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      pf(ye(ex, ey, ez + b)); pf(ze(ex, ey + b, ez));
#pragma unroll
      for (int c = 0; c < 2; ++c) { pf(xe(ex, ey + b, ez + c)); pf(vx(ex, ey + b, ez + c)); }
    }
  }
  double E = __shfl_down_sync(0xffffffffu, W, 1), Y1[2], Z1[2], V1[2][2];
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    Y1[b] = __shfl_down_sync(0xffffffffu, Y0[b], 1);
    Z1[b] = __shfl_down_sync(0xffffffffu, Z0[b], 1);
#pragma unroll
    for (int c = 0; c < 2; ++c) V1[b][c] = __shfl_down_sync(0xffffffffu, V0[b][c], 1);
  }
  if (last) {   // the row's (or the chunk's) last element: its ib = 1 entities directly
    E = ld(xf(ex + 1, ey, ez), dX1);
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      Y1[b] = ld(ye(ex + 1, ey, ez + b), dX1 || dZ[b]);
      Z1[b] = ld(ze(ex + 1, ey + b, ez), dX1 || dY[b]);
#pragma unroll
      for (int c = 0; c < 2; ++c) V1[b][c] = ld(vx(ex + 1, ey + b, ez + c), dX1 || dY[b] || dZ[c]);
    }
  }
  if (!act) {
    E = 0.0;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      Y1[b] = Z1[b] = 0.0;
      V1[b][0] = V1[b][1] = 0.0;
    }
  }

  // ---- a4-a6: condensed part (one interior point)
  const double a0 = cf.a0[0], lam = cf.lam[0], K00 = cf.K00, K0p = cf.K0p, w0 = cf.w0, w02 = w0 * w0;
  const double d0 = cf.d[0], d1 = cf.d[1], d2 = cf.d[2], d3 = cf.d[3];
  const double Dinv = 1.0 / (d0 + cf.dl[0][0] + cf.dl[1][0] + cf.dl[2][0]);
  const double v = (cf.c[0][0] * (W + E) + cf.c[1][0] * (S + N) + cf.c[2][0] * (Bf + T)) * Dinv;
  const double Qx = cf.c[0][0] * v, Qy = cf.c[1][0] * v, Qz = cf.c[2][0] * v;
  // ---- a7: primary part.  Faces: fd self + K0p opposite + bounding edges (Eq. 26 generalised)
  const double fdx = cf.F0[0] + cf.L[1][0] + cf.L[2][0], fdy = cf.F0[1] + cf.L[0][0] + cf.L[2][0],
               fdz = cf.F0[2] + cf.L[0][0] + cf.L[1][0];
  const double e0 = cf.e[0][0], e1 = cf.e[1][0], e2 = cf.e[2][0];
  const double oW = fdx * W + cf.k0p[0] * E + e1 * (Z0[0] + Z0[1]) + e2 * (Y0[0] + Y0[1]) - Qx;
  const double oE = fdx * E + cf.k0p[0] * W + e1 * (Z1[0] + Z1[1]) + e2 * (Y1[0] + Y1[1]) - Qx;
  const double oS = fdy * S + cf.k0p[1] * N + e0 * (Z0[0] + Z1[0]) + e2 * (Xe[0][0] + Xe[0][1]) - Qy;
  const double oN = fdy * N + cf.k0p[1] * S + e0 * (Z0[1] + Z1[1]) + e2 * (Xe[1][0] + Xe[1][1]) - Qy;
  const double oB = fdz * Bf + cf.k0p[2] * T + e0 * (Y0[0] + Y1[0]) + e1 * (Xe[0][0] + Xe[1][0]) - Qz;
  const double oT = fdz * T + cf.k0p[2] * Bf + e0 * (Y0[1] + Y1[1]) + e1 * (Xe[0][1] + Xe[1][1]) - Qz;
  // Ktilde row 0 (node at coordinate 0) / row p applied along a boundary direction: the pair of
  // nodes (lo, hi) plus the line's interior (one node, a0 u)
  auto row = [&](int hi, double lo_v, double hi_v, double line) {
    return (hi ? fma(K0p, lo_v, K00 * hi_v) : fma(K00, lo_v, K0p * hi_v)) + a0 * line;
  };
  // edges: x-edge (jb, kb): along x the two vertices; boundary y (bit jb): x-edges (0|1, kb) and
  // the z-face kb; boundary z (bit kb): x-edges (jb, 0|1) and the y-face jb
  const double Yf[2] = {S, N}, Zf[2] = {Bf, T}, Xf[2] = {W, E};
  double oX[2][2], oY[2][2], oZ[2][2], oV[2][2][2];
#pragma unroll
  for (int b = 0; b < 2; ++b)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const double u = Xe[b][c];
      const double tal = a0 * (V0[b][c] + V1[b][c]) + lam * u;
      const double t1 = row(b, Xe[0][c], Xe[1][c], Zf[c]);
      const double t2 = row(c, Xe[b][0], Xe[b][1], Yf[b]);
      oX[b][c] = w02 * (d0 * u + d1 * tal) + w0 * (d2 * t1 + d3 * t2);
    }
  // y-edge (ib, kb): along y the vertices (ib, 0|1, kb); boundary x: y-edges (0|1, kb), z-face kb;
  // boundary z: y-edges (ib, 0|1), x-face ib
#pragma unroll
  for (int ib = 0; ib < 2; ++ib)
#pragma unroll
    for (int kb = 0; kb < 2; ++kb) {
      const double u = ib ? Y1[kb] : Y0[kb];
      const double tal = a0 * ((ib ? V1[0][kb] : V0[0][kb]) + (ib ? V1[1][kb] : V0[1][kb])) + lam * u;
      const double t1 = row(ib, Y0[kb], Y1[kb], Zf[kb]);
      const double t2 = row(kb, ib ? Y1[0] : Y0[0], ib ? Y1[1] : Y0[1], Xf[ib]);
      oY[ib][kb] = w02 * (d0 * u + d2 * tal) + w0 * (d1 * t1 + d3 * t2);
    }
  // z-edge (ib, jb): along z the vertices (ib, jb, 0|1); boundary x: z-edges (0|1, jb), y-face jb;
  // boundary y: z-edges (ib, 0|1), x-face ib
#pragma unroll
  for (int ib = 0; ib < 2; ++ib)
#pragma unroll
    for (int jb = 0; jb < 2; ++jb) {
      const double u = ib ? Z1[jb] : Z0[jb];
      const double tal = a0 * ((ib ? V1[jb][0] : V0[jb][0]) + (ib ? V1[jb][1] : V0[jb][1])) + lam * u;
      const double t1 = row(ib, Z0[jb], Z1[jb], Yf[jb]);
      const double t2 = row(jb, ib ? Z1[0] : Z0[0], ib ? Z1[1] : Z0[1], Xf[ib]);
      oZ[ib][jb] = w02 * (d0 * u + d3 * tal) + w0 * (d1 * t1 + d2 * t2);
    }
  // vertices: along each direction the partner vertex and the edge through the vertex
#pragma unroll
  for (int ib = 0; ib < 2; ++ib)
#pragma unroll
    for (int jb = 0; jb < 2; ++jb)
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        const double u = ib ? V1[jb][kb] : V0[jb][kb];
        const double tx = row(ib, V0[jb][kb], V1[jb][kb], Xe[jb][kb]);
        const double ty = row(jb, ib ? V1[0][kb] : V0[0][kb], ib ? V1[1][kb] : V0[1][kb], ib ? Y1[kb] : Y0[kb]);
        const double tz = row(kb, ib ? V1[jb][0] : V0[jb][0], ib ? V1[jb][1] : V0[jb][1], ib ? Z1[jb] : Z0[jb]);
        oV[ib][jb][kb] = w02 * (w0 * d0 * u + d1 * tx + d2 * ty + d3 * tz);
      }

  // ---- a8: assembly.  ib = 0 entities: own + the previous lane's ib = 1 contribution; the last
  // element also writes its ib = 1 entities; every write is a read-modify-write of y.
  const bool first = lane == 0;
  auto up = [&](double val) {
    const double l = __shfl_up_sync(0xffffffffu, val, 1);
    return first ? 0.0 : l;
  };
  double w_[17];
  long long a_[17];
  bool m_[17];
  int n = 0;
  auto put = [&](long long a, bool dir, double val) { a_[n] = a; m_[n] = act && !dir; w_[n] = val; ++n; };
  put(xf(ex, ey, ez), dX0, oW + up(oE));
  put(yf(ex, ey, ez), dY[0], oS);
  put(yf(ex, ey + 1, ez), dY[1], oN);
  put(zf(ex, ey, ez), dZ[0], oB);
  put(zf(ex, ey, ez + 1), dZ[1], oT);
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    put(ye(ex, ey, ez + b), dX0 || dZ[b], oY[0][b] + up(oY[1][b]));
    put(ze(ex, ey + b, ez), dX0 || dY[b], oZ[0][b] + up(oZ[1][b]));
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      put(xe(ex, ey + b, ez + c), dY[b] || dZ[c], oX[b][c]);
      put(vx(ex, ey + b, ez + c), dX0 || dY[b] || dZ[c], oV[0][b][c] + up(oV[1][b][c]));
    }
  }
  double* Y = P.y;
  // the last lane's ib = 1 entities (next chunk's W side) join the batch: all old values are
  // loaded before the first store (a load after a store to y cannot be moved above it, so
  // read-modify-writes issued one by one run as a chain of DRAM round trips)
  const long long ae = xf(ex + 1, ey, ez);
  const bool lx = last && !dX1;
  long long at_[9];
  bool mt_[9];
  double wt_[9];
  int nt = 0;
  auto putt = [&](long long a, bool ok, double val) { at_[nt] = a; mt_[nt] = ok; wt_[nt] = val; ++nt; };
  putt(ae, lx, oE);
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    putt(ye(ex + 1, ey, ez + b), lx && !dZ[b], oY[1][b]);
    putt(ze(ex + 1, ey + b, ez), lx && !dY[b], oZ[1][b]);
#pragma unroll
    for (int c = 0; c < 2; ++c) putt(vx(ex + 1, ey + b, ez + c), lx && !(dY[b] || dZ[c]), oV[1][b][c]);
  }
  double old[17], oldt[9];
#pragma unroll
  for (int q = 0; q < 17; ++q) old[q] = m_[q] ? Y[a_[q]] : 0.0;
#pragma unroll
  for (int q = 0; q < 9; ++q) oldt[q] = mt_[q] ? Y[at_[q]] : 0.0;
#pragma unroll
  for (int q = 0; q < 17; ++q)
    if (m_[q]) Y[a_[q]] = old[q] + w_[q];
#pragma unroll
  for (int q = 0; q < 9; ++q)
    if (mt_[q]) Y[at_[q]] = oldt[q] + wt_[q];
}

// L2 prefetch of the 17 x rows (and y rows) of warp item wid: issued one item ahead, so the next
// item's loads find their lines in L2.
__device__ __forceinline__ void p2_prefetch(const P2Params& P, int colour, long long wid) {
  const Geom& g = P.g;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int cp = colour & 1, ry = (colour >> 1) & 1, rz = colour >> 2;
  const int nch = (nx + 31) >> 5;
  const int cc = (nch - cp + 1) >> 1, cy = (ny - ry + 1) >> 1, cz = (nz - rz + 1) >> 1;
  if (wid >= (long long)cc * cy * cz) return;
  const int lane = threadIdx.x & 31;
  const int chunk = cp + 2 * (int)(wid % cc);
  const int ey = ry + 2 * (int)((wid / cc) % cy), ez = rz + 2 * (int)(wid / ((long long)cc * cy));
  const int ex = chunk * 32 + lane;
  if ((lane & 15) != 0 || ex >= nx) return;
  const long long nx1 = nx + 1, ny1 = ny + 1;
  const long long a[17] = {
      g.off_f[0] + ex + nx1 * (ey + (long long)ny * ez), g.off_f[1] + ex + (long long)nx * (ey + ny1 * ez),
      g.off_f[1] + ex + (long long)nx * (ey + 1 + ny1 * ez), g.off_f[2] + ex + (long long)nx * (ey + (long long)ny * ez),
      g.off_f[2] + ex + (long long)nx * (ey + (long long)ny * (ez + 1)),
      g.off_e[1] + ex + nx1 * (ey + (long long)ny * ez), g.off_e[1] + ex + nx1 * (ey + (long long)ny * (ez + 1)),
      g.off_e[2] + ex + nx1 * (ey + ny1 * ez), g.off_e[2] + ex + nx1 * (ey + 1 + ny1 * ez),
      g.off_e[0] + ex + (long long)nx * (ey + ny1 * ez), g.off_e[0] + ex + (long long)nx * (ey + ny1 * (ez + 1)),
      g.off_e[0] + ex + (long long)nx * (ey + 1 + ny1 * ez), g.off_e[0] + ex + (long long)nx * (ey + 1 + ny1 * (ez + 1)),
      g.off_v + ex + nx1 * (ey + ny1 * ez), g.off_v + ex + nx1 * (ey + ny1 * (ez + 1)),
      g.off_v + ex + nx1 * (ey + 1 + ny1 * ez), g.off_v + ex + nx1 * (ey + 1 + ny1 * (ez + 1))};
#pragma unroll
  for (int q = 0; q < 17; ++q) asm volatile("prefetch.global.L2 [%0];" ::"l"(P.x + a[q]));
}

// SC_P2_ITEMS consecutive warp items per warp, each prefetching the next one's x rows.
__global__ void __launch_bounds__(256, SC_P2_MINB) k_apply_p2(const __grid_constant__ P2Params P, int colour) {
  if (P.done != nullptr && *P.done != 0.0) return;
  const long long w0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * SC_P2_ITEMS;
#pragma unroll 1
  for (int t = 0; t < SC_P2_ITEMS; ++t) {
    if (t + 1 < SC_P2_ITEMS) p2_prefetch(P, colour, w0 + t + 1);
    p2_item(P, colour, w0 + t);
  }
}

int launch_apply_p2(const Geom& g, const double* x, double* y, const double* done, const void* coef, void* stream,
                    int* nl, void* events) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  cudaError_t err = cudaMemsetAsync(y, 0, sizeof(double) * g.n_total, st);
  if (err != cudaSuccess) return err;
  if (ev) cudaEventRecord(ev[0], st);
  P2Params P;
  P.g = g; P.x = x; P.y = y; P.done = done;
  memcpy(&P.cf, coef, sizeof(BigCoef));
  const int nch = (g.nx + 31) >> 5;
  for (int c = 0; c < 8; ++c) {
    const int cp = c & 1, ry = (c >> 1) & 1, rz = c >> 2;
    const long long warps = (long long)((nch - cp + 1) >> 1) * ((g.ny - ry + 1) >> 1) * ((g.nz - rz + 1) >> 1);
    if (warps <= 0) continue;
    const long long wgroups = (warps + SC_P2_ITEMS - 1) / SC_P2_ITEMS;
    k_apply_p2<<<(unsigned)((wgroups + 7) / 8), 256, 0, st>>>(P, c);
    (*nl)++;
  }
  if (ev) cudaEventRecord(ev[1], st);
  return cudaGetLastError();
}

}  // namespace sc
