// Condensed operator for p = 3, 4 (n_I = 2, 3), uniform geometry:
// the row-warp scheme of kernels_p2.cu with the element data staged in shared memory.
//
// A warp takes 32 consecutive elements of one x-row, a lane one element.  The warp copies the
// rows its elements touch into its own shared-memory slice -- x-faces (33 entities), the S / N
// y-face rows, the B / T z-face rows, 4 x-edge rows, 2 y-edge and 2 z-edge rows (33 entities),
// 4 vertex rows (33) -- each a contiguous range of the skeleton vector, with
// 8-byte cp.async.  Every lane then computes its element (Table 2 / Eq. 26 of PAPER.md
// condensed part in registers, primary part of faces, edges and vertices from the
// arrowhead rows of Ktilde) and adds the results into y: entities shared with the x-neighbour
// (W/E face, y- and z-edges, vertices at fx) are summed by a lane shuffle and written once;
// warps are colour-scheduled by (x-chunk parity, ey parity, ez parity), so every write is a
// plain read-modify-write of y (zeroed first).  Warps are independent (no CTA barrier).
#include <cuda_runtime.h>
#include <string.h>
#include "sc_device.cuh"

namespace sc {

struct RWParams {
  Geom g;
  const double* x;
  double* y;
  const double* done;
  BigCoef cf;
  double dinv[64];   // D^{-1}(i,j,k), i fastest (n_I <= 4)
};

template <int NI>
struct RWL {
  static constexpr int N2 = NI * NI;
  static constexpr int XF = 0;                       // x-faces fx = x0 .. x0 + 32
  static constexpr int YF = XF + 33 * N2;            // [jb][32][N2]  (S: fy = ey, N: fy = ey + 1)
  static constexpr int ZF = YF + 2 * 32 * N2;        // [kb][32][N2]  (B, T)
  static constexpr int XE = ZF + 2 * 32 * N2;        // [jb][kb][32][NI]
  static constexpr int YE = XE + 4 * 32 * NI;        // [kb][33][NI]
  static constexpr int ZE = YE + 2 * 33 * NI;        // [jb][33][NI]
  static constexpr int VV = ZE + 2 * 33 * NI;        // [jb][kb][33]
  static constexpr int TOTAL = VV + 4 * 33 + 2;      // per warp (doubles, even)
  static constexpr int WARPS = 4;
};

__device__ __forceinline__ void cp8rw(double* s, const double* g) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ double sgnr(int m) { return (m & 1) ? -1.0 : 1.0; }
__device__ __forceinline__ double eorow(double rp, double rm, int hi) { return hi ? rp - rm : rp + rm; }

// Row [0, cap) of per-entity blocks of `per` doubles: entities [0, n) from global `g` (entity 0
// zero if zlo, entity n-1 zero if zhi, all zero if dir), the rest zero.
// The same range of y (read-modify-written at the end) is prefetched into L2 (one prefetch per
// 64 bytes): the output phase's read-modify-writes are issued one entity group after another (a
// load of y cannot move above an earlier store to y), so each group waits for its loads.
__device__ __forceinline__ void rw_row(double* s, const double* g, int n, int cap, int per, bool dir, bool zlo,
                                       bool zhi, int lane, ptrdiff_t ydelta) {
  const int len = n * per, lo = zlo ? per : 0, hi = zhi ? len - per : len;
  for (int t = lane; t < cap * per; t += 32) {
    if (t < len && !dir && t >= lo && t < hi) {
      cp8rw(s + t, g + t);
#if !(defined(SC_EXP) && SC_EXP == 46)
      if ((t & 7) == 0 || t == lo) asm volatile("prefetch.global.L2 [%0];" ::"l"(g + ydelta + t));
#endif
    } else {
      s[t] = 0.0;
    }
  }
}

template <int NI>
__global__ void __launch_bounds__(128) k_apply_rw(const __grid_constant__ RWParams P, int colour) {
  using L = RWL<NI>;
  constexpr int N2 = L::N2;
  if (P.done != nullptr && *P.done != 0.0) return;
  extern __shared__ double smw[];
  const Geom& g = P.g;
  const BigCoef& cf = P.cf;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int cp = colour & 1, ry = (colour >> 1) & 1, rz = colour >> 2;
  const int nch = (nx + 31) >> 5;
  const int cc = (nch - cp + 1) >> 1, cy = (ny - ry + 1) >> 1, cz = (nz - rz + 1) >> 1;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wid >= (long long)cc * cy * cz) return;   // warp-uniform
  const int lane = threadIdx.x & 31;
  double* const sm = smw + (threadIdx.x >> 5) * L::TOTAL;
  const int chunk = cp + 2 * (int)(wid % cc);
  const int ey = ry + 2 * (int)((wid / cc) % cy), ez = rz + 2 * (int)(wid / ((long long)cc * cy));
  const int x0 = chunk * 32, nel = min(32, nx - x0);
  const long long nx1 = nx + 1, ny1 = ny + 1;
  const bool dY[2] = {ey == 0, ey + 1 == ny}, dZ[2] = {zdir(g, ez), zdir(g, ez + 1)};
  const bool zx0 = x0 == 0, zx1 = x0 + nel == nx;     // x-planes fx = 0 / nx inside this chunk
  // ---- a3: the rows of this chunk (Dirichlet entities as 0)
  const double* X = P.x;
  const ptrdiff_t yd = P.y - P.x;   // y row = x row + yd (same layout)
  rw_row(sm + L::XF, X + g.off_f[0] + (x0 + nx1 * (ey + (long long)ny * ez)) * N2, nel + 1, 33, N2, false, zx0, zx1, lane, yd);
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    rw_row(sm + L::YF + b * 32 * N2, X + g.off_f[1] + (x0 + (long long)nx * (ey + b + ny1 * ez)) * N2, nel, 32, N2,
           dY[b], false, false, lane, yd);
    rw_row(sm + L::ZF + b * 32 * N2, X + g.off_f[2] + (x0 + (long long)nx * (ey + (long long)ny * (ez + b))) * N2, nel,
           32, N2, dZ[b], false, false, lane, yd);
    rw_row(sm + L::YE + b * 33 * NI, X + g.off_e[1] + (x0 + nx1 * (ey + (long long)ny * (ez + b))) * NI, nel + 1, 33, NI,
           dZ[b], zx0, zx1, lane, yd);
    rw_row(sm + L::ZE + b * 33 * NI, X + g.off_e[2] + (x0 + nx1 * (ey + b + ny1 * ez)) * NI, nel + 1, 33, NI, dY[b], zx0,
           zx1, lane, yd);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      rw_row(sm + L::XE + (b + 2 * c) * 32 * NI, X + g.off_e[0] + (x0 + (long long)nx * (ey + b + ny1 * (ez + c))) * NI,
             nel, 32, NI, dY[b] || dZ[c], false, false, lane, yd);
      rw_row(sm + L::VV + (b + 2 * c) * 33, X + g.off_v + x0 + nx1 * (ey + b + ny1 * (ez + c)), nel + 1, 33, 1,
             dY[b] || dZ[c], zx0, zx1, lane, yd);
    }
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  __syncwarp();

  // ---- element of this lane: shell accessors
  const int l = lane;
  const bool act = l < nel, last = act && l == nel - 1;
  const double* Fc[6] = {sm + L::XF + l * N2, sm + L::XF + (l + 1) * N2, sm + L::YF + l * N2,
                         sm + L::YF + (32 + l) * N2, sm + L::ZF + l * N2, sm + L::ZF + (32 + l) * N2};
  // edges: x (jb, kb), y (ib, kb), z (ib, jb); vertices (ib, jb, kb)
  auto XEp = [&](int jb, int kb) { return sm + L::XE + ((jb + 2 * kb) * 32 + l) * NI; };
  auto YEp = [&](int ib, int kb) { return sm + L::YE + (kb * 33 + l + ib) * NI; };
  auto ZEp = [&](int ib, int jb) { return sm + L::ZE + (jb * 33 + l + ib) * NI; };
  auto Vv = [&](int ib, int jb, int kb) { return sm[L::VV + (jb + 2 * kb) * 33 + l + ib]; };

  // ---- a4-a6: condensed part (registers)
  double qf[6][N2];
#pragma unroll
  for (int f = 0; f < 6; ++f)
#pragma unroll
    for (int q = 0; q < N2; ++q) qf[f][q] = 0.0;
  {
    const double *W = Fc[0], *E = Fc[1], *S = Fc[2], *N = Fc[3], *B = Fc[4], *T = Fc[5];
#pragma unroll
    for (int k = 0; k < NI; ++k)
#pragma unroll
      for (int j = 0; j < NI; ++j)
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int ox = j + NI * k, oy = i + NI * k, oz = i + NI * j;
          const double u = fma(cf.c[0][i], fma(sgnr(i), E[ox], W[ox]),
                               fma(cf.c[1][j], fma(sgnr(j), N[oy], S[oy]), cf.c[2][k] * fma(sgnr(k), T[oz], B[oz])));
          const double v = u * P.dinv[i + NI * (j + NI * k)];
          const double vx = cf.c[0][i] * v, vy = cf.c[1][j] * v, vz = cf.c[2][k] * v;
          qf[0][ox] += vx; qf[1][ox] = fma(sgnr(i), vx, qf[1][ox]);
          qf[2][oy] += vy; qf[3][oy] = fma(sgnr(j), vy, qf[3][oy]);
          qf[4][oz] += vz; qf[5][oz] = fma(sgnr(k), vz, qf[5][oz]);
        }
  }
  double* const Y = P.y;
  // Old values of y: within one colour launch every y entry is read and then written once, by
  // the same thread.  They were read through the non-coherent path (ld.global.nc) in round 1;
  // since this kernel writes y, that path is not guaranteed coherent for the kernel's lifetime
  // (ADVICE r1), so they are read with ld.global.cg (L2, coherent).
  auto Yr = [&](long long i) { return __ldcg(Y + i); };   // y is written by this kernel: coherent L2 load
  const long long xf0 = g.off_f[0] + (x0 + l + nx1 * (ey + (long long)ny * ez)) * N2;
  // ---- a7 + a8, faces: out = fd self + k0p opposite + bounding edges - Q
  // face f = 2 d + hi, coordinates (a, b) along (la, lb); bounding edges ea0 / ea1 at index b
  // (sign of a), eb0 / eb1 at index a (sign of b)
  auto face_out = [&](int f, int a, int b) -> double {
    const int d = f >> 1, q = a + NI * b;
    const int la = d == 0 ? 1 : 0, lb = d == 2 ? 1 : 2;
    const double *ea0, *ea1, *eb0, *eb1;
    switch (f) {
      case 0: ea0 = ZEp(0, 0); ea1 = ZEp(0, 1); eb0 = YEp(0, 0); eb1 = YEp(0, 1); break;
      case 1: ea0 = ZEp(1, 0); ea1 = ZEp(1, 1); eb0 = YEp(1, 0); eb1 = YEp(1, 1); break;
      case 2: ea0 = ZEp(0, 0); ea1 = ZEp(1, 0); eb0 = XEp(0, 0); eb1 = XEp(0, 1); break;
      case 3: ea0 = ZEp(0, 1); ea1 = ZEp(1, 1); eb0 = XEp(1, 0); eb1 = XEp(1, 1); break;
      case 4: ea0 = YEp(0, 0); ea1 = YEp(1, 0); eb0 = XEp(0, 0); eb1 = XEp(1, 0); break;
      default: ea0 = YEp(0, 1); ea1 = YEp(1, 1); eb0 = XEp(0, 1); eb1 = XEp(1, 1); break;
    }
    const double fd = cf.F0[d] + cf.L[la][a] + cf.L[lb][b];
    const double ta = cf.e[la][a] * fma(sgnr(a), ea1[b], ea0[b]);
    const double tb = cf.e[lb][b] * fma(sgnr(b), eb1[a], eb0[a]);
    return fma(fd, Fc[f][q], fma(cf.k0p[d], Fc[f ^ 1][q], ta + tb)) - qf[f][q];
  };
  {  // x-faces: face fx = x0 + l gets W of element l and E of element l - 1 (shuffle)
    double ow[N2], oe[N2], old[N2], olde[N2];
#pragma unroll
    for (int b = 0; b < NI; ++b)
#pragma unroll
      for (int a = 0; a < NI; ++a) {
        ow[a + NI * b] = face_out(0, a, b);
        oe[a + NI * b] = face_out(1, a, b);
      }
    const bool dw = (x0 + l == 0), de = (x0 + l + 1 == nx);
#pragma unroll
    for (int q = 0; q < N2; ++q) {
      old[q] = (act && !dw) ? Yr(xf0 + q) : 0.0;
      olde[q] = (last && !de) ? Yr(xf0 + N2 + q) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < N2; ++q) {
      const double em = __shfl_up_sync(0xffffffffu, oe[q], 1);
      if (act && !dw) Y[xf0 + q] = old[q] + ow[q] + (l > 0 ? em : 0.0);
      if (last && !de) Y[xf0 + N2 + q] = olde[q] + oe[q];
    }
  }
  // y- and z-faces: own entities (shared with other rows: colour-scheduled RMW)
#pragma unroll
  for (int f = 2; f < 6; ++f) {
    const int b_ = f & 1;
    const bool dir = f < 4 ? dY[b_] : dZ[b_];
    const long long base = f < 4 ? g.off_f[1] + (x0 + l + (long long)nx * (ey + b_ + ny1 * ez)) * N2
                                 : g.off_f[2] + (x0 + l + (long long)nx * (ey + (long long)ny * (ez + b_))) * N2;
    if (!act || dir) continue;
    double o[N2], old[N2];
#pragma unroll
    for (int b = 0; b < NI; ++b)
#pragma unroll
      for (int a = 0; a < NI; ++a) o[a + NI * b] = face_out(f, a, b);
#pragma unroll
    for (int q = 0; q < N2; ++q) old[q] = Yr(base + q);
#pragma unroll
    for (int q = 0; q < N2; ++q) Y[base + q] = old[q] + o[q];
  }

  // ---- edges and vertices (primary part only).  Line sums (R+, R-) of a face along one
  // coordinate at the other fixed, and of an edge.
  const double K00 = cf.K00, K0p = cf.K0p, w0 = cf.w0, w02 = w0 * w0;
  const double d0 = cf.d[0];
  auto lsum = [&](const double* F, int stride, double& rp, double& rm) {
    rp = 0.0; rm = 0.0;
#pragma unroll
    for (int m = 0; m < NI; ++m) {
      if (m & 1) rm = fma(cf.a0[m], F[m * stride], rm);
      else rp = fma(cf.a0[m], F[m * stride], rp);
    }
  };
  auto row2 = [&](int hi, double u0, double u1) { return hi ? fma(K0p, u0, K00 * u1) : fma(K00, u0, K0p * u1); };
  // x-edges (jb, kb), node i = c: along x the vertices (0|1, jb, kb); boundary y (bit jb): x-edges
  // (0|1, kb), z-face kb summed over j at i = c; boundary z (bit kb): x-edges (jb, 0|1), y-face jb
  // summed over k at i = c.  Own entities.
#pragma unroll
  for (int jb = 0; jb < 2; ++jb)
#pragma unroll
    for (int kb = 0; kb < 2; ++kb) {
      if (!act || dY[jb] || dZ[kb]) continue;
      const long long base = g.off_e[0] + (x0 + l + (long long)nx * (ey + jb + ny1 * (ez + kb))) * NI;
      double o[NI], old[NI];
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        const double u = XEp(jb, kb)[c];
        const double tal = cf.a0[c] * fma(sgnr(c), Vv(1, jb, kb), Vv(0, jb, kb)) + cf.lam[c] * u;
        double p1, m1, p2, m2;
        lsum(Fc[4 + kb] + c, NI, p1, m1);
        lsum(Fc[2 + jb] + c, NI, p2, m2);
        const double t1 = row2(jb, XEp(0, kb)[c], XEp(1, kb)[c]) + eorow(p1, m1, jb);
        const double t2 = row2(kb, XEp(jb, 0)[c], XEp(jb, 1)[c]) + eorow(p2, m2, kb);
        o[c] = w02 * (d0 * u + cf.d[1] * tal) + w0 * (cf.d[2] * t1 + cf.d[3] * t2);
      }
#pragma unroll
      for (int c = 0; c < NI; ++c) old[c] = Yr(base + c);
#pragma unroll
      for (int c = 0; c < NI; ++c) Y[base + c] = old[c] + o[c];
    }
  // y-edges (ib, kb) at fx = x0 + l + ib, node j = c: along y the vertices (ib, 0|1, kb);
  // boundary x (bit ib): y-edges (0|1, kb), z-face kb summed over i at j = c; boundary z (bit kb):
  // y-edges (ib, 0|1), x-face ib summed over k at j = c.  ib = 1 goes to the next lane.
#pragma unroll
  for (int kb = 0; kb < 2; ++kb) {
    double o[2][NI];
#pragma unroll
    for (int ib = 0; ib < 2; ++ib)
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        const double u = YEp(ib, kb)[c];
        const double tal = cf.a0[c] * fma(sgnr(c), Vv(ib, 1, kb), Vv(ib, 0, kb)) + cf.lam[c] * u;
        double p1, m1, p2, m2;
        lsum(Fc[4 + kb] + NI * c, 1, p1, m1);
        lsum(Fc[ib] + c, NI, p2, m2);
        const double t1 = row2(ib, YEp(0, kb)[c], YEp(1, kb)[c]) + eorow(p1, m1, ib);
        const double t2 = row2(kb, YEp(ib, 0)[c], YEp(ib, 1)[c]) + eorow(p2, m2, kb);
        o[ib][c] = w02 * (d0 * u + cf.d[2] * tal) + w0 * (cf.d[1] * t1 + cf.d[3] * t2);
      }
    const long long base = g.off_e[1] + (x0 + l + nx1 * (ey + (long long)ny * (ez + kb))) * NI;
    const bool d0x = x0 + l == 0 || dZ[kb], d1x = x0 + l + 1 == nx || dZ[kb];
    double old[NI], old1[NI];
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      old[c] = (act && !d0x) ? Yr(base + c) : 0.0;
      old1[c] = (last && !d1x) ? Yr(base + NI + c) : 0.0;
    }
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      const double m = __shfl_up_sync(0xffffffffu, o[1][c], 1);
      if (act && !d0x) Y[base + c] = old[c] + o[0][c] + (l > 0 ? m : 0.0);
      if (last && !d1x) Y[base + NI + c] = old1[c] + o[1][c];
    }
  }
  // z-edges (ib, jb) at fx = x0 + l + ib, node k = c: along z the vertices (ib, jb, 0|1);
  // boundary x (bit ib): z-edges (0|1, jb), y-face jb summed over i at k = c; boundary y (bit jb):
  // z-edges (ib, 0|1), x-face ib summed over j at k = c.
#pragma unroll
  for (int jb = 0; jb < 2; ++jb) {
    double o[2][NI];
#pragma unroll
    for (int ib = 0; ib < 2; ++ib)
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        const double u = ZEp(ib, jb)[c];
        const double tal = cf.a0[c] * fma(sgnr(c), Vv(ib, jb, 1), Vv(ib, jb, 0)) + cf.lam[c] * u;
        double p1, m1, p2, m2;
        lsum(Fc[2 + jb] + NI * c, 1, p1, m1);
        lsum(Fc[ib] + NI * c, 1, p2, m2);
        const double t1 = row2(ib, ZEp(0, jb)[c], ZEp(1, jb)[c]) + eorow(p1, m1, ib);
        const double t2 = row2(jb, ZEp(ib, 0)[c], ZEp(ib, 1)[c]) + eorow(p2, m2, jb);
        o[ib][c] = w02 * (d0 * u + cf.d[3] * tal) + w0 * (cf.d[1] * t1 + cf.d[2] * t2);
      }
    const long long base = g.off_e[2] + (x0 + l + nx1 * (ey + jb + ny1 * ez)) * NI;
    const bool d0x = x0 + l == 0 || dY[jb], d1x = x0 + l + 1 == nx || dY[jb];
    double old[NI], old1[NI];
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      old[c] = (act && !d0x) ? Yr(base + c) : 0.0;
      old1[c] = (last && !d1x) ? Yr(base + NI + c) : 0.0;
    }
#pragma unroll
    for (int c = 0; c < NI; ++c) {
      const double m = __shfl_up_sync(0xffffffffu, o[1][c], 1);
      if (act && !d0x) Y[base + c] = old[c] + o[0][c] + (l > 0 ? m : 0.0);
      if (last && !d1x) Y[base + NI + c] = old1[c] + o[1][c];
    }
  }
  // vertices (ib, jb, kb) at fx = x0 + l + ib: along each direction the partner vertex and the
  // edge through the vertex (line sum of Ktilde row 0 / p)
#pragma unroll
  for (int jb = 0; jb < 2; ++jb)
#pragma unroll
    for (int kb = 0; kb < 2; ++kb) {
      double o[2];
#pragma unroll
      for (int ib = 0; ib < 2; ++ib) {
        double px, mx, py, my, pz, mz;
        lsum(XEp(jb, kb), 1, px, mx);
        lsum(YEp(ib, kb), 1, py, my);
        lsum(ZEp(ib, jb), 1, pz, mz);
        const double tx = row2(ib, Vv(0, jb, kb), Vv(1, jb, kb)) + eorow(px, mx, ib);
        const double ty = row2(jb, Vv(ib, 0, kb), Vv(ib, 1, kb)) + eorow(py, my, jb);
        const double tz = row2(kb, Vv(ib, jb, 0), Vv(ib, jb, 1)) + eorow(pz, mz, kb);
        o[ib] = w02 * (w0 * d0 * Vv(ib, jb, kb) + cf.d[1] * tx + cf.d[2] * ty + cf.d[3] * tz);
      }
      const long long base = g.off_v + x0 + l + nx1 * (ey + jb + ny1 * (ez + kb));
      const bool dyz = dY[jb] || dZ[kb];
      const bool d0x = x0 + l == 0 || dyz, d1x = x0 + l + 1 == nx || dyz;
      const double old = (act && !d0x) ? Yr(base) : 0.0, old1 = (last && !d1x) ? Yr(base + 1) : 0.0;
      const double m = __shfl_up_sync(0xffffffffu, o[1], 1);
      if (act && !d0x) Y[base] = old + o[0] + (l > 0 ? m : 0.0);
      if (last && !d1x) Y[base + 1] = old1 + o[1];
    }
}

template <int NI>
static int launch_rw_t(const RWParams& P, cudaStream_t st, int* nl) {
  using L = RWL<NI>;
  const size_t smem = sizeof(double) * L::TOTAL * L::WARPS;
  static bool attr[kMaxDev];   // per device
  const int dv = dev_slot();
  if (!attr[dv]) {
    cudaFuncSetAttribute(k_apply_rw<NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[dv] = true;
  }
  const int nch = (P.g.nx + 31) >> 5;
  for (int c = 0; c < 8; ++c) {
    const int cp = c & 1, ry = (c >> 1) & 1, rz = c >> 2;
    const long long warps = (long long)((nch - cp + 1) >> 1) * ((P.g.ny - ry + 1) >> 1) * ((P.g.nz - rz + 1) >> 1);
    if (warps <= 0) continue;
    k_apply_rw<NI><<<(unsigned)((warps + L::WARPS - 1) / L::WARPS), 32 * L::WARPS, smem, st>>>(P, c);
    (*nl)++;
  }
  return cudaGetLastError();
}

bool rw_supported(int ni) { return ni == 2 || ni == 3; }

int launch_apply_rw(const Geom& g, const double* x, double* y, const double* done, const void* coef, void* stream,
                    int* nl, void* events) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  cudaError_t err = cudaMemsetAsync(y, 0, sizeof(double) * g.n_total, st);
  if (err != cudaSuccess) return err;
  if (ev) cudaEventRecord(ev[0], st);
  RWParams P;
  P.g = g; P.x = x; P.y = y; P.done = done;
  memcpy(&P.cf, coef, sizeof(BigCoef));
  const int ni = g.ni;
  for (int k = 0; k < ni; ++k)
    for (int j = 0; j < ni; ++j)
      for (int i = 0; i < ni; ++i)
        P.dinv[i + ni * (j + ni * k)] = 1.0 / (P.cf.d[0] + P.cf.dl[0][i] + P.cf.dl[1][j] + P.cf.dl[2][k]);
  int rc = cudaErrorInvalidValue;
  if (ni == 2) rc = launch_rw_t<2>(P, st, nl);
  else if (ni == 3) rc = launch_rw_t<3>(P, st, nl);
  if (ev) cudaEventRecord(ev[1], st);
  return rc;
}

}  // namespace sc
