// Condensed operator v3 (rows a3-a8 of SURVEY §8(a)): tile-column kernel, parity-class warps.
//
// Work decomposition.  The slab's elements are cut into xy-tiles of TX x TY = 8 x 4 elements;
// a work item is one tile-column (all nz element layers of the tile).  A persistent CTA (one
// per SM, 8 warps) takes items in ticket order and marches up the column one element layer at
// a time.  Every entity of the skeleton is assembled on chip except those on tile side
// boundaries, which are finished with a decoupled look-back: the lower-ticket contributor
// stores its partial sum straight into y (or, on the 4-tile corner lines, into a small corner
// record), publishes a per-(item, layer) flag, and the owner (highest-ticket contributor) adds
// it and writes the final value one step later.  Every skeleton entry is written exactly once
// (no memset, no atomics) and read from HBM once.
//
// Condensed part (faces-in, D^{-1}, faces-out; §6 Table 2) in the even/odd
// form: with ap = sigma .* a0 (sigma_m = (-1)^m, the parity of the m-th M-orthonormal
// eigenvector, R2),
//     u(i,j,k) = c1_i Px^{s_i}(j,k) + c2_j Py^{s_j}(i,k) + c3_k Pz^{s_k}(i,j),
//     Px^{s} = W + (-1)^s E,  Py^{s} = S + (-1)^s N,  Pz^{s} = B + (-1)^s T,  c_d = d_d a0,
//     v = u D^{-1},  Qx^{s}(j,k) = sum_{i of parity s} c1_i v,  W -= Qx^0 + Qx^1, E -= Qx^0 - Qx^1
// (and likewise in y and z): 7 FP64 instructions per interior point instead of 13, same result.
// The interior points of an element split into 8 parity classes (s_i, s_j, s_k); warp w of the
// CTA owns one class for all 32 elements of the tile (lane = element).  Every faces-out sum of
// a class then stays in one thread's registers, and every coefficient (c_d, D^{-1}) is warp-
// uniform and compile-time indexed, so it is read straight from the kernel-parameter constant
// bank.  The two parity classes of a direction add into the assembled face buffers in two
// barrier-separated rounds; the two elements of an x- (y-) face are summed with a lane shuffle.
// The primary part (Htilde_BB, Eq. 26 generalised) is applied entity-centrically.
#include <cuda_runtime.h>
#include <string.h>
#include "sc_device.cuh"

namespace sc {

// Launch-persistent device state: the ticket counter and the finished-CTA counter reset
// themselves at the end of every launch (last CTA out), and the epoch (flag value) is
// advanced there, so launches can be replayed from a CUDA graph.
struct ColState {
  unsigned long long ticket;
  unsigned int finished;
  int epoch;
};

// Uniform-geometry coefficients, passed by value and copied to shared memory per CTA.
struct ColCoef {
  double c[3][8];          // c[d][m] = d_{d+1} a0_m                       (condensed part)
  double e[3][8];          // e[d][m] = d_{d+1} w0 a0_m                    (face-edge coupling)
  double a[8];             // a0_m                                         (face line sums)
  double fd[3][64];        // face self terms: fd[0](j,k) = d0 w0 + d1 K00 + d2 w0 Lam_j + d3 w0 Lam_k,
                           //   fd[1](i,k), fd[2](i,j) likewise (first index fastest)
  double k0p[3];           // d_{d+1} K0p                                  (opposite-face coupling)
  double dinv[512];        // D^{-1}(i,j,k) = 1 / (d0 + d1 Lam_i + d2 Lam_j + d3 Lam_k), i fastest
};

struct ColParams {
  Geom g;
  const double* x;
  double* y;
  const double* done;
  ColState* st;
  int* flags;            // [nitems][nz+1]
  double* corner;        // [(nty+1)][(ntx+1)][nz+1][3][NI+1]
  double* pending;       // [nitems][2][PEND]
  int ntx, nty, nitems;
  ColCoef cf;
};

template <int NI>
struct CS {
  static constexpr int N2 = NI * NI;
  static constexpr int NT = 256;                      // 8 warps = 8 parity classes
  static constexpr int TX = 8, TY = 4, NE = TX * TY;  // one element per lane
  static constexpr int XF = TY * (TX + 1) * N2;
  static constexpr int YF = (TY + 1) * TX * N2;
  static constexpr int ZE = (TY + 1) * (TX + 1) * NI;
  static constexpr int SIDE = XF + YF + ZE;
  static constexpr int PZF = TY * TX * N2;
  static constexpr int PXE = (TY + 1) * TX * NI;
  static constexpr int PYE = TY * (TX + 1) * NI;
  static constexpr int PVV = (TY + 1) * (TX + 1);
  static constexpr int PLANE = PZF + PXE + PYE + PVV;
  // even/odd line reductions of the faces and edges (primary part of the edges / vertices)
  static constexpr int R_XJ = 0;                                   // x-faces over j: [TY][TX+1][2][NI]
  static constexpr int R_XK = R_XJ + TY * (TX + 1) * 2 * NI;       // x-faces over k
  static constexpr int R_YI = R_XK + TY * (TX + 1) * 2 * NI;       // y-faces over i: [TY+1][TX][2][NI]
  static constexpr int R_YK = R_YI + (TY + 1) * TX * 2 * NI;       // y-faces over k
  static constexpr int R_ZI = R_YK + (TY + 1) * TX * 2 * NI;       // z-faces over i: [2][TY][TX][2][NI]
  static constexpr int R_ZJ = R_ZI + 2 * TY * TX * 2 * NI;         // z-faces over j
  static constexpr int R_ZE = R_ZJ + 2 * TY * TX * 2 * NI;         // z-edges: [TY+1][TX+1][2]
  static constexpr int R_XE = R_ZE + (TY + 1) * (TX + 1) * 2;      // x-edges: [2][TY+1][TX][2]
  static constexpr int R_YE = R_XE + 2 * (TY + 1) * TX * 2;        // y-edges: [2][TY][TX+1][2]
  static constexpr int RED = R_YE + 2 * TY * (TX + 1) * 2;
  static constexpr int O_IS = 0;                     // 2 side input buffers
  static constexpr int O_IP = O_IS + 2 * SIDE;       // 2 plane input buffers
  static constexpr int O_AS = O_IP + 2 * PLANE;      // side accumulator
  static constexpr int O_AP = O_AS + SIDE;           // 2 plane accumulators
  static constexpr int O_RQ = O_AP + 2 * PLANE;      // reduction buffers
  static constexpr int O_TAB = O_RQ + RED;           // a0, lam (2 x 32)
  static constexpr int O_CF = O_TAB + 2 * 32;        // ColCoef copy
  static constexpr int TOTAL = O_CF + (int)(sizeof(ColCoef) / sizeof(double));
  // parked own partials of the W / S boundary entities (global, per tile, 2 step slots)
  static constexpr int PD_XF = 0;                                  // W column x-faces  [TY][N2]
  static constexpr int PD_YF = PD_XF + TY * N2;                    // S row y-faces     [TX N2]
  static constexpr int PD_XE = PD_YF + TX * N2;                    // S row x-edges     [TX NI]
  static constexpr int PD_YE = PD_XE + TX * NI;                    // W column y-edges  [TY][NI]
  static constexpr int PD_ZEW = PD_YE + TY * NI;                   // W column z-edges  [TY+1][NI]
  static constexpr int PD_ZES = PD_ZEW + (TY + 1) * NI;            // S row z-edges     [TX NI]
  static constexpr int PD_VW = PD_ZES + TX * NI;                   // W column vertices [TY+1]
  static constexpr int PD_VS = PD_VW + TY + 1;                     // S row vertices    [TX]
  static constexpr int PEND = PD_VS + TX;
  // sub-array offsets inside a side / plane block
  static constexpr int S_XF = 0, S_YF = XF, S_ZE = XF + YF;
  static constexpr int P_ZF = 0, P_XE = PZF, P_YE = PZF + PXE, P_VV = PZF + PXE + PYE;
};

// ---- shared-memory views --------------------------------------------------------------
template <int NI>
struct Side {
  double* b;
  __device__ double* xf(int iy, int ix) const { return b + CS<NI>::S_XF + (iy * (CS<NI>::TX + 1) + ix) * CS<NI>::N2; }
  __device__ double* yf(int iy, int ix) const { return b + CS<NI>::S_YF + (iy * CS<NI>::TX + ix) * CS<NI>::N2; }
  __device__ double* ze(int iy, int ix) const { return b + CS<NI>::S_ZE + (iy * (CS<NI>::TX + 1) + ix) * NI; }
};
template <int NI>
struct Plane {
  double* b;
  __device__ double* zf(int iy, int ix) const { return b + CS<NI>::P_ZF + (iy * CS<NI>::TX + ix) * CS<NI>::N2; }
  __device__ double* xe(int iy, int ix) const { return b + CS<NI>::P_XE + (iy * CS<NI>::TX + ix) * NI; }
  __device__ double* ye(int iy, int ix) const { return b + CS<NI>::P_YE + (iy * (CS<NI>::TX + 1) + ix) * NI; }
  __device__ double* vv(int iy, int ix) const { return b + CS<NI>::P_VV + iy * (CS<NI>::TX + 1) + ix; }
};

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

#if defined(SC_EXP) && SC_EXP == 9
__device__ unsigned long long g_phase_cycles[16];
#define SC_PHASE(k)                                                     \
  do {                                                                  \
    if (threadIdx.x == 0) {                                             \
      long long t_ = clock64();                                         \
      atomicAdd(&g_phase_cycles[k], (unsigned long long)(t_ - ph_t0));  \
      ph_t0 = t_;                                                       \
    }                                                                   \
  } while (0)
#else
#define SC_PHASE(k) do {} while (0)
#endif

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void flag_release(int* f, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}
__device__ __forceinline__ int flag_acquire(const int* f) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}

// ---- global addressing of the slab's entities ------------------------------------------
struct Addr {
  const Geom& g;
  __device__ long long xf(int fx, int ey, int ez) const {
    return g.off_f[0] + (fx + (long long)(g.nx + 1) * (ey + (long long)g.ny * ez)) * (long long)(g.ni * g.ni);
  }
  __device__ long long yf(int ex, int fy, int ez) const {
    return g.off_f[1] + (ex + (long long)g.nx * (fy + (long long)(g.ny + 1) * ez)) * (long long)(g.ni * g.ni);
  }
  __device__ long long zf(int ex, int ey, int fz) const {
    return g.off_f[2] + (ex + (long long)g.nx * (ey + (long long)g.ny * fz)) * (long long)(g.ni * g.ni);
  }
  __device__ long long xe(int ex, int fy, int fz) const {
    return g.off_e[0] + (ex + (long long)g.nx * (fy + (long long)(g.ny + 1) * fz)) * g.ni;
  }
  __device__ long long ye(int fx, int ey, int fz) const {
    return g.off_e[1] + (fx + (long long)(g.nx + 1) * (ey + (long long)g.ny * fz)) * g.ni;
  }
  __device__ long long ze(int fx, int fy, int ez) const {
    return g.off_e[2] + (fx + (long long)(g.nx + 1) * (fy + (long long)(g.ny + 1) * ez)) * g.ni;
  }
  __device__ long long vv(int fx, int fy, int fz) const {
    return g.off_v + fx + (long long)(g.nx + 1) * (fy + (long long)(g.ny + 1) * fz);
  }
};

// Row-contiguous async loads of one z-plane (fz) / one element layer (ez) of the tile into
// shared memory.  Every tile row of an entity class is one contiguous range in both the
// skeleton vector and the smem buffer; a warp copies a row with 8-byte cp.async (Dirichlet
// entities, which sit at the two ends of a row or fill a whole row, are written as 0).
template <int NI>
__device__ void load_plane(const ColParams& P, Plane<NI> pl, int x0, int y0, int tw, int th, int fz) {
#if defined(SC_EXP) && SC_EXP == 5
  return;
#endif
  using C = CS<NI>;
  constexpr int N2 = C::N2, NW = C::NT / 32;
  const Geom& g = P.g;
  Addr A{g};
  const bool zd = zdir(g, fz);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int x1 = x0 + tw;
  for (int row = warp; row < th; row += NW) {                      // z-faces
    double* sb = pl.zf(row, 0);
    const double* gb = P.x + A.zf(x0, y0 + row, fz);
    for (int t = lane; t < tw * N2; t += 32) {
      if (zd) sb[t] = 0.0; else cp_async8(sb + t, gb + t);
    }
  }
  for (int row = warp; row <= th; row += NW) {                     // x-edges (ex, fy)
    const int fy = y0 + row;
    const bool rd = zd || fy == 0 || fy == g.ny;
    double* sb = pl.xe(row, 0);
    const double* gb = P.x + A.xe(x0, fy, fz);
    for (int t = lane; t < tw * NI; t += 32) {
      if (rd) sb[t] = 0.0; else cp_async8(sb + t, gb + t);
    }
  }
  for (int row = warp; row < th; row += NW) {                      // y-edges (fx, ey)
    double* sb = pl.ye(row, 0);
    const double* gb = P.x + A.ye(x0, y0 + row, fz);
    const int zlo = (x0 == 0) ? NI : 0, zhi = (x1 == g.nx) ? tw * NI : (tw + 1) * NI;
    for (int t = lane; t < (tw + 1) * NI; t += 32) {
      if (zd || t < zlo || t >= zhi) sb[t] = 0.0; else cp_async8(sb + t, gb + t);
    }
  }
  for (int row = warp; row <= th; row += NW) {                     // vertices (fx, fy)
    const int fy = y0 + row;
    const bool rd = zd || fy == 0 || fy == g.ny;
    double* sb = pl.vv(row, 0);
    const double* gb = P.x + A.vv(x0, fy, fz);
    for (int t = lane; t <= tw; t += 32) {
      if (rd || (t == 0 && x0 == 0) || (t == tw && x1 == g.nx)) sb[t] = 0.0; else cp_async8(sb + t, gb + t);
    }
  }
}

template <int NI>
__device__ void load_side(const ColParams& P, Side<NI> sd, int x0, int y0, int tw, int th, int ez) {
#if defined(SC_EXP) && SC_EXP == 5
  return;
#endif
  using C = CS<NI>;
  constexpr int N2 = C::N2, NW = C::NT / 32;
  const Geom& g = P.g;
  Addr A{g};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int x1 = x0 + tw;
  for (int row = warp; row < th; row += NW) {                      // x-faces (fx, ey)
    double* sb = sd.xf(row, 0);
    const double* gb = P.x + A.xf(x0, y0 + row, ez);
    const int zlo = (x0 == 0) ? N2 : 0, zhi = (x1 == g.nx) ? tw * N2 : (tw + 1) * N2;
    for (int t = lane; t < (tw + 1) * N2; t += 32) {
      if (t < zlo || t >= zhi) sb[t] = 0.0; else cp_async8(sb + t, gb + t);
    }
  }
  for (int row = warp; row <= th; row += NW) {                     // y-faces (ex, fy)
    const int fy = y0 + row;
    const bool rd = fy == 0 || fy == g.ny;
    double* sb = sd.yf(row, 0);
    const double* gb = P.x + A.yf(x0, fy, ez);
    for (int t = lane; t < tw * N2; t += 32) {
      if (rd) sb[t] = 0.0; else cp_async8(sb + t, gb + t);
    }
  }
  for (int row = warp; row <= th; row += NW) {                     // z-edges (fx, fy)
    const int fy = y0 + row;
    const bool rd = fy == 0 || fy == g.ny;
    double* sb = sd.ze(row, 0);
    const double* gb = P.x + A.ze(x0, fy, ez);
    const int zlo = (x0 == 0) ? NI : 0, zhi = (x1 == g.nx) ? tw * NI : (tw + 1) * NI;
    for (int t = lane; t < (tw + 1) * NI; t += 32) {
      if (rd || t < zlo || t >= zhi) sb[t] = 0.0; else cp_async8(sb + t, gb + t);
    }
  }
}

// Corner record address: corner point (cx, cy) of the tile grid, step l, slot (0 SW, 1 S, 2 W).
__device__ __forceinline__ double* corner_rec(const ColParams& P, int cx, int cy, int l, int slot) {
  const int ni = P.g.ni;
  return P.corner + ((((long long)cy * (P.ntx + 1) + cx) * (P.g.nz + 1) + l) * 3 + slot) * (ni + 1);
}

// Even/odd partial sums of a0-weighted lines: returns (R+, R-) with
// R+ = sum_{a even} a0_a f[a*stride], R- = sum_{a odd} a0_a f[a*stride].
// Row 0 of Ktilde applied to the interior of a line is R+ + R-, row p is R+ - R-.
template <int NI>
__device__ __forceinline__ void eo_reduce(const double* f, int stride, const double* a0, double* out) {
  double rp = 0.0, rm = 0.0;
#pragma unroll
  for (int a = 0; a < NI; ++a) {
    if (a & 1) rm += a0[a] * f[a * stride];
    else rp += a0[a] * f[a * stride];
  }
  out[0] = rp;
  out[1] = rm;
}

// Row-0 / row-p application from an (R+, R-) pair: hi = 0 -> R+ + R-, hi = 1 -> R+ - R-.
__device__ __forceinline__ double eo_row(const double* r, int hi) { return hi ? r[0] - r[1] : r[0] + r[1]; }

// Deferred look-back for step ls of tile item: wait for the W, S, SW tiles' flags of step ls,
// then write the tile's W / S boundary entities of that step as own (parked) partial + the
// neighbours' partials (y-in-place, or the corner records on the 4-tile corner line).
// All entries of a step form one flat list; every thread first issues all of its loads
// (one L2 round trip per step), then all of its stores.  Dirichlet entities were already
// written as 0 and are skipped.
template <int NI>
__device__ void finish_boundary(const ColParams& P, long long item, int ls, int x0, int y0, int tw, int th,
                                const int* flag_w, const int* flag_s, const int* flag_sw, int epoch) {
  using C = CS<NI>;
  constexpr int N2 = C::N2, NT = C::NT, TX = C::TX, TY = C::TY;
  constexpr int MAXE = (C::PEND + NT - 1) / NT;
  const Geom& g = P.g;
  Addr A{g};
  const int tid = threadIdx.x;
  const bool last = (ls == g.nz), pzd = zdir(g, ls);
  const int x1 = x0 + tw, y1 = y0 + th;
  const bool hasE = x1 < g.nx, hasN = y1 < g.ny, hasW = x0 > 0, hasS = y0 > 0;
  if (!hasW && !hasS) return;
#if !defined(SC_EXP) || SC_EXP != 8
  if (tid == 0) {
    if (flag_w) while (flag_acquire(flag_w + ls) != epoch) __nanosleep(32);
    if (flag_s) while (flag_acquire(flag_s + ls) != epoch) __nanosleep(32);
    if (flag_sw) while (flag_acquire(flag_sw + ls) != epoch) __nanosleep(32);
  }
  __syncthreads();
#endif
  const double* pd = P.pending + (item * 2 + (ls & 1)) * (long long)C::PEND;
  // segment sizes of the flat list (0 when the segment does not apply at this step)
  const int n0 = (!last && hasW) ? th * N2 : 0;            // W col x-faces
  const int n1 = (!last && hasS) ? tw * N2 : 0;            // S row y-faces
  const int n2 = (!last && hasW) ? (th + 1) * NI : 0;      // W col z-edges
  const int n3 = (!last && hasS) ? (tw - 1) * NI : 0;      // S row z-edges, ix in [1, tw-1]
  const int n4 = (!pzd && hasS) ? tw * NI : 0;             // S row x-edges
  const int n5 = (!pzd && hasW) ? th * NI : 0;             // W col y-edges
  const int n6 = (!pzd && hasW) ? th + 1 : 0;              // W col vertices
  const int n7 = (!pzd && hasS) ? tw - 1 : 0;              // S row vertices, ix in [1, tw-1]
  const int ntot = n0 + n1 + n2 + n3 + n4 + n5 + n6 + n7;
  double val[MAXE];
  double* dst[MAXE];
#pragma unroll
  for (int k = 0; k < MAXE; ++k) {
    dst[k] = nullptr;
    val[k] = 0.0;
    int t = tid + k * NT;
    if (t >= ntot) continue;
    double* d = nullptr;
    int po = -1;                 // offset of the own parked partial
    int corner = -1;             // corner line entry: value index into the corner records
    if (t < n0) {
      d = P.y + A.xf(x0, y0 + t / N2, ls) + t % N2; po = C::PD_XF + t;
    } else if ((t -= n0) < n1) {
      d = P.y + A.yf(x0, y0, ls) + t; po = C::PD_YF + t;
    } else if ((t -= n1) < n2) {
      const int row = t / NI, c = t % NI, fy = y0 + row;
      if (fy == 0 || fy == g.ny || (row == th && hasN)) continue;
      d = P.y + A.ze(x0, fy, ls) + c; po = C::PD_ZEW + t;
      if (row == 0 && hasS) corner = c;
    } else if ((t -= n2) < n3) {
      d = P.y + A.ze(x0, y0, ls) + NI + t; po = C::PD_ZES + t;
    } else if ((t -= n3) < n4) {
      d = P.y + A.xe(x0, y0, ls) + t; po = C::PD_XE + t;
    } else if ((t -= n4) < n5) {
      d = P.y + A.ye(x0, y0 + t / NI, ls) + t % NI; po = C::PD_YE + t;
    } else if ((t -= n5) < n6) {
      const int fy = y0 + t;
      if (fy == 0 || fy == g.ny || (t == th && hasN)) continue;
      d = P.y + A.vv(x0, fy, ls); po = C::PD_VW + t;
      if (t == 0 && hasS) corner = NI;
    } else {
      t -= n6;
      d = P.y + A.vv(x0, y0, ls) + 1 + t; po = C::PD_VS + t;
    }
    double v = ld_cg(pd + po);
    if (corner >= 0) {
      const int cx = x0 / TX, cy = y0 / TY;
      v += ld_cg(corner_rec(P, cx, cy, ls, 0) + corner) + ld_cg(corner_rec(P, cx, cy, ls, 1) + corner) +
           ld_cg(corner_rec(P, cx, cy, ls, 2) + corner);
    } else {
      v += ld_cg(d);
    }
    val[k] = v;
    dst[k] = d;
  }
#pragma unroll
  for (int k = 0; k < MAXE; ++k)
    if (dst[k]) *dst[k] = val[k];
}


// ---- condensed part of one parity class (s_i, s_j, s_k) = (SI, SJ, SK) ---------------------
// Lane = element (ix, iy) of the tile.  All loops are unrolled with compile-time indices, so
// P.cf.* are constant-bank operands.  Outputs: round r of direction d is executed by the
// classes with s_d == r; round 0 initialises ac.xf / ac.yf / actp.zf, round 1 adds.
__device__ __forceinline__ void bar_named(int id) { asm volatile("bar.sync %0, 256;" ::"r"(id) : "memory"); }

// All eight classes run the same code (class parities are warp-uniform runtime values): a
// class-specialised, fully unrolled variant per warp does not fit the instruction cache.
// Face entry (a, b) of the class sits at base + 2 aa + 2 NI bb (a = s_a + 2 aa, b = s_b + 2 bb),
// so every shared-memory access below has a compile-time offset from a per-thread base.
template <int NI>
__device__ __forceinline__ void vol_class(const int cls, const ColCoef* cf, const Side<NI>& in, const Plane<NI>& inb,
                                          const Plane<NI>& intp, const Side<NI>& ac, const Plane<NI>& acb,
                                          const Plane<NI>& actp, double* rq, int ix, int iy, int tw, int th) {
  constexpr int M = (NI + 1) / 2, N2 = NI * NI, TX = CS<NI>::TX;
  constexpr int DO = NI >= 2 ? 1 : 0;   // parity class that adds the primary part and line sums
  const int si = cls >> 2, sj = (cls >> 1) & 1, sk = cls & 1;
  const int CI = (NI - si + 1) >> 1, CJ = (NI - sj + 1) >> 1, CK = (NI - sk + 1) >> 1;
  const double gi = si ? -1.0 : 1.0, gj = sj ? -1.0 : 1.0, gk = sk ? -1.0 : 1.0;
  const bool act = ix < tw && iy < th;
  const bool lastx = ix == tw - 1, lasty = iy == th - 1;
  const double* W = in.xf(iy, ix) + sj + NI * sk;
  const double* E = W + N2;
  const double* S = in.yf(iy, ix) + si + NI * sk;
  const double* N = S + TX * N2;
  const double* B = inb.zf(iy, ix) + si + NI * sj;
  const double* T = intp.zf(iy, ix) + si + NI * sj;
  double* const fX = ac.xf(iy, ix) + sj + NI * sk;
  double* const fY = ac.yf(iy, ix) + si + NI * sk;
  double* const fB = acb.zf(iy, ix) + si + NI * sj;
  double* const fT = actp.zf(iy, ix) + si + NI * sj;

  // ---- phase A: primary part of the faces (Eq. 26 generalised: self, opposite face, the four
  // bounding edges) and the parity component of the faces' a0-weighted line sums used by the
  // edge / vertex rows, by the class with s_d == DO of each direction d.  Initialises ac.xf,
  // ac.yf and actp.zf (plain stores), adds into acb.zf.
  if (si == DO) {   // x-faces: face ix = W of element ix, E of element ix-1
    const double* Z0 = in.ze(iy, ix) + sk;
    const double* Z1 = in.ze(iy + 1, ix) + sk;
    const double* Yb = inb.ye(iy, ix) + sj;
    const double* Yt = intp.ye(iy, ix) + sj;
    const double* fd = cf->fd[0] + sj + NI * sk;
    double* oj = rq + CS<NI>::R_XJ + (iy * (TX + 1) + ix) * 2 * NI + 2 * sk + sj;   // over j, keep k
    double* ok = rq + CS<NI>::R_XK + (iy * (TX + 1) + ix) * 2 * NI + 2 * sj + sk;   // over k, keep j
#pragma unroll
    for (int kk = 0; kk < M; ++kk) {
      if (kk >= CK) continue;
      const double zw = fma(gj, Z1[2 * kk], Z0[2 * kk]), ze = fma(gj, Z1[NI + 2 * kk], Z0[NI + 2 * kk]);
      const double ek = cf->e[2][sk + 2 * kk], ak = cf->a[sk + 2 * kk];
      double rwj = 0.0, rej = 0.0;
#pragma unroll
      for (int jj = 0; jj < M; ++jj) {
        if (jj >= CJ) continue;
        const int o = 2 * jj + 2 * NI * kk;
        const double w = W[o], e = E[o], f = fd[o], ej = cf->e[1][sj + 2 * jj], aj = cf->a[sj + 2 * jj];
        const double yw = fma(gk, Yt[2 * jj], Yb[2 * jj]), ye = fma(gk, Yt[NI + 2 * jj], Yb[NI + 2 * jj]);
        const double Wp = fma(f, w, fma(cf->k0p[0], e, fma(ej, zw, ek * yw)));
        const double Ep = fma(f, e, fma(cf->k0p[0], w, fma(ej, ze, ek * ye)));
        rwj = fma(aj, w, rwj);
        rej = fma(aj, e, rej);
        const double Em = __shfl_up_sync(0xffffffffu, Ep, 1);
        if (act) {
          fX[o] = ix > 0 ? Wp + Em : Wp;
          if (lastx) fX[o + N2] = Ep;
          if (kk == 0) {   // over k, keep j: one pass per j
            double rwk = 0.0, rek = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < M; ++k2)
              if (k2 < CK) {
                rwk = fma(cf->a[sk + 2 * k2], W[2 * jj + 2 * NI * k2], rwk);
                rek = fma(cf->a[sk + 2 * k2], E[2 * jj + 2 * NI * k2], rek);
              }
            ok[4 * jj] = rwk;
            if (lastx) ok[2 * NI + 4 * jj] = rek;
          }
        }
      }
      if (act) {
        oj[4 * kk] = rwj;
        if (lastx) oj[2 * NI + 4 * kk] = rej;
        if (NI == 1) {   // no odd interior index: the odd parity components are 0
          oj[1] = ok[1] = 0.0;
          if (lastx) oj[2 * NI + 1] = ok[2 * NI + 1] = 0.0;
        }
      }
      (void)ak;
    }
  }
  if (sj == DO) {   // y-faces: face row iy = S of element row iy, N of row iy-1
    const double* Z0 = in.ze(iy, ix) + sk;
    const double* Z1 = in.ze(iy + 1, ix) + sk;
    const double* Xb = inb.xe(iy, ix) + si;
    const double* Xt = intp.xe(iy, ix) + si;
    const double* fd = cf->fd[1] + si + NI * sk;
    double* oi = rq + CS<NI>::R_YI + (iy * TX + ix) * 2 * NI + 2 * sk + si;   // over i, keep k
    double* ok = rq + CS<NI>::R_YK + (iy * TX + ix) * 2 * NI + 2 * si + sk;   // over k, keep i
#pragma unroll
    for (int kk = 0; kk < M; ++kk) {
      if (kk >= CK) continue;
      const double zs = fma(gi, Z0[NI + 2 * kk], Z0[2 * kk]), zn = fma(gi, Z1[NI + 2 * kk], Z1[2 * kk]);
      const double ek = cf->e[2][sk + 2 * kk];
      double rsi = 0.0, rni = 0.0;
#pragma unroll
      for (int ii = 0; ii < M; ++ii) {
        if (ii >= CI) continue;
        const int o = 2 * ii + 2 * NI * kk;
        const double sv = S[o], nv = N[o], f = fd[o], ei_ = cf->e[0][si + 2 * ii], ai = cf->a[si + 2 * ii];
        const double xs = fma(gk, Xt[2 * ii], Xb[2 * ii]), xn = fma(gk, Xt[TX * NI + 2 * ii], Xb[TX * NI + 2 * ii]);
        const double Sp = fma(f, sv, fma(cf->k0p[1], nv, fma(ei_, zs, ek * xs)));
        const double Np = fma(f, nv, fma(cf->k0p[1], sv, fma(ei_, zn, ek * xn)));
        rsi = fma(ai, sv, rsi);
        rni = fma(ai, nv, rni);
        const double Nm = __shfl_up_sync(0xffffffffu, Np, TX);
        if (act) {
          fY[o] = iy > 0 ? Sp + Nm : Sp;
          if (lasty) fY[o + TX * N2] = Np;
          if (kk == 0) {
            double rsk = 0.0, rnk = 0.0;
#pragma unroll
            for (int k2 = 0; k2 < M; ++k2)
              if (k2 < CK) {
                rsk = fma(cf->a[sk + 2 * k2], S[2 * ii + 2 * NI * k2], rsk);
                rnk = fma(cf->a[sk + 2 * k2], N[2 * ii + 2 * NI * k2], rnk);
              }
            ok[4 * ii] = rsk;
            if (lasty) ok[TX * 2 * NI + 4 * ii] = rnk;
          }
        }
      }
      if (act) {
        oi[4 * kk] = rsi;
        if (lasty) oi[TX * 2 * NI + 4 * kk] = rni;
        if (NI == 1) {
          oi[1] = ok[1] = 0.0;
          if (lasty) oi[TX * 2 * NI + 1] = ok[TX * 2 * NI + 1] = 0.0;
        }
      }
    }
  }
  if (sk == DO && act) {   // z-faces: B of this layer (plane l), T (plane l+1)
    const double* Yb = inb.ye(iy, ix) + sj;
    const double* Yt = intp.ye(iy, ix) + sj;
    const double* Xb = inb.xe(iy, ix) + si;
    const double* Xt = intp.xe(iy, ix) + si;
    const double* fd = cf->fd[2] + si + NI * sj;
    constexpr int PO = CS<NI>::NE * 2 * NI;
    double* oi = rq + CS<NI>::R_ZI + (iy * TX + ix) * 2 * NI + 2 * sj + si;    // over i, keep j (l+1 at + PO)
    double* oj = rq + CS<NI>::R_ZJ + (iy * TX + ix) * 2 * NI + 2 * si + sj;    // over j, keep i
#pragma unroll
    for (int jj = 0; jj < M; ++jj) {
      if (jj >= CJ) continue;
      const double yb = fma(gi, Yb[NI + 2 * jj], Yb[2 * jj]), yt = fma(gi, Yt[NI + 2 * jj], Yt[2 * jj]);
      const double ej = cf->e[1][sj + 2 * jj], aj = cf->a[sj + 2 * jj];
      double rbi = 0.0, rti = 0.0;
#pragma unroll
      for (int ii = 0; ii < M; ++ii) {
        if (ii >= CI) continue;
        const int o = 2 * ii + 2 * NI * jj;
        const double bv = B[o], tv = T[o], f = fd[o], ei_ = cf->e[0][si + 2 * ii], ai = cf->a[si + 2 * ii];
        const double xb = fma(gj, Xb[TX * NI + 2 * ii], Xb[2 * ii]), xt = fma(gj, Xt[TX * NI + 2 * ii], Xt[2 * ii]);
        fB[o] += fma(f, bv, fma(cf->k0p[2], tv, fma(ei_, yb, ej * xb)));
        fT[o] = fma(f, tv, fma(cf->k0p[2], bv, fma(ei_, yt, ej * xt)));
        rbi = fma(ai, bv, rbi);
        rti = fma(ai, tv, rti);
        if (jj == 0) {
          double rbj = 0.0, rtj = 0.0;
#pragma unroll
          for (int j2 = 0; j2 < M; ++j2)
            if (j2 < CJ) {
              rbj = fma(cf->a[sj + 2 * j2], B[2 * ii + 2 * NI * j2], rbj);
              rtj = fma(cf->a[sj + 2 * j2], T[2 * ii + 2 * NI * j2], rtj);
            }
          oj[4 * ii] = rbj;
          oj[PO + 4 * ii] = rtj;
        }
      }
      oi[4 * jj] = rbi;
      oi[PO + 4 * jj] = rti;
      if (NI == 1) oi[1] = oi[PO + 1] = oj[1] = oj[PO + 1] = 0.0;
      (void)aj;
    }
  }

  // ---- phase B: condensed part of the class (registers only)
  const double* Dv = cf->dinv + si + NI * sj + N2 * sk;
  double qx[M][M], qy[M][M], qz[M][M];
  {
    double c1[M], c2[M], c3[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      c1[m] = cf->c[0][si + 2 * m];
      c2[m] = cf->c[1][sj + 2 * m];
      c3[m] = cf->c[2][sk + 2 * m];
    }
    double py[M][M];
#pragma unroll
    for (int ii = 0; ii < M; ++ii)
#pragma unroll
      for (int kk = 0; kk < M; ++kk) {
        py[ii][kk] = (ii < CI && kk < CK) ? fma(gj, N[2 * ii + 2 * NI * kk], S[2 * ii + 2 * NI * kk]) : 0.0;
        qy[ii][kk] = 0.0;
      }
#pragma unroll
    for (int jj = 0; jj < M; ++jj) {
#pragma unroll
      for (int kk = 0; kk < M; ++kk) qx[jj][kk] = 0.0;
#pragma unroll
      for (int ii = 0; ii < M; ++ii) qz[jj][ii] = 0.0;
      if (jj >= CJ) continue;
      double px[M], pz[M];
#pragma unroll
      for (int kk = 0; kk < M; ++kk)
        px[kk] = kk < CK ? fma(gi, E[2 * jj + 2 * NI * kk], W[2 * jj + 2 * NI * kk]) : 0.0;
#pragma unroll
      for (int ii = 0; ii < M; ++ii)
        pz[ii] = ii < CI ? fma(gk, T[2 * ii + 2 * NI * jj], B[2 * ii + 2 * NI * jj]) : 0.0;
#pragma unroll
      for (int ii = 0; ii < M; ++ii) {
        if (ii >= CI) continue;
#pragma unroll
        for (int kk = 0; kk < M; ++kk) {
          if (kk >= CK) continue;
          const double u = fma(c1[ii], px[kk], fma(c2[jj], py[ii][kk], c3[kk] * pz[ii]));
          const double v = u * Dv[2 * ii + 2 * NI * jj + 2 * N2 * kk];
          qx[jj][kk] = fma(c1[ii], v, qx[jj][kk]);
          qy[ii][kk] = fma(c2[jj], v, qy[ii][kk]);
          qz[jj][ii] = fma(c3[kk], v, qz[jj][ii]);
        }
      }
    }
  }
  // ---- output rounds: barrier (phase A complete), then round r of direction d by the classes
  // with s_d == r; W -= Q^0 + Q^1, E -= Q^0 - Q^1 (two elements of a face summed by shuffle).
#pragma unroll 1
  for (int r = 0; r < 2; ++r) {
    bar_named(1);
    if (r == si) {
#pragma unroll
      for (int jj = 0; jj < M; ++jj) {
        if (jj >= CJ) continue;
#pragma unroll
        for (int kk = 0; kk < M; ++kk) {
          if (kk >= CK) continue;
          const int o = 2 * jj + 2 * NI * kk;
          const double Q = qx[jj][kk];
          const double Qm = __shfl_up_sync(0xffffffffu, Q, 1);
          if (act) {
            fX[o] -= ix > 0 ? fma(gi, Qm, Q) : Q;
            if (lastx) fX[o + N2] -= gi * Q;
          }
        }
      }
    }
    if (r == sj) {
#pragma unroll
      for (int ii = 0; ii < M; ++ii) {
        if (ii >= CI) continue;
#pragma unroll
        for (int kk = 0; kk < M; ++kk) {
          if (kk >= CK) continue;
          const int o = 2 * ii + 2 * NI * kk;
          const double Q = qy[ii][kk];
          const double Qm = __shfl_up_sync(0xffffffffu, Q, TX);
          if (act) {
            fY[o] -= iy > 0 ? fma(gj, Qm, Q) : Q;
            if (lasty) fY[o + TX * N2] -= gj * Q;
          }
        }
      }
    }
    if (r == sk && act) {
#pragma unroll
      for (int jj = 0; jj < M; ++jj) {
        if (jj >= CJ) continue;
#pragma unroll
        for (int ii = 0; ii < M; ++ii) {
          if (ii >= CI) continue;
          const int o = 2 * ii + 2 * NI * jj;
          const double Q = qz[jj][ii];
          fB[o] -= Q;
          fT[o] -= gk * Q;
        }
      }
    }
  }
}

// warps w and w+4 share an SM sub-partition: pair the largest class with the smallest (class
// bits s_i s_j s_k; at n_I = 7 the point counts are 64+27, 48+36, 48+36, 48+36).
__device__ __constant__ int kWarpClass[8] = {0, 1, 2, 4, 7, 6, 5, 3};

template <int NI>
__global__ void __launch_bounds__(256, 1) k_apply_col(const __grid_constant__ ColParams P) {
  using C = CS<NI>;
  constexpr int N2 = C::N2, TX = C::TX, TY = C::TY, NT = C::NT;
  if (P.done != nullptr && *P.done != 0.0) return;
  const Geom& g = P.g;
  extern __shared__ double sm[];
  double* sA0 = sm + C::O_TAB;
  double* sLam = sA0 + 32;
  ColCoef* sCf = reinterpret_cast<ColCoef*>(sm + C::O_CF);
  double* const rq = sm + C::O_RQ;
  __shared__ unsigned long long sTicket;
  __shared__ int sEpoch;
  const int tid = threadIdx.x;
  if (tid == 0) sEpoch = *(volatile int*)&P.st->epoch + 1;
  long long ph_t0 = clock64();
  (void)ph_t0;
  Addr A{g};
  const double K00 = g.tab[TAB_SCAL + 0], K0p = g.tab[TAB_SCAL + 1], w0 = g.tab[TAB_SCAL + 2];
  const double w02 = w0 * w0;
  const double dA = g.d_uni[0], dB = g.d_uni[1], dC = g.d_uni[2], dD = g.d_uni[3];
  for (int t = tid; t < (int)(sizeof(ColCoef) / sizeof(double)); t += NT)
    sm[C::O_CF + t] = reinterpret_cast<const double*>(&P.cf)[t];
  for (int t = tid; t < NI; t += NT) {
    sA0[t] = g.tab[TAB_A0 + t];
    sLam[t] = g.tab[TAB_LAM + t];
  }
  // padding entries of y are written as 0 by the first CTA
  if (blockIdx.x == 0) {
    long long ends[7] = {g.off_f[0] + g.n_f[0] * N2, g.off_f[1] + g.n_f[1] * N2, g.off_f[2] + g.n_f[2] * N2,
                         g.off_e[0] + g.n_e[0] * NI, g.off_e[1] + g.n_e[1] * NI, g.off_e[2] + g.n_e[2] * NI,
                         g.off_v + g.n_v};
    long long nexts[7] = {g.off_f[1], g.off_f[2], g.off_e[0], g.off_e[1], g.off_e[2], g.off_v, g.n_total};
    for (int q = 0; q < 7; ++q)
      for (long long i = ends[q] + tid; i < nexts[q]; i += NT) P.y[i] = 0.0;
  }
  Side<NI> ac{sm + C::O_AS};
  // ---- lane tables of the edge / vertex primary part (no runtime division in the node loops)
  constexpr int NW = NT / 32;
  constexpr int EPW = 32 / NI;                               // edges per warp pass
  const int warp = tid >> 5, lane = tid & 31;
  const int vix = lane % TX, viy = lane / TX;                // element of this lane (condensed part)
  const int esub = lane / NI, ec = lane % NI;
  const bool evalid = lane < EPW * NI;
  // face-pass constants
  const double cx0 = dA * w0 + dB * K00, cy0 = dA * w0 + dC * K00, cz0 = dA * w0 + dD * K00;
  const double d1w0 = dB * w0, d2w0 = dC * w0, d3w0 = dD * w0;

  for (;;) {
    __syncthreads();
    if (tid == 0) sTicket = atomicAdd(&P.st->ticket, 1ULL);
    __syncthreads();
    const long long item = (long long)sTicket;
    if (item >= P.nitems) break;
    const int epoch = sEpoch;
    const int tx = (int)(item % P.ntx), ty = (int)(item / P.ntx);
    const int x0 = tx * TX, y0 = ty * TY;
    const int tw = min(TX, g.nx - x0), th = min(TY, g.ny - y0);
    int* const flag_me = P.flags + item * (g.nz + 1);
    const int* const flag_w = tx > 0 ? P.flags + (item - 1) * (g.nz + 1) : nullptr;
    const int* const flag_s = ty > 0 ? P.flags + (item - P.ntx) * (g.nz + 1) : nullptr;
    const int* const flag_sw = (tx > 0 && ty > 0) ? P.flags + (item - P.ntx - 1) * (g.nz + 1) : nullptr;

    // prologue: planes 0, 1 and side 0 as one cp.async group
    load_plane<NI>(P, Plane<NI>{sm + C::O_IP}, x0, y0, tw, th, 0);
    load_side<NI>(P, Side<NI>{sm + C::O_IS}, x0, y0, tw, th, 0);
    load_plane<NI>(P, Plane<NI>{sm + C::O_IP + C::PLANE}, x0, y0, tw, th, 1);
    cp_commit();
    for (int t = tid; t < C::PLANE; t += NT) sm[C::O_AP + t] = 0.0;

    for (int l = 0; l <= g.nz; ++l) {
      const bool last = (l == g.nz);         // final step: only plane nz remains
      const Side<NI> in{sm + C::O_IS + (l & 1) * C::SIDE};
      const Plane<NI> inb{sm + C::O_IP + (l & 1) * C::PLANE}, intp{sm + C::O_IP + ((l + 1) & 1) * C::PLANE};
      const Plane<NI> acb{sm + C::O_AP + (l & 1) * C::PLANE}, actp{sm + C::O_AP + ((l + 1) & 1) * C::PLANE};
      // early prefetch: side l+1 (overlaps this step's compute)
      if (l + 1 < g.nz) load_side<NI>(P, Side<NI>{sm + C::O_IS + ((l + 1) & 1) * C::SIDE}, x0, y0, tw, th, l + 1);
      cp_commit();
      cp_wait<1>();
      __syncthreads();
      SC_PHASE(0);
      if (!last) {
        // accumulators written with += below: z-edges of the side, edges / vertices of plane l+1
        for (int t = tid; t < C::ZE; t += NT) ac.b[C::S_ZE + t] = 0.0;
        for (int t = tid; t < C::PLANE - C::PZF; t += NT) actp.b[C::P_XE + t] = 0.0;
        // even / odd line sums of the edges (the faces' line sums come from the class warps)
        {
          constexpr int NZE = (TY + 1) * (TX + 1), NXE = (TY + 1) * TX, NYE = TY * (TX + 1);
          for (int t = tid; t < NZE + 2 * NXE + 2 * NYE; t += NT) {
            int r = t;
            if (r < NZE) { eo_reduce<NI>(in.b + C::S_ZE + r * NI, 1, sA0, rq + C::R_ZE + r * 2); continue; }
            r -= NZE;
            if (r < 2 * NXE) {
              const int kb = r / NXE, e = r - kb * NXE;
              eo_reduce<NI>((kb ? intp : inb).b + C::P_XE + e * NI, 1, sA0, rq + C::R_XE + r * 2);
              continue;
            }
            r -= 2 * NXE;
            const int kb = r / NYE, e = r - kb * NYE;
            eo_reduce<NI>((kb ? intp : inb).b + C::P_YE + e * NI, 1, sA0, rq + C::R_YE + r * 2);
          }
        }
        SC_PHASE(1);
        // ============ condensed part: parity-class warps, two output rounds ============
        vol_class<NI>(kWarpClass[warp], sCf, in, inb, intp, ac, acb, actp, rq, vix, viy, tw, th);
        __syncthreads();
        SC_PHASE(2);
        // ============ primary part Htilde_BB, entity-centric over the tile's elements ============
#if !defined(SC_EXP) || SC_EXP != 2
        // (Mtilde = diag(w0, 1..1, w0); Ktilde arrowhead: row 0 = (K00, a0, K0p),
        //  row p = (K0p, ap, K00), interior row m = (a0_m @0, Lam_m @m, ap_m @p).)
        // Faces: a warp (or a lane group) per face, lanes over the in-face nodes; edges: lane
        // groups of n_I per edge; vertices: a lane each.  Each accumulator entry is owned by
        // exactly one lane, which sums the contributions of the tile's adjacent elements.
        {
          auto present = [&](int ix, int iy) { return ix >= 0 && iy >= 0 && ix < tw && iy < th; };
          // ---- z-edges (fx = ix, fy = iy), coord k = c
          for (int e0 = warp * EPW; e0 < (TY + 1) * (TX + 1); e0 += NW * EPW) {
            const int e = e0 + esub, ix = e % (TX + 1), iy = e / (TX + 1), c = ec;
            if (!evalid || e >= (TY + 1) * (TX + 1) || ix > tw || iy > th) continue;
            const double u = in.ze(iy, ix)[c];
            const double tz = sA0[c] * (*inb.vv(iy, ix) + ((c & 1) ? -*intp.vv(iy, ix) : *intp.vv(iy, ix))) + sLam[c] * u;
            double y = 0.0;
#pragma unroll
            for (int el = 0; el < 4; ++el) {
              const int ib = el & 1, jb = el >> 1, ex = ix - ib, ey = iy - jb;
              if (!present(ex, ey)) continue;
              
              const double txl = (ib ? K0p : K00) * in.ze(iy, ex)[c] + (ib ? K00 : K0p) * in.ze(iy, ex + 1)[c] +
                                 eo_row(rq + C::R_YI + (iy * TX + ex) * 2 * NI + 2 * c, ib);
              const double tyl = (jb ? K0p : K00) * in.ze(ey, ix)[c] + (jb ? K00 : K0p) * in.ze(ey + 1, ix)[c] +
                                 eo_row(rq + C::R_XJ + (ey * (TX + 1) + ix) * 2 * NI + 2 * c, jb);
              y += dA * w02 * u + dB * w0 * txl + dC * w0 * tyl + dD * w02 * tz;
            }
            ac.ze(iy, ix)[c] += y;
          }
          // ---- x-edges (ex = ix, fy = iy) of planes l, l+1, coord i = c
          for (int e0 = warp * EPW; e0 < 2 * (TY + 1) * TX; e0 += NW * EPW) {
            const int e = e0 + esub, kb = e / ((TY + 1) * TX), ff = e % ((TY + 1) * TX), ix = ff % TX, iy = ff / TX;
            const int c = ec;
            if (!evalid || e >= 2 * (TY + 1) * TX || ix >= tw || iy > th) continue;
            const Plane<NI> pk = kb ? intp : inb;
            const double u = pk.xe(iy, ix)[c];
            const double txl = sA0[c] * (*pk.vv(iy, ix) + ((c & 1) ? -*pk.vv(iy, ix + 1) : *pk.vv(iy, ix + 1))) + sLam[c] * u;
            const double tzl = (kb ? K0p : K00) * inb.xe(iy, ix)[c] + (kb ? K00 : K0p) * intp.xe(iy, ix)[c] +
                               eo_row(rq + C::R_YK + (iy * TX + ix) * 2 * NI + 2 * c, kb);
            double y = 0.0;
#pragma unroll
            for (int el = 0; el < 2; ++el) {
              const int jb = el, ey = iy - jb;
              if (!present(ix, ey)) continue;
              
              const double tyl = (jb ? K0p : K00) * pk.xe(ey, ix)[c] + (jb ? K00 : K0p) * pk.xe(ey + 1, ix)[c] +
                                 eo_row(rq + C::R_ZJ + (kb * TY * TX + ey * TX + ix) * 2 * NI + 2 * c, jb);
              y += dA * w02 * u + dB * w02 * txl + dC * w0 * tyl + dD * w0 * tzl;
            }
            (kb ? actp : acb).xe(iy, ix)[c] += y;
          }
          // ---- y-edges (fx = ix, ey = iy) of planes l, l+1, coord j = c
          for (int e0 = warp * EPW; e0 < 2 * TY * (TX + 1); e0 += NW * EPW) {
            const int e = e0 + esub, kb = e / (TY * (TX + 1)), ff = e % (TY * (TX + 1)), ix = ff % (TX + 1),
                      iy = ff / (TX + 1);
            const int c = ec;
            if (!evalid || e >= 2 * TY * (TX + 1) || ix > tw || iy >= th) continue;
            const Plane<NI> pk = kb ? intp : inb;
            const double u = pk.ye(iy, ix)[c];
            const double tyl = sA0[c] * (*pk.vv(iy, ix) + ((c & 1) ? -*pk.vv(iy + 1, ix) : *pk.vv(iy + 1, ix))) + sLam[c] * u;
            const double tzl = (kb ? K0p : K00) * inb.ye(iy, ix)[c] + (kb ? K00 : K0p) * intp.ye(iy, ix)[c] +
                               eo_row(rq + C::R_XK + (iy * (TX + 1) + ix) * 2 * NI + 2 * c, kb);
            double y = 0.0;
#pragma unroll
            for (int el = 0; el < 2; ++el) {
              const int ib = el, ex = ix - ib;
              if (!present(ex, iy)) continue;
              
              const double txl = (ib ? K0p : K00) * pk.ye(iy, ex)[c] + (ib ? K00 : K0p) * pk.ye(iy, ex + 1)[c] +
                                 eo_row(rq + C::R_ZI + (kb * TY * TX + iy * TX + ex) * 2 * NI + 2 * c, ib);
              y += dA * w02 * u + dB * w0 * txl + dC * w02 * tyl + dD * w0 * tzl;
            }
            (kb ? actp : acb).ye(iy, ix)[c] += y;
          }
          // ---- vertices (fx = ix, fy = iy) of planes l, l+1
          for (int v = tid; v < 2 * (TY + 1) * (TX + 1); v += NT) {
            const int kb = v / ((TY + 1) * (TX + 1)), ff = v % ((TY + 1) * (TX + 1)), ix = ff % (TX + 1),
                      iy = ff / (TX + 1);
            if (ix > tw || iy > th) continue;
            const Plane<NI> pk = kb ? intp : inb;
            const double u = *pk.vv(iy, ix);
            const double tzl = (kb ? K0p : K00) * *inb.vv(iy, ix) + (kb ? K00 : K0p) * *intp.vv(iy, ix) +
                               eo_row(rq + C::R_ZE + (iy * (TX + 1) + ix) * 2, kb);
            double y = 0.0;
#pragma unroll
            for (int el = 0; el < 4; ++el) {
              const int ib = el & 1, jb = el >> 1, ex = ix - ib, ey = iy - jb;
              if (!present(ex, ey)) continue;
              
              const double txl = (ib ? K0p : K00) * *pk.vv(iy, ex) + (ib ? K00 : K0p) * *pk.vv(iy, ex + 1) +
                                 eo_row(rq + C::R_XE + (kb * (TY + 1) * TX + iy * TX + ex) * 2, ib);
              const double tyl = (jb ? K0p : K00) * *pk.vv(ey, ix) + (jb ? K00 : K0p) * *pk.vv(ey + 1, ix) +
                                 eo_row(rq + C::R_YE + (kb * TY * (TX + 1) + ey * (TX + 1) + ix) * 2, jb);
              y += dA * w02 * w0 * u + w02 * (dB * txl + dC * tyl + dD * tzl);
            }
            *(kb ? actp : acb).vv(iy, ix) += y;
          }
        }
#endif
        __syncthreads();
        SC_PHASE(6);
      }
      // late prefetch: plane l+2 into the buffer of plane l (no longer read)
      if (l + 2 <= g.nz) load_plane<NI>(P, Plane<NI>{sm + C::O_IP + (l & 1) * C::PLANE}, x0, y0, tw, th, l + 2);
      cp_commit();
      // ================= finalize step l: publish / write owned / park ==========================
      // Ownership: the highest-ticket contributing tile (tiles are ticketed x-fastest): a tile
      // owns its W / S boundaries (finished one step later from parked partials) and publishes
      // its E / N boundaries (y-in-place; the three 4-tile rim corners go to corner records).
      // Every loop below is a warp per contiguous row with range-only classification.
      {
        const bool pzd = zdir(g, l);
        const int x1 = x0 + tw, y1 = y0 + th;
        const bool hasE = x1 < g.nx, hasN = y1 < g.ny, hasW = x0 > 0, hasS = y0 > 0;
        const bool dW = (x0 == 0), dE = (x1 == g.nx);                 // Dirichlet row ends
        double* const pd = P.pending + (item * 2 + (l & 1)) * (long long)C::PEND;
#if !defined(SC_EXP) || SC_EXP != 1
        // ---- (a) publish
        if (!last) {
          if (hasE)
            for (int row = warp; row < th; row += NW) {
              double* yo = P.y + A.xf(x1, y0 + row, l);
              const double* s = ac.xf(row, tw);
              for (int t = lane; t < N2; t += 32) yo[t] = s[t];
            }
          if (hasN) {
            double* yo = P.y + A.yf(x0, y1, l);
            const double* s = ac.yf(th, 0);
            for (int t = tid; t < tw * N2; t += NT) yo[t] = s[t];
          }
        }
        if (!pzd) {
          if (hasN) {
            double* yo = P.y + A.xe(x0, y1, l);
            const double* s = acb.xe(th, 0);
            for (int t = tid; t < tw * NI; t += NT) yo[t] = s[t];
          }
          if (hasE)
            for (int row = warp; row < th; row += NW) {
              double* yo = P.y + A.ye(x1, y0 + row, l);
              const double* s = acb.ye(row, tw);
              for (int t = lane; t < NI; t += 32) yo[t] = s[t];
            }
        }
        // z-edges (layer l, c < NI) / vertices (plane l, c == NI) on the E column and N row
        if (warp == 0) {
          const int nE = hasE ? th + 1 : 0, nN = hasN ? tw : 0;
          for (int t = lane; t < (nE + nN) * (NI + 1); t += 32) {
            const int ent = t / (NI + 1), c = t - ent * (NI + 1);
            const bool isv = (c == NI);
            if (isv ? pzd : last) continue;
            int ix, iy;
            if (ent < nE) { ix = tw; iy = ent; } else { ix = ent - nE; iy = th; }
            const int fx = x0 + ix, fy = y0 + iy;
            if (fx == 0 || fy == 0 || fy == g.ny) continue;          // Dirichlet
            const bool ex_ = (ix == tw && hasE), ny_ = (iy == th && hasN);
            const double v = isv ? *acb.vv(iy, ix) : ac.ze(iy, ix)[c];
            if (ex_ && ny_) corner_rec(P, fx / TX, fy / TY, l, 0)[c] = v;                   // SW of owner
            else if (ex_ && iy == 0 && hasS) corner_rec(P, fx / TX, fy / TY, l, 2)[c] = v;   // W of owner
            else if (ny_ && ix == 0 && hasW) corner_rec(P, fx / TX, fy / TY, l, 1)[c] = v;   // S of owner
            else if (isv) P.y[A.vv(fx, fy, l)] = v;
            else P.y[A.ze(fx, fy, l) + c] = v;
          }
        }
#endif
        // publication: the CTA barrier orders every thread's stores before thread 0's GPU-scope
        // fence + release store of the flag (cumulativity of bar.sync + fence.acq_rel.gpu)
        __syncthreads();
        SC_PHASE(7);
        if (tid == 0) {
          __threadfence();
          flag_release(flag_me + l, epoch);
        }
#if !defined(SC_EXP) || SC_EXP != 1
#if defined(SC_EXP) && SC_EXP == 7
        if (false)
#endif
        // ---- (b) owned entities (incl. Dirichlet zeros) and (b') parked W / S partials.
        // Flat loops over the whole tile of each class (all warps busy); smem rows and global
        // rows are both contiguous, so entry (row, c) is base + row * stride + c on both sides.
        {
          const unsigned nxf = (unsigned)(g.nx + 1) * N2, nyf = (unsigned)g.nx * N2;
          const unsigned nxe = (unsigned)g.nx * NI, nye = (unsigned)(g.nx + 1) * NI;
          const unsigned nze = (unsigned)(g.nx + 1) * NI, nvv = (unsigned)(g.nx + 1);
          if (!last) {
            {   // x-faces: rows iy < th, entries c < (tw + 1) N2
              constexpr unsigned RL = (TX + 1) * N2;
              double* yo = P.y + A.xf(x0, y0, l);
              const unsigned t1 = hasE ? tw * N2 : (tw + 1) * N2;
              for (unsigned t = tid; t < th * RL; t += NT) {
                const unsigned row = t / RL, c = t - row * RL;
                if (c >= t1) continue;
                const double v = ac.b[C::S_XF + t];
                if (c < N2 && hasW) { pd[C::PD_XF + row * N2 + c] = v; continue; }
                yo[row * nxf + c] = ((dW && c < N2) || (dE && c >= tw * N2)) ? 0.0 : v;
              }
            }
            {   // y-faces: rows iy <= th
              constexpr unsigned RL = TX * N2;
              double* yo = P.y + A.yf(x0, y0, l);
              for (unsigned t = tid; t < (th + 1) * RL; t += NT) {
                const unsigned row = t / RL, c = t - row * RL;
                if (c >= tw * N2 || (row == th && hasN)) continue;
                const double v = ac.b[C::S_YF + t];
                if (row == 0 && hasS) { pd[C::PD_YF + c] = v; continue; }
                const int fy = y0 + row;
                yo[row * nyf + c] = (fy == 0 || fy == g.ny) ? 0.0 : v;
              }
            }
            {   // z-edges: rows iy <= th, entries c < (tw + 1) NI
              constexpr unsigned RL = (TX + 1) * NI;
              double* yo = P.y + A.ze(x0, y0, l);
              for (unsigned t = tid; t < (th + 1) * RL; t += NT) {
                const unsigned row = t / RL, c = t - row * RL;
                if (c >= (tw + 1) * NI) continue;
                const bool lo = c < NI, hi = c >= tw * NI;
                if ((row == th && hasN) || (hi && hasE)) continue;               // published
                const int fy = y0 + row;
                const bool rd = fy == 0 || fy == g.ny;
                const double v = ac.b[C::S_ZE + t];
                if (rd || (lo && dW) || (hi && dE)) { yo[row * nze + c] = 0.0; continue; }
                if (lo && hasW) { pd[C::PD_ZEW + row * NI + c] = v; continue; }    // W column
                if (row == 0 && hasS) { pd[C::PD_ZES + c - NI] = v; continue; }   // S row
                yo[row * nze + c] = v;
              }
            }
          }
          {   // z-faces of plane l
            constexpr unsigned RL = TX * N2;
            double* yo = P.y + A.zf(x0, y0, l);
            for (unsigned t = tid; t < th * RL; t += NT) {
              const unsigned row = t / RL, c = t - row * RL;
              if (c < tw * N2) yo[row * nyf + c] = pzd ? 0.0 : acb.b[C::P_ZF + t];
            }
          }
          {   // x-edges of plane l: rows iy <= th
            constexpr unsigned RL = TX * NI;
            double* yo = P.y + A.xe(x0, y0, l);
            for (unsigned t = tid; t < (th + 1) * RL; t += NT) {
              const unsigned row = t / RL, c = t - row * RL;
              if (c >= tw * NI || (row == th && hasN && !pzd)) continue;
              const int fy = y0 + row;
              const bool rd = pzd || fy == 0 || fy == g.ny;
              const double v = acb.b[C::P_XE + t];
              if (row == 0 && hasS && !rd) { pd[C::PD_XE + c] = v; continue; }
              yo[row * nxe + c] = rd ? 0.0 : v;
            }
          }
          {   // y-edges of plane l: rows iy < th, entries c < (tw + 1) NI
            constexpr unsigned RL = (TX + 1) * NI;
            double* yo = P.y + A.ye(x0, y0, l);
            for (unsigned t = tid; t < th * RL; t += NT) {
              const unsigned row = t / RL, c = t - row * RL;
              if (c >= (tw + 1) * NI) continue;
              const bool lo = c < NI, hi = c >= tw * NI;
              if (hi && hasE && !pzd) continue;
              const double v = acb.b[C::P_YE + t];
              if (pzd || (lo && dW) || (hi && dE)) { yo[row * nye + c] = 0.0; continue; }
              if (lo && hasW) { pd[C::PD_YE + row * NI + c] = v; continue; }
              yo[row * nye + c] = v;
            }
          }
          {   // vertices of plane l: rows iy <= th, entries c <= tw
            constexpr unsigned RL = TX + 1;
            double* yo = P.y + A.vv(x0, y0, l);
            for (unsigned t = tid; t < (th + 1) * RL; t += NT) {
              const unsigned row = t / RL, c = t - row * RL;
              if (c > (unsigned)tw) continue;
              const bool lo = c == 0, hi = c == (unsigned)tw;
              if ((row == th && hasN && !pzd) || (hi && hasE && !pzd)) continue;
              const int fy = y0 + row;
              const bool rd = pzd || fy == 0 || fy == g.ny;
              const double v = acb.b[C::P_VV + t];
              if (rd || (lo && dW) || (hi && dE)) { yo[row * nvv + c] = 0.0; continue; }
              if (lo && hasW) { pd[C::PD_VW + row] = v; continue; }
              if (row == 0 && hasS) { pd[C::PD_VS + c - 1] = v; continue; }
              yo[row * nvv + c] = v;
            }
          }
        }
#endif
      }
      // (c, d) finish the W / S boundary entities of the PREVIOUS step
#if !defined(SC_EXP) || (SC_EXP != 1 && SC_EXP != 6)
      if (l >= 1) finish_boundary<NI>(P, item, l - 1, x0, y0, tw, th, flag_w, flag_s, flag_sw, epoch);
#endif
      __syncthreads();
      SC_PHASE(8);
    }
    finish_boundary<NI>(P, item, g.nz, x0, y0, tw, th, flag_w, flag_s, flag_sw, epoch);
    __syncthreads();
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&P.st->finished, 1u) == gridDim.x - 1) {
      P.st->ticket = 0ULL;
      P.st->finished = 0u;
      atomicAdd(&P.st->epoch, 1);
      __threadfence();
    }
  }
}


template <int NI>
static int launch_col_t(const ColParams& P, cudaStream_t st, int* nl, int* grid_out) {
  using C = CS<NI>;
  static_assert(sizeof(double) * C::TOTAL <= 227 * 1024, "shared memory budget");
  const size_t smem = sizeof(double) * C::TOTAL;
  static int max_active = -1, nsm = 0;
  if (max_active < 0) {
    cudaFuncSetAttribute(k_apply_col<NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_active, k_apply_col<NI>, C::NT, smem);
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (max_active < 1) max_active = 1;
  }
  int grid = max_active * nsm;
  if (grid > P.nitems) grid = P.nitems;
  *grid_out = grid;
  k_apply_col<NI><<<grid, C::NT, smem, st>>>(P);
  (*nl)++;
  return cudaGetLastError();
}

#if defined(SC_EXP) && SC_EXP == 9
extern "C" int sc_exp_phase_cycles(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 16);
}
#endif

bool col_supported(int ni) { return ni >= 1 && ni <= 7; }

void col_tile(int ni, int* tx, int* ty, int* pend) {
  switch (ni) {
#define TCASE(N) case N: *tx = CS<N>::TX; *ty = CS<N>::TY; *pend = CS<N>::PEND; return;
    TCASE(1) TCASE(2) TCASE(3) TCASE(4) TCASE(5) TCASE(6) TCASE(7)
#undef TCASE
    default: *tx = *ty = *pend = 0;
  }
}

// Host-side coefficient block of the uniform-geometry kernel (c[d][m] = d_{d+1} a0_m, D^{-1}).
void col_make_coef(int ni, const double* d, const double* a0, const double* lam, double K00, double K0p, double w0,
                   std::vector<unsigned char>& out) {
  ColCoef cf;
  memset(&cf, 0, sizeof(cf));
  for (int m = 0; m < ni && m < 8; ++m) {
    cf.a[m] = a0[m];
    for (int q = 0; q < 3; ++q) {
      cf.c[q][m] = d[q + 1] * a0[m];
      cf.e[q][m] = d[q + 1] * w0 * a0[m];
    }
  }
  for (int q = 0; q < 3; ++q) cf.k0p[q] = d[q + 1] * K0p;
  if (ni <= 8)
    for (int b = 0; b < ni; ++b)
      for (int a = 0; a < ni; ++a) {
        cf.fd[0][a + ni * b] = d[0] * w0 + d[1] * K00 + d[2] * w0 * lam[a] + d[3] * w0 * lam[b];
        cf.fd[1][a + ni * b] = d[0] * w0 + d[1] * w0 * lam[a] + d[2] * K00 + d[3] * w0 * lam[b];
        cf.fd[2][a + ni * b] = d[0] * w0 + d[1] * w0 * lam[a] + d[2] * w0 * lam[b] + d[3] * K00;
      }
  if (ni <= 8)
    for (int k = 0; k < ni; ++k)
      for (int j = 0; j < ni; ++j)
        for (int i = 0; i < ni; ++i)
          cf.dinv[i + ni * (j + ni * k)] = 1.0 / (d[0] + d[1] * lam[i] + d[2] * lam[j] + d[3] * lam[k]);
  out.resize(sizeof(cf));
  memcpy(out.data(), &cf, sizeof(cf));
}

int launch_apply_col(const ColParams& P, void* stream, int* nl, int* grid_out, void* events) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  if (ev) cudaEventRecord(ev[0], st);
  int r;
  switch (P.g.ni) {
#define LCASE(N) case N: r = launch_col_t<N>(P, st, nl, grid_out); break;
    LCASE(1) LCASE(2) LCASE(3) LCASE(4) LCASE(5) LCASE(6) LCASE(7)
#undef LCASE
    default: return cudaErrorInvalidValue;
  }
  if (ev) cudaEventRecord(ev[1], st);
  return r;
}

int launch_apply_col_raw(const Geom& g, const double* x, double* y, const double* done, void* state, int* flags,
                         double* corner, double* pending, int ntx, int nty, const void* coef, void* stream, int* nl,
                         void* events) {
  ColParams P;
  P.g = g; P.x = x; P.y = y; P.done = done; P.st = (ColState*)state; P.flags = flags; P.corner = corner;
  P.pending = pending;
  P.ntx = ntx; P.nty = nty; P.nitems = ntx * nty;
  memcpy(&P.cf, coef, sizeof(ColCoef));
  int grid = 0;
  return launch_apply_col(P, stream, nl, &grid, events);
}

}  // namespace sc
