// Condensed operator v2 (rows a3-a8 of SURVEY §8(a)): tile-column kernel.
//
// Work decomposition.  The slab's elements are cut into xy-tiles of TX x TY elements; a work
// item is one tile-column (all nz element layers of the tile).  A persistent CTA takes items
// in ticket order and marches up the column one element layer at a time.  All entities of
// the skeleton are assembled on chip except those on tile side boundaries, which are
// finished with a decoupled look-back: the lower-ticket contributor stores its partial sum
// straight into y (or, on the 4-tile corner lines, into a small corner record), publishes a
// per-(item, layer) flag, and the owner (highest-ticket contributor) adds it and writes the
// final value.  Items only ever wait on lower tickets, which are held by running CTAs, so
// the scheme is deadlock free.  Every skeleton entry is written exactly once (no memset, no
// atomics) and read from HBM once (re-reads of shared entities hit L2).
//
// Per element (transformed basis, §6, Table 2, Eq. 26):
//   faces-in + D^{-1} + faces-out in the even/odd form: with ap = sigma .* a0 (sigma_m = (-1)^m,
//   the parity of the m-th M-orthonormal eigenvector), the six rank-1 face terms combine to
//     u(i,j,k) = a_i Px^{s_i}(j,k) + a_j Py^{s_j}(i,k) + a_k Pz^{s_k}(i,j),  P^{+-} = d (F_lo +- F_hi)
//   and the six faces-out reductions to even/odd partial sums Q^{+-}, F_lo -= d (Q+ + Q-),
//   F_hi -= d (Q+ - Q-): 7 instead of 13 FP64 instructions per interior point, same result.
//   Thread (e, k) owns the k-plane of element e: x- and y-reductions stay in registers, the
//   z-reduction is a parity-preserving butterfly (xor 2, xor 4) across the k lanes.
//   The primary part Htilde_BB is applied per element and accumulated in shared memory in
//   four colour phases (elements of one colour share no entity).
#include <cuda_runtime.h>
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
};

template <int NI>
struct CS {
  static constexpr int N2 = NI * NI;
  static constexpr int LPE = NI <= 1 ? 1 : (NI <= 2 ? 2 : (NI <= 4 ? 4 : 8));   // k lanes per element
  static constexpr int JS = NI >= 2 ? 2 : 1;                                     // j-splits per k-plane
  static constexpr int JH = (NI + JS - 1) / JS;                                  // j rows per thread (j = JS jj + jh)
  static constexpr int NT = 256;
  static constexpr int NE = NT / (LPE * JS);
  static constexpr int TX = NE >= 256 ? 16 : (NE >= 32 ? 8 : 4);
  static constexpr int TY = NE / TX;
  static constexpr int XF = TY * (TX + 1) * N2;
  static constexpr int YF = (TY + 1) * TX * N2;
  static constexpr int ZE = (TY + 1) * (TX + 1) * NI;
  static constexpr int SIDE = XF + YF + ZE;
  static constexpr int PZF = TY * TX * N2;
  static constexpr int PXE = (TY + 1) * TX * NI;
  static constexpr int PYE = TY * (TX + 1) * NI;
  static constexpr int PVV = (TY + 1) * (TX + 1);
  static constexpr int PLANE = PZF + PXE + PYE + PVV;
  static constexpr int QZ = NE * 2 * N2;
  // even/odd reduction buffers (aliased with QZ: used after the z outputs are consumed)
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
  static constexpr int RQ = QZ > RED ? QZ : RED;
  static constexpr int DINV = NI * NI * NI;
  static constexpr int O_IS = 0;                     // 2 side input buffers
  static constexpr int O_IP = O_IS + 2 * SIDE;       // 2 plane input buffers
  static constexpr int O_AS = O_IP + 2 * PLANE;      // side accumulator
  static constexpr int O_AP = O_AS + SIDE;           // 2 plane accumulators
  static constexpr int O_RQ = O_AP + 2 * PLANE;      // QZ staging / reduction buffers
  static constexpr int O_DINV = O_RQ + RQ;
  static constexpr int O_D = O_DINV + DINV;          // per-element d: NE x 4
  static constexpr int O_TAB = O_D + 4 * NE;         // a0, ap, lam (3 x 32)
  static constexpr int TOTAL = O_TAB + 3 * 32;
  static constexpr int NSH = 6 * N2 + 12 * NI + 8;   // element shell nodes
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

template <int NI, bool UNIFORM>
__global__ void __launch_bounds__(256, 2) k_apply_col(ColParams P) {
  using C = CS<NI>;
  constexpr int N2 = C::N2, TX = C::TX, TY = C::TY, NT = C::NT, LPE = C::LPE, JS = C::JS, JH = C::JH;
  if (P.done != nullptr && *P.done != 0.0) return;
  const Geom& g = P.g;
  extern __shared__ double sm[];
  double* sDinv = sm + C::O_DINV;
  double* sD = sm + C::O_D;
  double* sA0 = sm + C::O_TAB;
  double* sLam = sA0 + 64;
  double* const rq = sm + C::O_RQ;
  __shared__ unsigned long long sTicket;
  __shared__ int sEpoch;
  const int tid = threadIdx.x;
  if (tid == 0) sEpoch = *(volatile int*)&P.st->epoch + 1;
  long long ph_t0 = clock64();
  Addr A{g};
  const double K00 = g.tab[TAB_SCAL + 0], K0p = g.tab[TAB_SCAL + 1], w0 = g.tab[TAB_SCAL + 2];
  const double w02 = w0 * w0;
  for (int t = tid; t < NI; t += NT) {
    sA0[t] = g.tab[TAB_A0 + t];
    sLam[t] = g.tab[TAB_LAM + t];
  }
  if (UNIFORM)
    for (int t = tid; t < C::DINV; t += NT) sDinv[t] = g.dinv[t];
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
  // ---- per-thread constants of the volume phase: thread (e, k)
  const int ve = tid / (LPE * JS), vk = tid % LPE, vjh = (tid / LPE) % JS;
  const bool vact = vk < NI;
  const int vix = ve % TX, viy = ve / TX;
  const double sk = (vk & 1) ? -1.0 : 1.0;
  const int kk = vact ? vk : 0;
  // ---- lane tables of the edge / vertex primary part (no runtime division in the node loops)
  constexpr int NW = NT / 32;
  constexpr int EPW = 32 / NI;                               // edges per warp pass
  const int warp = tid >> 5, lane = tid & 31;
  const int esub = lane / NI, ec = lane % NI;
  const bool evalid = lane < EPW * NI;

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
    const bool eact = vact && vix < tw && viy < th;

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
        for (int t = tid; t < C::SIDE; t += NT) ac.b[t] = 0.0;
        for (int t = tid; t < C::PLANE; t += NT) actp.b[t] = 0.0;
        if (UNIFORM) {
          for (int t = tid; t < 4 * C::NE; t += NT) sD[t] = g.d_uni[t & 3];
        } else {
          for (int t = tid; t < C::NE; t += NT) {
            int ex = x0 + min(t % TX, tw - 1), ey = y0 + min(t / TX, th - 1);
            double d[4];
            metric(g, ex, ey, l, d);
            for (int q = 0; q < 4; ++q) sD[t * 4 + q] = d[q];
          }
        }
        __syncthreads();
        SC_PHASE(1);
#if !defined(SC_EXP) || SC_EXP != 3
        // ============ condensed part (faces-in, D^{-1}, faces-out; even / odd form of Table 2)
        //              fused with the primary part of the element's x- and y-faces ============
        // Thread (e, jh, k): k-plane of element e, rows j = 2 jj + jh (all of one parity, so
        // sigma_j is a per-thread constant and the y-reduction yields one parity class).
        {
          const double* d = sD + ve * 4;
          const double d0 = d[0], d1 = d[1], d2 = d[2], d3 = d[3];
          const double ak = eact ? sA0[kk] : 0.0;
          const double akd3 = ak * d3;
          const double lamk = sLam[kk];
          const double sj = (JS == 2 && vjh) ? -1.0 : 1.0;
          double pxp[JH], pxm[JH], ajr[JH], py[NI];
          double qxp[JH], qxm[JH], qy[NI];
          const double* W = in.xf(viy, vix);
          const double* E = in.xf(viy, vix + 1);
          const double* S = in.yf(viy, vix);
          const double* N = in.yf(viy + 1, vix);
          const double* B = inb.zf(viy, vix);
          const double* T = intp.zf(viy, vix);
#pragma unroll
          for (int jj = 0; jj < JH; ++jj) {
            const int j = JS * jj + vjh;
            const bool ok = eact && j < NI;
            const double w = ok ? W[j + NI * kk] : 0.0, e = ok ? E[j + NI * kk] : 0.0;
            pxp[jj] = d1 * (w + e);
            pxm[jj] = d1 * (w - e);
            ajr[jj] = ok ? sA0[j] : 0.0;
            qxp[jj] = qxm[jj] = 0.0;
          }
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            py[i] = eact ? d2 * fma(sj, N[i + NI * kk], S[i + NI * kk]) : 0.0;
            qy[i] = 0.0;
          }
          double* const qz = rq;
#pragma unroll
          for (int jj = 0; jj < JH; ++jj) {
            const int j = min(JS * jj + vjh, NI - 1);
            const bool jok = (JS * jj + vjh) < NI;
            const double aj = ajr[jj];
            const double* Bj = B + NI * j;
            const double* Tj = T + NI * j;
            const double* Dj = sDinv + NI * j + N2 * kk;
#pragma unroll
            for (int i = 0; i < NI; ++i) {
              const double pz = fma(sk, Tj[i], Bj[i]);
              const double u = fma(sA0[i], (i & 1) ? pxm[jj] : pxp[jj], fma(aj, py[i], akd3 * pz));
              double v;
              if (UNIFORM) v = u * Dj[i];
              else v = u / (d0 + d1 * sLam[i] + d2 * sLam[j] + d3 * lamk);
              if (i & 1) qxm[jj] = fma(sA0[i], v, qxm[jj]); else qxp[jj] = fma(sA0[i], v, qxp[jj]);
              qy[i] = fma(aj, v, qy[i]);
              double c = ak * v;
              if (LPE >= 4) c += __shfl_xor_sync(0xffffffffu, c, 2);
              if (LPE >= 8) c += __shfl_xor_sync(0xffffffffu, c, 4);
              if (vk < 2 && eact && jok) qz[(ve * 2 + vk) * N2 + i + NI * j] = c;
            }
          }
          // y-reduction: this thread holds Q_y^{sigma = (-1)^jh}(i) for all i; fetch the other class
          double qyo[NI];
#pragma unroll
          for (int i = 0; i < NI; ++i) qyo[i] = (JS == 2) ? __shfl_xor_sync(0xffffffffu, qy[i], LPE) : 0.0;
          // primary part of the element's four side faces at this k (Eq. 26 generalised):
          //   W/E node (j,k): (d0 w0 + d1 K00 + d2 w0 Lam_j + d3 w0 Lam_k) u + d1 K0p u_opp
          //                   + d2 w0 a0_j (Z(ib,0)[k] + s_j Z(ib,1)[k]) + d3 w0 a0_k (Y(ib,0)[j] + s_k Y(ib,1)[j])
          //   S/N node (i,k): (d0 w0 + d1 w0 Lam_i + d2 K00 + d3 w0 Lam_k) u + d2 K0p u_opp
          //                   + d1 w0 a0_i (Z(0,jb)[k] + s_i Z(1,jb)[k]) + d3 w0 a0_k (X(jb,0)[i] + s_k X(jb,1)[i])
          // This thread owns rows j = i = 2 jj + jh of the four faces.
          const double z00 = in.ze(viy, vix)[kk], z10 = in.ze(viy, vix + 1)[kk];
          const double z01 = in.ze(viy + 1, vix)[kk], z11 = in.ze(viy + 1, vix + 1)[kk];
          const double base = d0 * w0 + d3 * w0 * lamk;
          const double wak = d3 * w0 * ak;
          double oW[JH], oE[JH], oS[JH], oN[JH];
#pragma unroll
          for (int jj = 0; jj < JH; ++jj) {
            const int r = min(JS * jj + vjh, NI - 1);         // row index (j for W/E, i for S/N)
            const double ar = sA0[r], lr = sLam[r];
            const double w = W[r + NI * kk], e = E[r + NI * kk], s = S[r + NI * kk], n = N[r + NI * kk];
            const double dxy = base + d1 * K00 + d2 * w0 * lr;
            const double dyx = base + d2 * K00 + d1 * w0 * lr;
            oW[jj] = dxy * w + d1 * K0p * e + d2 * w0 * ar * fma(sj, z01, z00) +
                     wak * fma(sk, intp.ye(viy, vix)[r], inb.ye(viy, vix)[r]);
            oE[jj] = dxy * e + d1 * K0p * w + d2 * w0 * ar * fma(sj, z11, z10) +
                     wak * fma(sk, intp.ye(viy, vix + 1)[r], inb.ye(viy, vix + 1)[r]);
            oS[jj] = dyx * s + d2 * K0p * n + d1 * w0 * ar * fma(sj, z10, z00) +
                     wak * fma(sk, intp.xe(viy, vix)[r], inb.xe(viy, vix)[r]);
            oN[jj] = dyx * n + d2 * K0p * s + d1 * w0 * ar * fma(sj, z11, z01) +
                     wak * fma(sk, intp.xe(viy + 1, vix)[r], inb.xe(viy + 1, vix)[r]);
          }
          // outputs: low faces first, high faces after a barrier (race-free accumulation)
          double qyp_r[JH], qym_r[JH];
#pragma unroll
          for (int jj = 0; jj < JH; ++jj) {
            const int i0 = min(JS * jj, NI - 1), i1 = min(JS * jj + 1, NI - 1);
            // row i = 2 jj + jh: Q+ is held by the jh = 0 thread, Q- by the jh = 1 thread
            qyp_r[jj] = (JS == 1 || vjh == 0) ? qy[i0] : qyo[i1];
            qym_r[jj] = (JS == 1) ? 0.0 : (vjh == 0 ? qyo[i0] : qy[i1]);
          }
          if (eact) {
            double* aW = ac.xf(viy, vix);
            double* aS = ac.yf(viy, vix);
#pragma unroll
            for (int jj = 0; jj < JH; ++jj) {
              const int r = JS * jj + vjh;
              if (r >= NI) continue;
              aW[r + NI * kk] += oW[jj] - d1 * (qxp[jj] + qxm[jj]);
              aS[r + NI * kk] += oS[jj] - d2 * (qyp_r[jj] + qym_r[jj]);
            }
          }
          __syncthreads();
          SC_PHASE(2);
          if (eact) {
            double* aE = ac.xf(viy, vix + 1);
            double* aN = ac.yf(viy + 1, vix);
#pragma unroll
            for (int jj = 0; jj < JH; ++jj) {
              const int r = JS * jj + vjh;
              if (r >= NI) continue;
              aE[r + NI * kk] += oE[jj] - d1 * (qxp[jj] - qxm[jj]);
              aN[r + NI * kk] += oN[jj] - d2 * (qyp_r[jj] - qym_r[jj]);
            }
          }
        }
        __syncthreads();
        SC_PHASE(3);
#endif
#if !defined(SC_EXP) || SC_EXP != 4
        // z outputs: B -= d3 (Q+ + Q-), T -= d3 (Q+ - Q-), plus the primary part of the element's
        // B and T faces: (d0 w0 + d1 w0 Lam_i + d2 w0 Lam_j + d3 K00) u + d3 K0p u_opp
        //   + d1 w0 a0_i (Y(0,kb)[j] + s_i Y(1,kb)[j]) + d2 w0 a0_j (X(0,kb)[i] + s_j X(1,kb)[i])
        for (int t = tid; t < C::NE * N2; t += NT) {
          const int e = t / N2, q = t % N2, ix = e % TX, iy = e / TX;
          if (ix >= tw || iy >= th) continue;
          const int a = q % NI, b = q / NI;
          const double* d = sD + e * 4;
          const double qp = rq[(e * 2) * N2 + q], qm = NI > 1 ? rq[(e * 2 + 1) * N2 + q] : 0.0;
          const double ub = inb.zf(iy, ix)[q], ut = intp.zf(iy, ix)[q];
          const double sa = (a & 1) ? -1.0 : 1.0, sb = (b & 1) ? -1.0 : 1.0;
          const double dz = d[0] * w0 + (d[1] * sLam[a] + d[2] * sLam[b]) * w0 + d[3] * K00;
          const double c1 = d[1] * w0 * sA0[a], c2 = d[2] * w0 * sA0[b];
          const double pb = dz * ub + d[3] * K0p * ut + c1 * fma(sa, inb.ye(iy, ix + 1)[b], inb.ye(iy, ix)[b]) +
                            c2 * fma(sb, inb.xe(iy + 1, ix)[a], inb.xe(iy, ix)[a]);
          const double pt = dz * ut + d[3] * K0p * ub + c1 * fma(sa, intp.ye(iy, ix + 1)[b], intp.ye(iy, ix)[b]) +
                            c2 * fma(sb, intp.xe(iy + 1, ix)[a], intp.xe(iy, ix)[a]);
          acb.zf(iy, ix)[q] += pb - d[3] * (qp + qm);
          actp.zf(iy, ix)[q] += pt - d[3] * (qp - qm);
        }
        __syncthreads();
        SC_PHASE(4);
#endif
        // ============ even / odd line reductions of faces and edges (primary part) ============
#if !defined(SC_EXP) || SC_EXP != 2
        {
          constexpr int NXR = TY * (TX + 1) * NI, NYR = (TY + 1) * TX * NI, NZR = TY * TX * NI;
          constexpr int NZE = (TY + 1) * (TX + 1), NXE = (TY + 1) * TX, NYE = TY * (TX + 1);
          constexpr int TOT = 2 * NXR + 2 * NYR + 4 * NZR + NZE + 2 * NXE + 2 * NYE;
          for (int t = tid; t < TOT; t += NT) {
            int r = t;
            if (r < 2 * NXR) {                       // x-face (iy, ix): over j (keep k = c) / over k (keep j = c)
              const int dir = r / NXR, rr = r % NXR, c = rr % NI, f = rr / NI;
              const double* F = in.b + C::S_XF + f * N2;
              double* o = rq + (dir == 0 ? C::R_XJ : C::R_XK) + f * 2 * NI;
              eo_reduce<NI>(dir == 0 ? F + NI * c : F + c, dir == 0 ? 1 : NI, sA0, o + 2 * c);
              continue;
            }
            r -= 2 * NXR;
            if (r < 2 * NYR) {                       // y-face (iy, ix): over i (keep k) / over k (keep i)
              const int dir = r / NYR, rr = r % NYR, c = rr % NI, f = rr / NI;
              const double* F = in.b + C::S_YF + f * N2;
              double* o = rq + (dir == 0 ? C::R_YI : C::R_YK) + f * 2 * NI;
              eo_reduce<NI>(dir == 0 ? F + NI * c : F + c, dir == 0 ? 1 : NI, sA0, o + 2 * c);
              continue;
            }
            r -= 2 * NYR;
            if (r < 4 * NZR) {                       // z-face plane kb: over i (keep j) / over j (keep i)
              const int dir = r / (2 * NZR), rr = r % (2 * NZR), kb = rr / NZR, r3 = rr % NZR, c = r3 % NI,
                        f = r3 / NI;
              const double* F = (kb ? intp : inb).b + C::P_ZF + f * N2;
              double* o = rq + (dir == 0 ? C::R_ZI : C::R_ZJ) + (kb * TY * TX + f) * 2 * NI;
              eo_reduce<NI>(dir == 0 ? F + NI * c : F + c, dir == 0 ? 1 : NI, sA0, o + 2 * c);
              continue;
            }
            r -= 4 * NZR;
            if (r < NZE) {                           // z-edges of layer l
              eo_reduce<NI>(in.b + C::S_ZE + r * NI, 1, sA0, rq + C::R_ZE + r * 2);
              continue;
            }
            r -= NZE;
            if (r < 2 * NXE) {                       // x-edges of planes l, l+1
              const int kb = r / NXE, e = r % NXE;
              eo_reduce<NI>((kb ? intp : inb).b + C::P_XE + e * NI, 1, sA0, rq + C::R_XE + r * 2);
              continue;
            }
            r -= 2 * NXE;
            {                                        // y-edges of planes l, l+1
              const int kb = r / NYE, e = r % NYE;
              eo_reduce<NI>((kb ? intp : inb).b + C::P_YE + e * NI, 1, sA0, rq + C::R_YE + r * 2);
            }
          }
        }
        __syncthreads();
        SC_PHASE(5);
#endif
        // ============ primary part Htilde_BB, entity-centric over the tile's elements ============
#if !defined(SC_EXP) || SC_EXP != 2
        // (Mtilde = diag(w0, 1..1, w0); Ktilde arrowhead: row 0 = (K00, a0, K0p),
        //  row p = (K0p, ap, K00), interior row m = (a0_m @0, Lam_m @m, ap_m @p).)
        // Faces: a warp (or a lane group) per face, lanes over the in-face nodes; edges: lane
        // groups of n_I per edge; vertices: a lane each.  Each accumulator entry is owned by
        // exactly one lane, which sums the contributions of the tile's adjacent elements.
        {
          auto present = [&](int ix, int iy) { return ix >= 0 && iy >= 0 && ix < tw && iy < th; };
          auto dd = [&](int ix, int iy) { return sD + (iy * TX + ix) * 4; };
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
              const double* d = dd(ex, ey);
              const double txl = (ib ? K0p : K00) * in.ze(iy, ex)[c] + (ib ? K00 : K0p) * in.ze(iy, ex + 1)[c] +
                                 eo_row(rq + C::R_YI + (iy * TX + ex) * 2 * NI + 2 * c, ib);
              const double tyl = (jb ? K0p : K00) * in.ze(ey, ix)[c] + (jb ? K00 : K0p) * in.ze(ey + 1, ix)[c] +
                                 eo_row(rq + C::R_XJ + (ey * (TX + 1) + ix) * 2 * NI + 2 * c, jb);
              y += d[0] * w02 * u + d[1] * w0 * txl + d[2] * w0 * tyl + d[3] * w02 * tz;
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
              const double* d = dd(ix, ey);
              const double tyl = (jb ? K0p : K00) * pk.xe(ey, ix)[c] + (jb ? K00 : K0p) * pk.xe(ey + 1, ix)[c] +
                                 eo_row(rq + C::R_ZJ + (kb * TY * TX + ey * TX + ix) * 2 * NI + 2 * c, jb);
              y += d[0] * w02 * u + d[1] * w02 * txl + d[2] * w0 * tyl + d[3] * w0 * tzl;
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
              const double* d = dd(ex, iy);
              const double txl = (ib ? K0p : K00) * pk.ye(iy, ex)[c] + (ib ? K00 : K0p) * pk.ye(iy, ex + 1)[c] +
                                 eo_row(rq + C::R_ZI + (kb * TY * TX + iy * TX + ex) * 2 * NI + 2 * c, ib);
              y += d[0] * w02 * u + d[1] * w0 * txl + d[2] * w02 * tyl + d[3] * w0 * tzl;
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
              const double* d = dd(ex, ey);
              const double txl = (ib ? K0p : K00) * *pk.vv(iy, ex) + (ib ? K00 : K0p) * *pk.vv(iy, ex + 1) +
                                 eo_row(rq + C::R_XE + (kb * (TY + 1) * TX + iy * TX + ex) * 2, ib);
              const double tyl = (jb ? K0p : K00) * *pk.vv(ey, ix) + (jb ? K00 : K0p) * *pk.vv(ey + 1, ix) +
                                 eo_row(rq + C::R_YE + (kb * TY * (TX + 1) + ey * (TX + 1) + ix) * 2, jb);
              y += d[0] * w02 * w0 * u + w02 * (d[1] * txl + d[2] * tyl + d[3] * tzl);
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

template <int NI, bool U>
static int launch_col_u(const ColParams& P, cudaStream_t st, int* nl, int* grid_out) {
  using C = CS<NI>;
  const size_t smem = sizeof(double) * C::TOTAL;
  static int max_active = -1, nsm = 0;
  if (max_active < 0) {
    cudaFuncSetAttribute(k_apply_col<NI, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_active, k_apply_col<NI, U>, C::NT, smem);
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (max_active < 1) max_active = 1;
  }
  int grid = max_active * nsm;
  if (grid > P.nitems) grid = P.nitems;
  *grid_out = grid;
  k_apply_col<NI, U><<<grid, C::NT, smem, st>>>(P);
  (*nl)++;
  return cudaGetLastError();
}

template <int NI>
static int launch_col_t(const ColParams& P, cudaStream_t st, int* nl, int* grid_out) {
  return P.g.dinv ? launch_col_u<NI, true>(P, st, nl, grid_out) : launch_col_u<NI, false>(P, st, nl, grid_out);
}

#if defined(SC_EXP) && SC_EXP == 9
extern "C" int sc_exp_phase_cycles(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 16);
}
#endif

bool col_supported(int ni) { return ni >= 1 && ni <= 8; }

void col_tile(int ni, int* tx, int* ty, int* pend) {
  switch (ni) {
#define TCASE(N) case N: *tx = CS<N>::TX; *ty = CS<N>::TY; *pend = CS<N>::PEND; return;
    TCASE(1) TCASE(2) TCASE(3) TCASE(4) TCASE(5) TCASE(6) TCASE(7) TCASE(8)
#undef TCASE
    default: *tx = *ty = *pend = 0;
  }
}

int launch_apply_col(const ColParams& P, void* stream, int* nl, int* grid_out, void* events);

int launch_apply_col_raw(const Geom& g, const double* x, double* y, const double* done, void* state, int* flags,
                         double* corner, double* pending, int ntx, int nty, void* stream, int* nl, void* events) {
  ColParams P;
  P.g = g; P.x = x; P.y = y; P.done = done; P.st = (ColState*)state; P.flags = flags; P.corner = corner;
  P.pending = pending;
  P.ntx = ntx; P.nty = nty; P.nitems = ntx * nty;
  int grid = 0;
  return launch_apply_col(P, stream, nl, &grid, events);
}

int launch_apply_col(const ColParams& P, void* stream, int* nl, int* grid_out, void* events) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  if (ev) cudaEventRecord(ev[0], st);
  int r;
  switch (P.g.ni) {
#define LCASE(N) case N: r = launch_col_t<N>(P, st, nl, grid_out); break;
    LCASE(1) LCASE(2) LCASE(3) LCASE(4) LCASE(5) LCASE(6) LCASE(7) LCASE(8)
#undef LCASE
    default: return cudaErrorInvalidValue;
  }
  if (ev) cudaEventRecord(ev[1], st);
  return r;
}

}  // namespace sc
