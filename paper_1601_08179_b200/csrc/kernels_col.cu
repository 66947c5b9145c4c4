// Condensed operator v3 (rows a3-a8 of SURVEY §8(a)): tile-column kernel, parity-class warps.
//
// Work decomposition.  The slab's elements are cut into xy-tiles of TX x TY = 8 x 4 elements;
// a work item is one tile-column (all nz element layers of the tile).  A persistent CTA (one
// per SM, 8 warps) takes items in ticket order and marches up the column one element layer at
// a time.  Every entity of the skeleton is assembled on chip except those on tile side
// boundaries, which are finished with a decoupled look-back (distance kLB = 3): the lower-ticket contributor
// stores its partial sum straight into y (or, on the 4-tile corner lines, into a small corner
// record), publishes a per-(item, layer) flag, and the owner (highest-ticket contributor) adds
// it and writes the final value two steps later.  Every skeleton entry is written exactly once
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
#include <stdint.h>
#include <stdlib.h>
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
  unsigned long long* prog;   // [nitems] publication progress: (epoch << 32) | (last published step + 1)
  double* corner;        // [(nty+1)][(ntx+1)][nz+1][3][NI+1]
  double* pending;       // [nitems][2][PEND]
  int ntx, nty, nitems;  // nitems = ntx nty nseg (item = seg * ntx nty + tile)
  int nseg, zseg;        // z-segments of a tile column: element layers [s zseg, min(nz, (s+1) zseg))
  double* dotp;          // optional: per-item partial sums of x . y over final entries [nitems]
  ColCoef cf;
};

// decoupled look-back distance: a tile finishes its W / S boundary entities of step l - kLB at
// step l (neighbours publish step l - kLB at their step l - kLB + 1: kLB - 1 steps of slack);
// own partials are parked in kSlots = kLB + 1 rotating slots
#ifndef SC_KLB
#define SC_KLB 3
#endif
constexpr int kLB = SC_KLB, kSlots = kLB + 1;
template <int NI>
struct CS {
  static constexpr int N2 = NI * NI;
  static constexpr int NT = 256;                      // 8 warps = 8 parity classes
  // tile: 8 x 4 elements (one per lane, a parity class per warp) for n_I >= 4; for n_I <= 3
  // one element per thread (all classes in the thread) on larger tiles: 16 x 16 (n_I = 1),
  // 16 x 8 (n_I = 2, 3; the largest that fits the shared-memory budget at n_I = 3)
  static constexpr bool PER_ELEM = NI <= 3;
  // entry-per-thread loads / finalize (short rows) for n_I <= 2; row per warp (4 predicated
  // accesses per lane and pass) from n_I = 3 on (measured: p=4 4.56 -> 3.47 ms, p=3 3.70 vs 3.78)
  static constexpr bool FLAT_IO = NI <= 2;
  static constexpr int TX = NI <= 3 ? 16 : 8, TY = NI == 1 ? 16 : (NI <= 3 ? 8 : 4), NE = TX * TY;
  static constexpr int MAXROWS = 7 * TY + 4;          // row descriptors per tile
  // row strides of the x-face and z-edge blocks (doubles): padded to 8 mod 16 for the class
  // warps (lane (ix, iy) at iy RS + ix N2: the two element rows of a half-warp then fall on
  // disjoint bank pairs -- unpadded, 64-bit accesses to x-faces were 2-way conflicted)
  static constexpr int pad8(int v) { return PER_ELEM ? v : v + ((8 - v % 16) + 16) % 16; }
  static constexpr int XRS = pad8((TX + 1) * N2), ZRS = pad8((TX + 1) * NI);
  static constexpr int XF = TY * XRS;
  static constexpr int YF = (TY + 1) * TX * N2;
  static constexpr int ZE = (TY + 1) * ZRS;
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
  static constexpr int O_IP = O_IS + 2 * SIDE;       // 3 plane input buffers (plane q in q % 3)
  static constexpr int O_AS = O_IP + 3 * PLANE;      // side accumulator
  static constexpr int O_AP = O_AS + SIDE;           // 2 plane accumulators
  static constexpr int O_RQ = O_AP + 2 * PLANE;      // reduction buffers
  static constexpr int O_TAB = O_RQ + RED;           // a0, lam (2 x 32)
  static constexpr int O_CF = O_TAB + 2 * 32;        // ColCoef copy
  static constexpr int TOTAL = O_CF + (int)(sizeof(ColCoef) / sizeof(double));
  // parked own partials of the W / S boundary entities (global, per tile, LB + 1 step slots)
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
  __device__ double* xf(int iy, int ix) const { return b + CS<NI>::S_XF + iy * CS<NI>::XRS + ix * CS<NI>::N2; }
  __device__ double* yf(int iy, int ix) const { return b + CS<NI>::S_YF + (iy * CS<NI>::TX + ix) * CS<NI>::N2; }
  __device__ double* ze(int iy, int ix) const { return b + CS<NI>::S_ZE + iy * CS<NI>::ZRS + ix * NI; }
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
__device__ unsigned long long g_phase_cycles[8 * 16];   // [warp][phase]
#define SC_PHASE(k)                                                                         \
  do {                                                                                      \
    if ((threadIdx.x & 31) == 0) {                                                          \
      long long t_ = clock64();                                                             \
      atomicAdd(&g_phase_cycles[(threadIdx.x >> 5) * 16 + (k)], (unsigned long long)(t_ - ph_t0)); \
      ph_t0 = t_;                                                                           \
    }                                                                                       \
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

__device__ __forceinline__ void prog_release(unsigned long long* f, unsigned long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(f), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long prog_acquire(const unsigned long long* f) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
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

// ---- row-structured I/O ----------------------------------------------------------------
// Every tile row of an entity class is one contiguous range in both the skeleton vector and
// the shared-memory buffer.  Rows are dealt to the 8 warps round-robin; a warp moves a row with
// one 8-byte cp.async per lane and iteration (Dirichlet sub-ranges are written as 0), so the
// per-entry cost is an address increment, a compare and the copy.
__device__ __forceinline__ void cp8(unsigned s, const double* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void row_load(double* sb, const double* gb, int len, int zlo, int zhi, int lane) {
  for (int t = lane; t < zlo; t += 32) sb[t] = 0.0;
  for (int t = zhi + lane; t < len; t += 32) sb[t] = 0.0;
  const unsigned s0 = (unsigned)__cvta_generic_to_shared(sb + zlo);
  const double* g0 = gb + zlo;
  const int cnt = zhi - zlo;
  if (cnt > 8 && ((s0 ^ (unsigned)reinterpret_cast<uintptr_t>(g0)) & 15u) == 0) {
    // both sides at the same 16-byte phase: an 8-byte head if needed, then 16-byte copies
    const int h = (s0 & 15u) ? 1 : 0, npair = (cnt - h) >> 1;
    if (h && lane == 0) cp8(s0, g0);
    if (((cnt - h) & 1) && lane == 1) cp8(s0 + 8u * (cnt - 1), g0 + cnt - 1);
    unsigned s = s0 + 8u * h + 16u * lane;
    const double* gp = g0 + h + 2 * lane;
    for (int n = npair - lane; n > 0; n -= 64, s += 1024u, gp += 128) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gp) : "memory");
      if (n > 32) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s + 512u), "l"(gp + 64) : "memory");
    }
    return;
  }
  unsigned s = s0 + 8u * lane;
  const double* gp = g0 + lane;
  for (int n = cnt - lane; n > 0; n -= 128, s += 1024u, gp += 128) {   // predicated 4-wide, no tail loop
    cp8(s, gp);
    if (n > 32) cp8(s + 256u, gp + 32);
    if (n > 64) cp8(s + 512u, gp + 64);
    if (n > 96) cp8(s + 768u, gp + 96);
  }
}

// Row descriptors of a tile (built once per work item, shared memory).  Rows of the side
// (element layer) block: x-faces (th), y-faces (th+1), z-edges (th+1); rows of the plane block:
// z-faces (th), x-edges (th+1), y-edges (th), vertices (th+1).  The skeleton offset of a row at
// layer / plane l is g + l gs.  Load: [0, zlo) and [zhi, len) are Dirichlet entries (written as
// 0).  Finalize: W end [0, a), middle [a, b), E end [b, len), each with a mode (copy to y, zero,
// park in `pending` at offset p + c, or skip = published by the corner pass).
enum { M_SKIP = 0, M_Y = 1, M_ZERO = 2, M_PARK = 3 };
struct RowIO {
  long long g, gs;
  int s, len, zlo, zhi;
  short a, b, pw, pm;
  unsigned char mw, mm, me, pub;   // pub: bit 1 middle, bit 2 E end are published partials (not final)
};

template <int NI>
__device__ void build_rows(const ColParams& P, RowIO* io, int x0, int y0, int tw, int th, int* ns_out) {
  using C = CS<NI>;
  constexpr int N2 = NI * NI, TX = C::TX;
  const Geom& g = P.g;
  const int nx = g.nx, ny = g.ny;
  const bool hasW = x0 > 0, hasE = x0 + tw < nx, hasS = y0 > 0, hasN = y0 + th < ny;
  const int ns = 3 * th + 2, np = 4 * th + 2;
  *ns_out = ns;
  for (int r = threadIdx.x; r < ns + np; r += CS<NI>::NT) {
  RowIO d;
  d.a = 0; d.pw = 0; d.pm = 0; d.mw = M_SKIP; d.me = M_SKIP; d.pub = 0;
  if (r < th) {                                            // x-faces row r
    d.g = g.off_f[0] + ((long long)x0 + (long long)(nx + 1) * (y0 + r)) * N2;
    d.gs = (long long)(nx + 1) * ny * N2;
    d.s = C::S_XF + r * C::XRS; d.len = (tw + 1) * N2;
    d.zlo = hasW ? 0 : N2; d.zhi = hasE ? d.len : tw * N2;
    d.a = N2; d.b = tw * N2;
    d.mw = hasW ? M_PARK : M_ZERO; d.pw = C::PD_XF + r * N2; d.mm = M_Y; d.me = hasE ? M_Y : M_ZERO;
    d.pub = hasE ? 4 : 0;
  } else if (r < 2 * th + 1) {                             // y-faces row q
    const int q = r - th, fy = y0 + q;
    const bool z = fy == 0 || fy == ny;
    d.g = g.off_f[1] + ((long long)x0 + (long long)nx * fy) * N2;
    d.gs = (long long)nx * (ny + 1) * N2;
    d.s = C::S_YF + q * TX * N2; d.len = tw * N2;
    d.zlo = z ? d.len : 0; d.zhi = d.len;
    d.b = d.len;
    d.mm = z ? M_ZERO : ((q == 0 && hasS) ? M_PARK : M_Y); d.pm = C::PD_YF;
    d.pub = (q == th && hasN) ? 2 : 0;
  } else if (r < ns) {                                     // z-edges row q
    const int q = r - 2 * th - 1, fy = y0 + q;
    const bool z = fy == 0 || fy == ny, nrow = q == th && hasN, srow = q == 0 && hasS;
    d.g = g.off_e[2] + ((long long)x0 + (long long)(nx + 1) * fy) * NI;
    d.gs = (long long)(nx + 1) * (ny + 1) * NI;
    d.s = C::S_ZE + q * C::ZRS; d.len = (tw + 1) * NI;
    d.zlo = z ? d.len : (hasW ? 0 : NI); d.zhi = hasE ? d.len : tw * NI;
    d.a = NI; d.b = tw * NI;
    d.mw = z ? M_ZERO : (nrow ? M_SKIP : (hasW ? M_PARK : M_ZERO)); d.pw = C::PD_ZEW + q * NI;
    d.mm = z ? M_ZERO : (srow ? M_PARK : M_Y); d.pm = C::PD_ZES - NI;
    d.me = (z || !hasE) ? M_ZERO : ((nrow || srow) ? M_SKIP : M_Y);
    d.pub = (nrow ? 2 : 0) | (hasE ? 4 : 0);
  } else {
    const int u = r - ns;
    if (u < th) {                                          // z-faces row u
      d.g = g.off_f[2] + ((long long)x0 + (long long)nx * (y0 + u)) * N2;
      d.gs = (long long)nx * ny * N2;
      d.s = C::P_ZF + u * TX * N2; d.len = tw * N2;
      d.zlo = 0; d.zhi = d.len; d.b = d.len; d.mm = M_Y;
    } else if (u < 2 * th + 1) {                           // x-edges row q
      const int q = u - th, fy = y0 + q;
      const bool z = fy == 0 || fy == ny;
      d.g = g.off_e[0] + ((long long)x0 + (long long)nx * fy) * NI;
      d.gs = (long long)nx * (ny + 1) * NI;
      d.s = C::P_XE + q * TX * NI; d.len = tw * NI;
      d.zlo = z ? d.len : 0; d.zhi = d.len; d.b = d.len;
      d.mm = z ? M_ZERO : ((q == 0 && hasS) ? M_PARK : M_Y); d.pm = C::PD_XE;
      d.pub = (q == th && hasN) ? 2 : 0;
    } else if (u < 3 * th + 1) {                           // y-edges row q
      const int q = u - 2 * th - 1;
      d.g = g.off_e[1] + ((long long)x0 + (long long)(nx + 1) * (y0 + q)) * NI;
      d.gs = (long long)(nx + 1) * ny * NI;
      d.s = C::P_YE + q * (TX + 1) * NI; d.len = (tw + 1) * NI;
      d.zlo = hasW ? 0 : NI; d.zhi = hasE ? d.len : tw * NI;
      d.a = NI; d.b = tw * NI;
      d.mw = hasW ? M_PARK : M_ZERO; d.pw = C::PD_YE + q * NI; d.mm = M_Y; d.me = hasE ? M_Y : M_ZERO;
      d.pub = hasE ? 4 : 0;
    } else {                                               // vertices row q
      const int q = u - 3 * th - 1, fy = y0 + q;
      const bool z = fy == 0 || fy == ny, nrow = q == th && hasN, srow = q == 0 && hasS;
      d.g = g.off_v + (long long)x0 + (long long)(nx + 1) * fy;
      d.gs = (long long)(nx + 1) * (ny + 1);
      d.s = C::P_VV + q * (TX + 1); d.len = tw + 1;
      d.zlo = z ? d.len : (hasW ? 0 : 1); d.zhi = hasE ? d.len : tw;
      d.a = 1; d.b = tw;
      d.mw = z ? M_ZERO : (nrow ? M_SKIP : (hasW ? M_PARK : M_ZERO)); d.pw = C::PD_VW + q;
      d.mm = z ? M_ZERO : (srow ? M_PARK : M_Y); d.pm = C::PD_VS - 1;
      d.me = (z || !hasE) ? M_ZERO : ((nrow || srow) ? M_SKIP : M_Y);
      d.pub = (nrow ? 2 : 0) | (hasE ? 4 : 0);
    }
  }
  io[r] = d;
  }
}

// Rows [r0, r1) of the descriptor table into the block at `base` for layer / plane l (one warp
// per row); zero_all: the whole block is Dirichlet (a Dirichlet z-plane).
__device__ __forceinline__ void load_rows(const double* x, const RowIO* io, int r0, int r1, double* base, int l,
                                          bool zero_all) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = r0 + warp; r < r1; r += 8) {
    const RowIO& d = io[r];
    const int len = d.len;
    row_load(base + d.s, x + d.g + (long long)l * d.gs, len, zero_all ? len : d.zlo, d.zhi, lane);
  }
}

// Flat view of a side / plane block for the small-n_I tiles (short rows: one warp per row
// leaves most lanes idle): block entry t -> descriptor row and column (compile-time strides),
// -1 for padding rows.  The shared-memory position of an entry is the block base + t.
template <int NI>
__device__ __forceinline__ int flat_row(int t, bool plane, int th, int ns, int& col) {
  using C = CS<NI>;
  constexpr int N2 = C::N2, TX = C::TX;
  int q;
  if (!plane) {
    if (t < C::XF) { q = t / ((TX + 1) * N2); col = t - q * ((TX + 1) * N2); return q < th ? q : -1; }
    t -= C::XF;
    if (t < C::YF) { q = t / (TX * N2); col = t - q * (TX * N2); return q <= th ? th + q : -1; }
    t -= C::YF;
    q = t / ((TX + 1) * NI); col = t - q * ((TX + 1) * NI); return q <= th ? 2 * th + 1 + q : -1;
  }
  if (t < C::PZF) { q = t / (TX * N2); col = t - q * (TX * N2); return q < th ? ns + q : -1; }
  t -= C::PZF;
  if (t < C::PXE) { q = t / (TX * NI); col = t - q * (TX * NI); return q <= th ? ns + th + q : -1; }
  t -= C::PXE;
  if (t < C::PYE) { q = t / ((TX + 1) * NI); col = t - q * ((TX + 1) * NI); return q < th ? ns + 2 * th + 1 + q : -1; }
  t -= C::PYE;
  q = t / (TX + 1); col = t - q * (TX + 1); return q <= th ? ns + 3 * th + 1 + q : -1;
}

// Side (plane == false) or plane block of layer / plane l into `base`: rows [0, ns) or
// [ns, ns + 4 th + 2) of the descriptor table; zero_all: a Dirichlet z-plane.
template <int NI>
__device__ __forceinline__ void load_block(const double* x, const RowIO* io, bool plane, int ns, int th, double* base,
                                           int l, bool zero_all) {
  using C = CS<NI>;
  if constexpr (C::FLAT_IO) {
    const int nb = plane ? C::PLANE : C::SIDE;
    for (int t = threadIdx.x; t < nb; t += C::NT) {
      int col;
      const int r = flat_row<NI>(t, plane, th, ns, col);
      if (r < 0) continue;
      const RowIO& d = io[r];
      if (col >= d.len) continue;
      if (zero_all || col < d.zlo || col >= d.zhi) base[t] = 0.0;
      else cp_async8(base + t, x + d.g + (long long)l * d.gs + col);
    }
  } else {
    if (plane) load_rows(x, io, ns, ns + 4 * th + 2, base, l, zero_all);
    else load_rows(x, io, 0, ns, base, l, zero_all);
  }
}

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

// Segment [a, b) of a shared-memory row to a global row: mode 0 skip, 1 copy, 2 zero.
__device__ __forceinline__ void seg_out(double* __restrict__ dst, const double* __restrict__ s, int a, int b, int mode,
                                        int lane) {
  if (mode == 1) {
    // 4 predicated loads in flight before the stores; one pass covers any segment of <= 128
    // entries (most segments: face / edge ends and edge rows), no scalar tail loop
    const double* sp = s + a + lane;
    double* dp = dst + a + lane;
    for (int n = b - a - lane; n > 0; n -= 128, sp += 128, dp += 128) {
      const double v0 = sp[0];
      const double v1 = n > 32 ? sp[32] : 0.0, v2 = n > 64 ? sp[64] : 0.0, v3 = n > 96 ? sp[96] : 0.0;
      dp[0] = v0;
      if (n > 32) dp[32] = v1;
      if (n > 64) dp[64] = v2;
      if (n > 96) dp[96] = v3;
    }
  } else if (mode == 2) {
    for (int t = a + lane; t < b; t += 32) dst[t] = 0.0;
  }
}
enum { SEG_SKIP = 0, SEG_COPY = 1, SEG_ZERO = 2 };

// ---- finalize step l: write every entity of the step that this tile completes or publishes.
// Ownership: the highest-ticket contributing tile (tiles are ticketed x-fastest) owns an
// entity.  A tile owns its W / S boundaries: its own partials are parked in `pending` and
// finished one step later.  It publishes its E / N boundaries as partial sums straight into y,
// except the three 4-tile corner lines it does not own, whose partials go to corner records.
// Segments per row: W end | middle | E end, each copied, zeroed (Dirichlet), parked or skipped.
__device__ __forceinline__ void seg_mode(double* yo, double* pk, const double* s, int a, int b, int mode, int lane) {
  if (mode == M_Y) seg_out(yo, s, a, b, SEG_COPY, lane);
  else if (mode == M_ZERO) seg_out(yo, s, a, b, SEG_ZERO, lane);
  else if (mode == M_PARK) seg_out(pk, s, a, b, SEG_COPY, lane);
}
// Final entries: copy to y and accumulate x . y (x = the operator's input, same row layout).
__device__ __forceinline__ double seg_final(double* __restrict__ dst, const double* __restrict__ s,
                                            const double* __restrict__ xs, int a, int b, int lane) {
  double acc = 0.0;
  int t = a + lane;
  for (; t + 96 < b; t += 128) {
    const double v0 = s[t], v1 = s[t + 32], v2 = s[t + 64], v3 = s[t + 96];
    const double u0 = xs[t], u1 = xs[t + 32], u2 = xs[t + 64], u3 = xs[t + 96];
    dst[t] = v0; dst[t + 32] = v1; dst[t + 64] = v2; dst[t + 96] = v3;
    acc = fma(v0, u0, acc); acc = fma(v1, u1, acc); acc = fma(v2, u2, acc); acc = fma(v3, u3, acc);
  }
  for (; t < b; t += 32) {
    const double v = s[t];
    dst[t] = v;
    acc = fma(v, xs[t], acc);
  }
  return acc;
}

// Finalize of layer l (side rows, when side == true) and plane l (plane rows): accumulators
// ac / acb, the operator's input of the same layer / plane in xin / xinb (for x . y).
template <int NI>
__device__ void finalize_step(const ColParams& P, long long item, int l, int x0, int y0, int tw, int th,
                              const Side<NI>& ac, const Plane<NI>& acb, const Side<NI>& xin, const Plane<NI>& xinb,
                              const RowIO* io, int ns, bool side_rows, double& dot) {
  using C = CS<NI>;
  constexpr int NW = C::NT / 32, TX = C::TX, TY = C::TY;
  const Geom& g = P.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool last = !side_rows, pzd = zdir(g, l);
  const int x1 = x0 + tw, y1 = y0 + th;
  const bool hasE = x1 < g.nx, hasN = y1 < g.ny, hasW = x0 > 0, hasS = y0 > 0;
  double* const pd = P.pending + (item * kSlots + l % kSlots) * (long long)C::PEND;
  const bool want_dot = P.dotp != nullptr;
  const int nr = ns + 4 * th + 2;
  if constexpr (C::FLAT_IO) {
    // flat: every thread takes block entries t, t + NT, ... (side block, then plane block);
    // all values are read before any store
    constexpr int NF = (C::SIDE + C::PLANE + C::NT - 1) / C::NT;
    double val[NF], xv[NF];
    double* dst[NF];
#pragma unroll
    for (int k = 0; k < NF; ++k) {
      dst[k] = nullptr;
      val[k] = xv[k] = 0.0;
      const int t = (last ? C::SIDE : 0) + (int)threadIdx.x + k * C::NT;
      if (t >= C::SIDE + C::PLANE) continue;
      const bool side = t < C::SIDE;
      const int tb = side ? t : t - C::SIDE;
      int col;
      const int r = flat_row<NI>(tb, !side, th, ns, col);
      if (r < 0) continue;
      const RowIO& d = io[r];
      if (col >= d.len) continue;
      double* yo = P.y + d.g + (long long)l * d.gs + col;
      const double s = (side ? ac.b : acb.b)[tb];
      if (!side && pzd) { dst[k] = yo; continue; }
      int mode, bit, po;
      if (col < d.a) { mode = d.mw; bit = 0; po = d.pw; }
      else if (col < d.b) { mode = d.mm; bit = 2; po = d.pm; }
      else { mode = d.me; bit = 4; po = 0; }
      if (mode == M_SKIP) continue;
      if (mode == M_PARK) { dst[k] = pd + po + col; val[k] = s; continue; }
      dst[k] = yo;
      if (mode == M_Y) {
        val[k] = s;
        if (want_dot && bit && !(d.pub & bit)) xv[k] = (side ? xin.b : xinb.b)[tb];
      }
    }
#pragma unroll
    for (int k = 0; k < NF; ++k)
      if (dst[k]) {
        *dst[k] = val[k];
        dot = fma(val[k], xv[k], dot);
      }
  } else
  for (int r = (last ? ns : 0) + warp; r < nr; r += NW) {
    const RowIO& d = io[r];
    const bool side = r < ns;
    const double* s = (side ? ac.b : acb.b) + d.s;
    const double* xs = (side ? xin.b : xinb.b) + d.s;
    double* yo = P.y + d.g + (long long)l * d.gs;
    if (!side && pzd) { seg_out(yo, s, 0, d.len, SEG_ZERO, lane); continue; }
    seg_mode(yo, pd + d.pw, s, 0, d.a, d.mw, lane);
    if (want_dot && d.mm == M_Y && !(d.pub & 2)) dot += seg_final(yo, s, xs, d.a, d.b, lane);
    else seg_mode(yo, pd + d.pm, s, d.a, d.b, d.mm, lane);
    if (want_dot && d.me == M_Y && !(d.pub & 4)) dot += seg_final(yo, s, xs, d.b, d.len, lane);
    else seg_mode(yo, pd, s, d.b, d.len, d.me, lane);
  }
  // corner pass: the three 4-tile corner lines this tile contributes to but does not own
  // (NE -> slot 0 of the NE tile's SW corner, NW -> slot 1, SE -> slot 2); z-edges (c < NI)
  // of layer l and the vertex (c == NI) of plane l.
  if (warp == NW - 1) {
    const int cc = lane % (NI + 1), kind = lane / (NI + 1);
    if (kind < 3) {
      const bool isv = cc == NI;
      int ix = 0, iy = 0, slot = -1;
      if (kind == 0 && hasE && hasN) { ix = tw; iy = th; slot = 0; }
      if (kind == 1 && hasW && hasN) { ix = 0; iy = th; slot = 1; }
      if (kind == 2 && hasE && hasS) { ix = tw; iy = 0; slot = 2; }
      if (slot >= 0 && !(isv ? pzd : last)) {
        const double v = isv ? *acb.vv(iy, ix) : ac.ze(iy, ix)[cc];
        corner_rec(P, (x0 + ix) / TX, (y0 + iy) / TY, l, slot)[cc] = v;
      }
    }
  }
}

// Deferred look-back for step ls of tile item: wait for the W, S, SW tiles' flags of step ls
// (one lane per flag), then write the tile's W / S boundary entities of that step as own
// (parked) partial + the neighbours' partials (y-in-place, or the corner records on the 4-tile
// corner line).  Row base addresses of the step are built once in shared memory; every
// thread then issues all of its loads before any store.  Dirichlet entities were written as 0
// in the finalize pass and are skipped.
// Prologue of the look-back for step ls (warp 0): acquire the W, S, SW tiles' flags of step ls
// (one lane per flag) and build the step's row base addresses in shared memory; the CTA barrier
// that follows orders every thread's data loads after the acquire.  (Hoisting it to the top of
// step ls + kLB measured slower: the acquire then delays the step's load barrier.)
template <int NI>
__device__ __forceinline__ void finish_prepare(const ColParams& P, int ls, int th, const unsigned long long* flag_w,
                                               const unsigned long long* flag_s, const unsigned long long* flag_sw,
                                               int epoch, long long* sRow, const RowIO* io, unsigned long long* sKnown) {
  using C = CS<NI>;
  constexpr int TY = C::TY;
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int lane = tid;
    if (lane < 3) {
      // neighbour progress words: one acquire usually reveals several published steps, which
      // later look-backs then need not reload (the earlier acquire already orders our loads)
      const unsigned long long* f = lane == 0 ? flag_w : (lane == 1 ? flag_s : flag_sw);
      const unsigned long long need = ((unsigned long long)(unsigned)epoch << 32) | (unsigned)(ls + 1);
#if defined(SC_EXP) && SC_EXP == 27
      (void)f; (void)need;                                              // ablation: no wait
#else
      if (f && sKnown[lane] < need) {
        unsigned long long v;
        while ((v = prog_acquire(f)) < need) __nanosleep(32);
        sKnown[lane] = v;
      }
#endif
    }
    // row bases from the descriptor table (x-face rows 0.., y-face row 0 at th, z-edge rows at
    // 2 th + 1, x-edge row 0 at ns + th, y-edge rows at ns + 2 th + 1, vertex rows at ns + 3 th + 1)
    const int ns = 3 * th + 2;
    auto at = [&](int r) { return io[r].g + (long long)ls * io[r].gs; };
    if (lane < TY + 1) {
      if (lane < th) sRow[lane] = at(lane), sRow[2 * TY + 1 + lane] = at(ns + 2 * th + 1 + lane);
      if (lane <= th) sRow[TY + lane] = at(2 * th + 1 + lane), sRow[3 * TY + 1 + lane] = at(ns + 3 * th + 1 + lane);
    }
    if (lane == 0) {
      sRow[4 * TY + 2] = at(th);
      sRow[4 * TY + 3] = at(2 * th + 1);
      sRow[4 * TY + 4] = at(ns + th);
      sRow[4 * TY + 5] = at(ns + 3 * th + 1);
    }
  }
}

template <int NI>
__device__ void finish_gather(const ColParams& P, long long item, int ls, int x0, int y0, int tw, int th,
                              const unsigned long long* flag_w, const unsigned long long* flag_s,
                              const unsigned long long* flag_sw, int epoch, long long* sRow, const RowIO* io,
                              unsigned long long* sKnown, double (&val)[(CS<NI>::PEND + CS<NI>::NT - 1) / CS<NI>::NT],
                              double* (&dst)[(CS<NI>::PEND + CS<NI>::NT - 1) / CS<NI>::NT]) {
  using C = CS<NI>;
  constexpr int N2 = C::N2, NT = C::NT, TX = C::TX, TY = C::TY;
  constexpr int MAXE = (C::PEND + NT - 1) / NT;
  const Geom& g = P.g;
  Addr A{g};
  const int tid = threadIdx.x;
  const bool last = (ls == g.nz), pzd = zdir(g, ls);
  const int x1 = x0 + tw, y1 = y0 + th;
  const bool hasN = y1 < g.ny, hasW = x0 > 0, hasS = y0 > 0;
  (void)x1;
  if (!hasW && !hasS) return;
  // row bases: [0, th) W col x-faces, [TY, TY+th] W col z-edges, [2TY+1, 2TY+1+th) W col y-edges,
  // [3TY+1, 3TY+1+th] W col vertices, 4TY+2: S row y-faces, +1 S row z-edges, +2 S row x-edges,
  // +3 S row vertices
  finish_prepare<NI>(P, ls, th, flag_w, flag_s, flag_sw, epoch, sRow, io, sKnown);
  __syncthreads();
  const double* pd = P.pending + (item * kSlots + ls % kSlots) * (long long)C::PEND;
  // segment sizes of the flat list (0 when the segment does not apply at this step)
  const int n0 = (!last && hasW) ? th * N2 : 0;            // W col x-faces
  const int n1 = (!last && hasS) ? tw * N2 : 0;            // S row y-faces
  const int n2 = (!last && hasW) ? (th + 1) * NI : 0;      // W col z-edges
  const int n3 = (!last && hasS) ? (tw - 1) * NI : 0;      // S row z-edges, ix in [1, tw-1]
  const int n4 = (!pzd && hasS) ? tw * NI : 0;             // S row x-edges
  const int n5 = (!pzd && hasW) ? th * NI : 0;             // W col y-edges
  const int n6 = (!pzd && hasW) ? th + 1 : 0;              // W col vertices
  const int n7 = (!pzd && hasS) ? tw - 1 : 0;              // S row vertices, ix in [1, tw-1]
  const int c1 = n0, c2 = c1 + n1, c3 = c2 + n2, c4 = c3 + n3, c5 = c4 + n4, c6 = c5 + n5, c7 = c6 + n6;
  const int ntot = c7 + n7;
#pragma unroll
  for (int k = 0; k < MAXE; ++k) {
    dst[k] = nullptr;
    val[k] = 0.0;
    const int t = tid + k * NT;
    if (t >= ntot) continue;
    long long o;
    int po, corner = -1;
    if (t < c1) {
      const int row = t / N2;
      o = sRow[row] + (t - row * N2); po = C::PD_XF + t;
    } else if (t < c2) {
      o = sRow[4 * TY + 2] + (t - c1); po = C::PD_YF + (t - c1);
    } else if (t < c3) {
      const int u = t - c2, row = u / NI, fy = y0 + row;
      if (fy == 0 || fy == g.ny || (row == th && hasN)) continue;
      o = sRow[TY + row] + (u - row * NI); po = C::PD_ZEW + u;
      if (row == 0 && hasS) corner = u;
    } else if (t < c4) {
      o = sRow[4 * TY + 3] + NI + (t - c3); po = C::PD_ZES + (t - c3);
    } else if (t < c5) {
      o = sRow[4 * TY + 4] + (t - c4); po = C::PD_XE + (t - c4);
    } else if (t < c6) {
      const int u = t - c5, row = u / NI;
      o = sRow[2 * TY + 1 + row] + (u - row * NI); po = C::PD_YE + u;
    } else if (t < c7) {
      const int row = t - c6, fy = y0 + row;
      if (fy == 0 || fy == g.ny || (row == th && hasN)) continue;
      o = sRow[3 * TY + 1 + row]; po = C::PD_VW + row;
      if (row == 0 && hasS) corner = NI;
    } else {
      o = sRow[4 * TY + 5] + 1 + (t - c7); po = C::PD_VS + (t - c7);
    }
    double* d = P.y + o;
#if defined(SC_EXP) && SC_EXP == 28
    val[k] = 0.0; dst[k] = d; (void)pd; (void)po; (void)corner; continue;   // ablation: no gather loads
#endif
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
}

// Second half of the look-back: x . y partials (fused dot only) and the stores.  The values
// were gathered before the step's finalize, so their load latency overlaps it.
template <int NI>
__device__ __forceinline__ void finish_scatter(const ColParams& P, const double (&val)[(CS<NI>::PEND + CS<NI>::NT - 1) / CS<NI>::NT],
                                               double* const (&dst)[(CS<NI>::PEND + CS<NI>::NT - 1) / CS<NI>::NT],
                                               double& dot) {
  constexpr int MAXE = (CS<NI>::PEND + CS<NI>::NT - 1) / CS<NI>::NT;
  double xv[MAXE];
#pragma unroll
  for (int k = 0; k < MAXE; ++k) xv[k] = (dst[k] && P.dotp) ? ld_cg(P.x + (dst[k] - P.y)) : 0.0;
#pragma unroll
  for (int k = 0; k < MAXE; ++k)
    if (dst[k]) {
      *dst[k] = val[k];
      dot = fma(val[k], xv[k], dot);
    }
}

template <int NI>
__device__ void finish_boundary(const ColParams& P, long long item, int ls, int x0, int y0, int tw, int th,
                                const unsigned long long* flag_w, const unsigned long long* flag_s,
                                const unsigned long long* flag_sw, int epoch, long long* sRow, const RowIO* io,
                                unsigned long long* sKnown, double& dot) {
  constexpr int MAXE = (CS<NI>::PEND + CS<NI>::NT - 1) / CS<NI>::NT;
  double val[MAXE];
  double* dst[MAXE];
#pragma unroll
  for (int k = 0; k < MAXE; ++k) { val[k] = 0.0; dst[k] = nullptr; }
  finish_gather<NI>(P, item, ls, x0, y0, tw, th, flag_w, flag_s, flag_sw, epoch, sRow, io, sKnown, val, dst);
  finish_scatter<NI>(P, val, dst, dot);
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
                                          const Plane<NI>& actp, double* rq, int ix, int iy, int tw, int th,
                                          long long& ph_t0) {
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
  // ac.yf and actp.zf (plain stores), adds into acb.zf.  Per direction: all shared-memory
  // loads, then the arithmetic, then all stores.
#if defined(SC_EXP) && SC_EXP == 30
  const bool nonempty = false;   // ablation: no phase A
#else
  const bool nonempty = CI > 0 && CJ > 0 && CK > 0;
#endif
  if (si == DO && nonempty) {   // x-faces: face ix = W of element ix, E of element ix-1 (entries (j,k))
    const double* Z0 = in.ze(iy, ix) + sk;
    const double* Z1 = in.ze(iy + 1, ix) + sk;
    const double* Yb = inb.ye(iy, ix) + sj;
    const double* Yt = intp.ye(iy, ix) + sj;
    const double* fd = cf->fd[0] + sj + NI * sk;
    double w[M][M], e[M][M], f[M][M], zw[M], ze[M], yw[M], ye[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      zw[m] = fma(gj, Z1[2 * m], Z0[2 * m]);
      ze[m] = fma(gj, Z1[NI + 2 * m], Z0[NI + 2 * m]);
      yw[m] = fma(gk, Yt[2 * m], Yb[2 * m]);
      ye[m] = fma(gk, Yt[NI + 2 * m], Yb[NI + 2 * m]);
    }
#pragma unroll
    for (int jj = 0; jj < M; ++jj)
#pragma unroll
      for (int kk = 0; kk < M; ++kk) {
        const bool ok = jj < CJ && kk < CK;
        const int o = 2 * jj + 2 * NI * kk;
        w[jj][kk] = ok ? W[o] : 0.0;
        e[jj][kk] = ok ? E[o] : 0.0;
        f[jj][kk] = ok ? fd[o] : 0.0;
      }
    double rwj[M], rej[M], rwk[M], rek[M];
#pragma unroll
    for (int m = 0; m < M; ++m) rwj[m] = rej[m] = rwk[m] = rek[m] = 0.0;
#pragma unroll
    for (int jj = 0; jj < M; ++jj) {
      const double ej = cf->e[1][sj + 2 * jj], aj = cf->a[sj + 2 * jj];
#pragma unroll
      for (int kk = 0; kk < M; ++kk) {
        const double ek = cf->e[2][sk + 2 * kk], ak = cf->a[sk + 2 * kk];
        const double wv = w[jj][kk], ev = e[jj][kk];
        const double Wp = fma(f[jj][kk], wv, fma(cf->k0p[0], ev, fma(ej, zw[kk], ek * yw[jj])));
        const double Ep = fma(f[jj][kk], ev, fma(cf->k0p[0], wv, fma(ej, ze[kk], ek * ye[jj])));
        rwj[kk] = fma(aj, wv, rwj[kk]);
        rej[kk] = fma(aj, ev, rej[kk]);
        rwk[jj] = fma(ak, wv, rwk[jj]);
        rek[jj] = fma(ak, ev, rek[jj]);
        const double Em = __shfl_up_sync(0xffffffffu, Ep, 1);
        w[jj][kk] = ix > 0 ? Wp + Em : Wp;
        e[jj][kk] = Ep;
      }
    }
    if (act) {
      double* oj = rq + CS<NI>::R_XJ + (iy * (TX + 1) + ix) * 2 * NI + 2 * sk + sj;   // over j, keep k
      double* okk = rq + CS<NI>::R_XK + (iy * (TX + 1) + ix) * 2 * NI + 2 * sj + sk;  // over k, keep j
#pragma unroll
      for (int jj = 0; jj < M; ++jj)
#pragma unroll
        for (int kk = 0; kk < M; ++kk)
          if (jj < CJ && kk < CK) {
            const int o = 2 * jj + 2 * NI * kk;
            fX[o] = w[jj][kk];
            if (lastx) fX[o + N2] = e[jj][kk];
          }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        if (m < CK) { oj[4 * m] = rwj[m]; if (lastx) oj[2 * NI + 4 * m] = rej[m]; }
        if (m < CJ) { okk[4 * m] = rwk[m]; if (lastx) okk[2 * NI + 4 * m] = rek[m]; }
      }
      if (NI == 1) {   // no odd interior index: the odd parity components are 0
        oj[1] = okk[1] = 0.0;
        if (lastx) oj[2 * NI + 1] = okk[2 * NI + 1] = 0.0;
      }
    }
  }
  if (sj == DO && nonempty) {   // y-faces: face row iy = S of element row iy, N of row iy-1 (entries (i,k))
    const double* Z0 = in.ze(iy, ix) + sk;
    const double* Z1 = in.ze(iy + 1, ix) + sk;
    const double* Xb = inb.xe(iy, ix) + si;
    const double* Xt = intp.xe(iy, ix) + si;
    const double* fd = cf->fd[1] + si + NI * sk;
    double sv_[M][M], nv_[M][M], f[M][M], zs[M], zn[M], xs[M], xn[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      zs[m] = fma(gi, Z0[NI + 2 * m], Z0[2 * m]);
      zn[m] = fma(gi, Z1[NI + 2 * m], Z1[2 * m]);
      xs[m] = fma(gk, Xt[2 * m], Xb[2 * m]);
      xn[m] = fma(gk, Xt[TX * NI + 2 * m], Xb[TX * NI + 2 * m]);
    }
#pragma unroll
    for (int ii = 0; ii < M; ++ii)
#pragma unroll
      for (int kk = 0; kk < M; ++kk) {
        const bool ok = ii < CI && kk < CK;
        const int o = 2 * ii + 2 * NI * kk;
        sv_[ii][kk] = ok ? S[o] : 0.0;
        nv_[ii][kk] = ok ? N[o] : 0.0;
        f[ii][kk] = ok ? fd[o] : 0.0;
      }
    double rsi[M], rni[M], rsk[M], rnk[M];
#pragma unroll
    for (int m = 0; m < M; ++m) rsi[m] = rni[m] = rsk[m] = rnk[m] = 0.0;
#pragma unroll
    for (int ii = 0; ii < M; ++ii) {
      const double ei_ = cf->e[0][si + 2 * ii], ai = cf->a[si + 2 * ii];
#pragma unroll
      for (int kk = 0; kk < M; ++kk) {
        const double ek = cf->e[2][sk + 2 * kk], ak = cf->a[sk + 2 * kk];
        const double sv = sv_[ii][kk], nv = nv_[ii][kk];
        const double Sp = fma(f[ii][kk], sv, fma(cf->k0p[1], nv, fma(ei_, zs[kk], ek * xs[ii])));
        const double Np = fma(f[ii][kk], nv, fma(cf->k0p[1], sv, fma(ei_, zn[kk], ek * xn[ii])));
        rsi[kk] = fma(ai, sv, rsi[kk]);
        rni[kk] = fma(ai, nv, rni[kk]);
        rsk[ii] = fma(ak, sv, rsk[ii]);
        rnk[ii] = fma(ak, nv, rnk[ii]);
        const double Nm = __shfl_up_sync(0xffffffffu, Np, TX);
        sv_[ii][kk] = iy > 0 ? Sp + Nm : Sp;
        nv_[ii][kk] = Np;
      }
    }
    if (act) {
      double* oi = rq + CS<NI>::R_YI + (iy * TX + ix) * 2 * NI + 2 * sk + si;   // over i, keep k
      double* okk = rq + CS<NI>::R_YK + (iy * TX + ix) * 2 * NI + 2 * si + sk;  // over k, keep i
#pragma unroll
      for (int ii = 0; ii < M; ++ii)
#pragma unroll
        for (int kk = 0; kk < M; ++kk)
          if (ii < CI && kk < CK) {
            const int o = 2 * ii + 2 * NI * kk;
            fY[o] = sv_[ii][kk];
            if (lasty) fY[o + TX * N2] = nv_[ii][kk];
          }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        if (m < CK) { oi[4 * m] = rsi[m]; if (lasty) oi[TX * 2 * NI + 4 * m] = rni[m]; }
        if (m < CI) { okk[4 * m] = rsk[m]; if (lasty) okk[TX * 2 * NI + 4 * m] = rnk[m]; }
      }
      if (NI == 1) {
        oi[1] = okk[1] = 0.0;
        if (lasty) oi[TX * 2 * NI + 1] = okk[TX * 2 * NI + 1] = 0.0;
      }
    }
  }
  if (sk == DO && nonempty && act) {   // z-faces: B of this layer (plane l), T (plane l+1) (entries (i,j))
    const double* Yb = inb.ye(iy, ix) + sj;
    const double* Yt = intp.ye(iy, ix) + sj;
    const double* Xb = inb.xe(iy, ix) + si;
    const double* Xt = intp.xe(iy, ix) + si;
    const double* fd = cf->fd[2] + si + NI * sj;
    double bv_[M][M], tv_[M][M], f[M][M], ob[M][M], yb[M], yt[M], xb[M], xt[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      yb[m] = fma(gi, Yb[NI + 2 * m], Yb[2 * m]);
      yt[m] = fma(gi, Yt[NI + 2 * m], Yt[2 * m]);
      xb[m] = fma(gj, Xb[TX * NI + 2 * m], Xb[2 * m]);
      xt[m] = fma(gj, Xt[TX * NI + 2 * m], Xt[2 * m]);
    }
#pragma unroll
    for (int jj = 0; jj < M; ++jj)
#pragma unroll
      for (int ii = 0; ii < M; ++ii) {
        const bool ok = ii < CI && jj < CJ;
        const int o = 2 * ii + 2 * NI * jj;
        bv_[jj][ii] = ok ? B[o] : 0.0;
        tv_[jj][ii] = ok ? T[o] : 0.0;
        f[jj][ii] = ok ? fd[o] : 0.0;
        ob[jj][ii] = ok ? fB[o] : 0.0;
      }
    double rbi[M], rti[M], rbj[M], rtj[M];
#pragma unroll
    for (int m = 0; m < M; ++m) rbi[m] = rti[m] = rbj[m] = rtj[m] = 0.0;
#pragma unroll
    for (int jj = 0; jj < M; ++jj) {
      const double ej = cf->e[1][sj + 2 * jj], aj = cf->a[sj + 2 * jj];
#pragma unroll
      for (int ii = 0; ii < M; ++ii) {
        const double ei_ = cf->e[0][si + 2 * ii], ai = cf->a[si + 2 * ii];
        const double bv = bv_[jj][ii], tv = tv_[jj][ii];
        ob[jj][ii] += fma(f[jj][ii], bv, fma(cf->k0p[2], tv, fma(ei_, yb[jj], ej * xb[ii])));
        const double Tp = fma(f[jj][ii], tv, fma(cf->k0p[2], bv, fma(ei_, yt[jj], ej * xt[ii])));
        rbi[jj] = fma(ai, bv, rbi[jj]);
        rti[jj] = fma(ai, tv, rti[jj]);
        rbj[ii] = fma(aj, bv, rbj[ii]);
        rtj[ii] = fma(aj, tv, rtj[ii]);
        tv_[jj][ii] = Tp;
      }
    }
#pragma unroll
    for (int jj = 0; jj < M; ++jj)
#pragma unroll
      for (int ii = 0; ii < M; ++ii)
        if (ii < CI && jj < CJ) {
          const int o = 2 * ii + 2 * NI * jj;
          fB[o] = ob[jj][ii];
          fT[o] = tv_[jj][ii];
        }
    constexpr int PO = CS<NI>::NE * 2 * NI;
    double* oi = rq + CS<NI>::R_ZI + (iy * TX + ix) * 2 * NI + 2 * sj + si;    // over i, keep j (l+1 at + PO)
    double* oj = rq + CS<NI>::R_ZJ + (iy * TX + ix) * 2 * NI + 2 * si + sj;    // over j, keep i
#pragma unroll
    for (int m = 0; m < M; ++m) {
      if (m < CJ) { oi[4 * m] = rbi[m]; oi[PO + 4 * m] = rti[m]; }
      if (m < CI) { oj[4 * m] = rbj[m]; oj[PO + 4 * m] = rtj[m]; }
    }
    if (NI == 1) oi[1] = oi[PO + 1] = oj[1] = oj[PO + 1] = 0.0;
  }
  SC_PHASE(3);
  // ---- phase B: condensed part of the class (registers only)
  const double* Dv = cf->dinv + si + NI * sj + N2 * sk;
  double qx[M][M], qy[M][M], qz[M][M];
#if defined(SC_EXP) && SC_EXP == 31
#pragma unroll
  for (int a = 0; a < M; ++a)
#pragma unroll
    for (int b = 0; b < M; ++b) qx[a][b] = qy[a][b] = qz[a][b] = 0.0;   // ablation: no phase B
  if (false)
#endif
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
  SC_PHASE(4);
#pragma unroll 1
  for (int r = 0; r < 2; ++r) {
    bar_named(1);
#if defined(SC_EXP) && SC_EXP == 32
    continue;   // ablation: no output rounds
#endif
    SC_PHASE(5 + 6 * r);
    // The two classes of a direction (s_d = 0, 1) update the same entries; each round splits
    // them in halves (class s_d takes half h = r ^ s_d), so every warp does half of each of its
    // three directions in each round (balanced rounds, no warp idles while its SM-sub-partition
    // partner works).  Stores are predicated: the shuffles run converged.
    {   // x-faces, entries (jj, kk), halves by kk: W -= Q(ix) + g Q(ix-1), last element E -= g Q
      const int h = r ^ si;
      double o0[M][2], o1[M][2];
#pragma unroll
      for (int jj = 0; jj < M; ++jj)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int kk = 2 * h + t;
          const bool ok = act && jj < CJ && kk < CK && kk < M;
          const int o = 2 * jj + 2 * NI * kk;
          o0[jj][t] = ok ? fX[o] : 0.0;
          o1[jj][t] = (ok && lastx) ? fX[o + N2] : 0.0;
        }
#pragma unroll
      for (int jj = 0; jj < M; ++jj)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int kk = 2 * h + t;
          const bool ok = act && jj < CJ && kk < CK && kk < M;
          const int o = 2 * jj + 2 * NI * kk;
          const double Q = h ? (2 + t < M ? qx[jj][(2 + t) % M] : 0.0) : qx[jj][t % M];
          const double Qm = __shfl_up_sync(0xffffffffu, Q, 1);
          const double n0 = o0[jj][t] - (ix > 0 ? fma(gi, Qm, Q) : Q), n1 = fma(-gi, Q, o1[jj][t]);
          if (ok) fX[o] = n0;
          if (ok && lastx) fX[o + N2] = n1;
        }
    }
    {   // y-faces, entries (ii, kk), halves by kk
      const int h = r ^ sj;
      double o0[M][2], o1[M][2];
#pragma unroll
      for (int ii = 0; ii < M; ++ii)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int kk = 2 * h + t;
          const bool ok = act && ii < CI && kk < CK && kk < M;
          const int o = 2 * ii + 2 * NI * kk;
          o0[ii][t] = ok ? fY[o] : 0.0;
          o1[ii][t] = (ok && lasty) ? fY[o + TX * N2] : 0.0;
        }
#pragma unroll
      for (int ii = 0; ii < M; ++ii)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int kk = 2 * h + t;
          const bool ok = act && ii < CI && kk < CK && kk < M;
          const int o = 2 * ii + 2 * NI * kk;
          const double Q = h ? (2 + t < M ? qy[ii][(2 + t) % M] : 0.0) : qy[ii][t % M];
          const double Qm = __shfl_up_sync(0xffffffffu, Q, TX);
          const double n0 = o0[ii][t] - (iy > 0 ? fma(gj, Qm, Q) : Q), n1 = fma(-gj, Q, o1[ii][t]);
          if (ok) fY[o] = n0;
          if (ok && lasty) fY[o + TX * N2] = n1;
        }
    }
    if (act) {   // z-faces, entries (jj, ii), halves by ii: B -= Q, T -= g Q
      const int h = r ^ sk;
      double o0[M][2], o1[M][2];
#pragma unroll
      for (int jj = 0; jj < M; ++jj)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int ii = 2 * h + t;
          const bool ok = ii < CI && jj < CJ && ii < M;
          const int o = 2 * ii + 2 * NI * jj;
          o0[jj][t] = ok ? fB[o] : 0.0;
          o1[jj][t] = ok ? fT[o] : 0.0;
        }
#pragma unroll
      for (int jj = 0; jj < M; ++jj)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int ii = 2 * h + t;
          const bool ok = ii < CI && jj < CJ && ii < M;
          const int o = 2 * ii + 2 * NI * jj;
          const double Q = h ? (2 + t < M ? qz[jj][(2 + t) % M] : 0.0) : qz[jj][t % M];
          if (ok) {
            fB[o] = o0[jj][t] - Q;
            fT[o] = fma(-gk, Q, o1[jj][t]);
          }
        }
    }
    SC_PHASE(10 + 2 * r);
  }
}

// ---- n_I <= 3: one element per thread, all parity classes in the thread --------------------
// Same arithmetic as the class warps (faces-in, D^{-1}, faces-out of Table 2; primary part of
// the faces, Eq. 26 generalised; a0-weighted face line sums for the edge / vertex rows), in the
// plain (not even / odd) form.  Order: line sums of the input faces, condensed part (Q of the six
// faces in registers), then per direction primary - Q and the stores (the faces are re-read from
// shared memory, which keeps the register count down).  x-faces of a tile row are summed with a
// lane shuffle (rows of TX consecutive threads in one warp), y-faces in two barrier-separated
// rounds by element-row parity, z-faces as in the class version.
template <int NI>
__device__ __forceinline__ void vol_elem(const ColCoef* cf, const Side<NI>& in, const Plane<NI>& inb,
                                         const Plane<NI>& intp, const Side<NI>& ac, const Plane<NI>& acb,
                                         const Plane<NI>& actp, double* rq, int ix, int iy, int tw, int th) {
  constexpr int N2 = NI * NI, TX = CS<NI>::TX, NE = CS<NI>::NE;
  const bool act = (int)threadIdx.x < NE && ix < tw && iy < th;
  const bool lastx = ix == tw - 1, lasty = iy == th - 1;
  const int ex = min(ix, TX - 1), ey = min(iy, CS<NI>::TY - 1);
  const double* W = in.xf(ey, ex);
  const double* E = W + N2;
  const double* S = in.yf(ey, ex);
  const double* N = S + TX * N2;
  const double* B = inb.zf(ey, ex);
  const double* T = intp.zf(ey, ex);
  // a0-weighted line sums (R+, R-) of the input faces, for the edge / vertex rows: x-face W (and
  // E for the last element of the row), y-face S (and N), z-faces B and T
  if (act) {
    auto lsum = [&](const double* f, int stride_a, int stride_c, double* o) {
#pragma unroll
      for (int c = 0; c < NI; ++c) {
        double rp = 0.0, rm = 0.0;
#pragma unroll
        for (int a = 0; a < NI; ++a) {
          const double t = cf->a[a] * f[a * stride_a + c * stride_c];
          if (a & 1) rm += t; else rp += t;
        }
        o[2 * c] = rp;
        o[2 * c + 1] = rm;
      }
    };
    double* xj = rq + CS<NI>::R_XJ + (iy * (TX + 1) + ix) * 2 * NI;
    double* xk = rq + CS<NI>::R_XK + (iy * (TX + 1) + ix) * 2 * NI;
    lsum(W, 1, NI, xj);        // over j, keep k
    lsum(W, NI, 1, xk);        // over k, keep j
    if (lastx) { lsum(E, 1, NI, xj + 2 * NI); lsum(E, NI, 1, xk + 2 * NI); }
    double* yi = rq + CS<NI>::R_YI + (iy * TX + ix) * 2 * NI;
    double* yk = rq + CS<NI>::R_YK + (iy * TX + ix) * 2 * NI;
    lsum(S, 1, NI, yi);        // over i, keep k
    lsum(S, NI, 1, yk);        // over k, keep i
    if (lasty) { lsum(N, 1, NI, yi + TX * 2 * NI); lsum(N, NI, 1, yk + TX * 2 * NI); }
    constexpr int PO = NE * 2 * NI;
    double* zi = rq + CS<NI>::R_ZI + (iy * TX + ix) * 2 * NI;
    double* zj = rq + CS<NI>::R_ZJ + (iy * TX + ix) * 2 * NI;
    lsum(B, 1, NI, zi);        // over i, keep j
    lsum(B, NI, 1, zj);        // over j, keep i
    lsum(T, 1, NI, zi + PO);
    lsum(T, NI, 1, zj + PO);
  }
  // condensed part: u = d1 (W + g_i E) + d2 (S + g_j N) + d3 (B + g_k T) (a0-weighted: c_d),
  // v = u D^{-1}; Q_W += c1 v, Q_E += g_i c1 v, ...
  double qw[N2], qe[N2], qs[N2], qn[N2], qb[N2], qt[N2];
#pragma unroll
  for (int q = 0; q < N2; ++q) qw[q] = qe[q] = qs[q] = qn[q] = qb[q] = qt[q] = 0.0;
#pragma unroll
  for (int k = 0; k < NI; ++k)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const double gi = (i & 1) ? -1.0 : 1.0, gj = (j & 1) ? -1.0 : 1.0, gk = (k & 1) ? -1.0 : 1.0;
        const int ox = j + NI * k, oy = i + NI * k, oz = i + NI * j;
        const double u = fma(cf->c[0][i], fma(gi, E[ox], W[ox]),
                             fma(cf->c[1][j], fma(gj, N[oy], S[oy]), cf->c[2][k] * fma(gk, T[oz], B[oz])));
        const double v = u * cf->dinv[i + NI * (j + NI * k)];
        const double vx = cf->c[0][i] * v, vy = cf->c[1][j] * v, vz = cf->c[2][k] * v;
        qw[ox] += vx; qe[ox] = fma(gi, vx, qe[ox]);
        qs[oy] += vy; qn[oy] = fma(gj, vy, qn[oy]);
        qb[oz] += vz; qt[oz] = fma(gk, vz, qt[oz]);
      }
  const double* Z0 = in.ze(ey, ex);                    // z-edges at (fx, fy), (fx+1, fy)
  const double* Z1 = in.ze(ey + 1, ex);                // z-edges at (fx, fy+1), (fx+1, fy+1)
  const double* Yb = inb.ye(ey, ex);                   // y-edges of planes l, l+1 at fx, fx+1
  const double* Yt = intp.ye(ey, ex);
  const double* Xb = inb.xe(ey, ex);                   // x-edges of planes l, l+1 at fy, fy+1
  const double* Xt = intp.xe(ey, ex);
  // x-faces, entries (a, b) = (j, k): primary (self, opposite face, z-edges at k, y-edges at j)
  // minus Q; face ix = W part of element ix + E part of element ix-1 (lane - 1)
  {
    double* fX = ac.xf(ey, ex);
#pragma unroll
    for (int b = 0; b < NI; ++b)
#pragma unroll
      for (int a = 0; a < NI; ++a) {
        const int q = a + NI * b;
        const double ga = (a & 1) ? -1.0 : 1.0, gb = (b & 1) ? -1.0 : 1.0;
        const double w = W[q], e = E[q];
        const double zw = fma(ga, Z1[b], Z0[b]), ze_ = fma(ga, Z1[NI + b], Z0[NI + b]);
        const double yw = fma(gb, Yt[a], Yb[a]), ye_ = fma(gb, Yt[NI + a], Yb[NI + a]);
        const double Wp = fma(cf->fd[0][q], w, fma(cf->k0p[0], e, fma(cf->e[1][a], zw, cf->e[2][b] * yw))) - qw[q];
        const double Ep = fma(cf->fd[0][q], e, fma(cf->k0p[0], w, fma(cf->e[1][a], ze_, cf->e[2][b] * ye_))) - qe[q];
        const double Em = __shfl_up_sync(0xffffffffu, Ep, 1);
        if (act) {
          fX[q] = ix > 0 ? Wp + Em : Wp;
          if (lastx) fX[q + N2] = Ep;
        }
      }
  }
  // z-faces, entries (a, b) = (i, j): y-edges at j, x-edges at i; B of this layer (plane l,
  // added), T (plane l+1, initialised)
  if (act) {
    double* fB = acb.zf(ey, ex);
    double* fT = actp.zf(ey, ex);
#pragma unroll
    for (int b = 0; b < NI; ++b)
#pragma unroll
      for (int a = 0; a < NI; ++a) {
        const int q = a + NI * b;
        const double ga = (a & 1) ? -1.0 : 1.0, gb = (b & 1) ? -1.0 : 1.0;
        const double bv = B[q], tv = T[q];
        const double yb = fma(ga, Yb[NI + b], Yb[b]), yt = fma(ga, Yt[NI + b], Yt[b]);
        const double xb = fma(gb, Xb[TX * NI + a], Xb[a]), xt = fma(gb, Xt[TX * NI + a], Xt[a]);
        const double Bp = fma(cf->fd[2][q], bv, fma(cf->k0p[2], tv, fma(cf->e[0][a], yb, cf->e[1][b] * xb))) - qb[q];
        const double Tp = fma(cf->fd[2][q], tv, fma(cf->k0p[2], bv, fma(cf->e[0][a], yt, cf->e[1][b] * xt))) - qt[q];
        fB[q] += Bp;
        fT[q] = Tp;
      }
  }
  // y-faces, entries (a, b) = (i, k): z-edges at k, x-edges at i.  Round 0: even element rows
  // (plain stores of S and N); round 1: odd rows add (the tile's last face row is plain when no
  // even row wrote it)
  {
    double* fY = ac.yf(ey, ex);
    double sp[N2], np[N2];
#pragma unroll
    for (int b = 0; b < NI; ++b)
#pragma unroll
      for (int a = 0; a < NI; ++a) {
        const int q = a + NI * b;
        const double ga = (a & 1) ? -1.0 : 1.0, gb = (b & 1) ? -1.0 : 1.0;
        const double sv = S[q], nv = N[q];
        const double zs = fma(ga, Z0[NI + b], Z0[b]), zn = fma(ga, Z1[NI + b], Z1[b]);
        const double xs = fma(gb, Xt[a], Xb[a]), xn = fma(gb, Xt[TX * NI + a], Xb[TX * NI + a]);
        sp[q] = fma(cf->fd[1][q], sv, fma(cf->k0p[1], nv, fma(cf->e[0][a], zs, cf->e[2][b] * xs))) - qs[q];
        np[q] = fma(cf->fd[1][q], nv, fma(cf->k0p[1], sv, fma(cf->e[0][a], zn, cf->e[2][b] * xn))) - qn[q];
      }
    if (act && (iy & 1) == 0) {
#pragma unroll
      for (int q = 0; q < N2; ++q) { fY[q] = sp[q]; fY[q + TX * N2] = np[q]; }
    }
    bar_named(1);
    if (act && (iy & 1) == 1) {
#pragma unroll
      for (int q = 0; q < N2; ++q) {
        fY[q] += sp[q];
        if (lasty) fY[q + TX * N2] = np[q]; else fY[q + TX * N2] += np[q];
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
  __shared__ long long sRow[C::MAXROWS];
  __shared__ RowIO sIO[C::MAXROWS];
  __shared__ int sEpoch;
  __shared__ unsigned long long sKnown[3];   // neighbours' progress already acquired (this item)
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
#pragma unroll 1
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

  for (;;) {
    __syncthreads();
    if (tid == 0) sTicket = atomicAdd(&P.st->ticket, 1ULL);
    __syncthreads();
    const long long item = (long long)sTicket;
    if (item >= P.nitems) break;
    const int epoch = sEpoch;
    const int ntile = P.ntx * P.nty;
    const int seg = (int)(item / ntile), tile = (int)(item - (long long)seg * ntile);
    const int tx = tile % P.ntx, ty = tile / P.ntx;
    const int x0 = tx * TX, y0 = ty * TY;
    const int tw = min(TX, g.nx - x0), th = min(TY, g.ny - y0);
    // z-segment: steps [lfin0, lend] are finalized here; a segment above the first starts one
    // step early (lbeg = lfin0 - 1) and recomputes element layer lbeg, whose side / plane lbeg
    // the segment below finalizes, for the complete accumulator of plane lfin0 (no z exchange)
    const int lfin0 = seg * P.zseg;
    const int lbeg = seg > 0 ? lfin0 - 1 : 0;
    const int lend = seg == P.nseg - 1 ? g.nz : min(g.nz, lfin0 + P.zseg) - 1;
    unsigned long long* const flag_me = P.prog + item;
    const unsigned long long* const flag_w = tx > 0 ? P.prog + (item - 1) : nullptr;
    const unsigned long long* const flag_s = ty > 0 ? P.prog + (item - P.ntx) : nullptr;
    const unsigned long long* const flag_sw = (tx > 0 && ty > 0) ? P.prog + (item - P.ntx - 1) : nullptr;
    if (tid < 3) sKnown[tid] = 0ULL;

    // row descriptors of the tile, then the prologue: planes 0, 1 and side 0 as one cp.async group
    int ns;
    build_rows<NI>(P, sIO, x0, y0, tw, th, &ns);
    __syncthreads();
    load_block<NI>(P.x, sIO, true, ns, th, sm + C::O_IP + (lbeg % 3) * C::PLANE, lbeg, zdir(g, lbeg));
    load_block<NI>(P.x, sIO, false, ns, th, sm + C::O_IS + (lbeg & 1) * C::SIDE, lbeg, false);
    load_block<NI>(P.x, sIO, true, ns, th, sm + C::O_IP + ((lbeg + 1) % 3) * C::PLANE, lbeg + 1, zdir(g, lbeg + 1));
    cp_commit();
    for (int t = tid; t < C::PLANE; t += NT) sm[C::O_AP + (lbeg & 1) * C::PLANE + t] = 0.0;
    double dot = 0.0;

    // Step l computes element layer l (l < nz) and finalizes layer l / plane l.  Inputs: side l
    // in buffer l & 1, plane q in q % 3 (so plane l+2 is prefetched at the top of step l into
    // the buffer of plane l-1); accumulators: side (one buffer), plane q in q & 1.
    for (int l = lbeg; l <= lend; ++l) {
      const bool last = (l == g.nz);         // final step: only plane nz remains
      const Side<NI> in{sm + C::O_IS + (l & 1) * C::SIDE};
      const Plane<NI> inb{sm + C::O_IP + (l % 3) * C::PLANE}, intp{sm + C::O_IP + ((l + 1) % 3) * C::PLANE};
      const Plane<NI> acb{sm + C::O_AP + (l & 1) * C::PLANE}, actp{sm + C::O_AP + ((l + 1) & 1) * C::PLANE};
      // prefetch side l+1 and plane l+2 (overlap this step's compute); wait for side l, plane l+1
#if !(defined(SC_EXP) && SC_EXP == 25)
      if (l + 1 < g.nz && l + 1 <= lend)
        load_block<NI>(P.x, sIO, false, ns, th, sm + C::O_IS + ((l + 1) & 1) * C::SIDE, l + 1, false);
      if (l + 2 <= g.nz && l + 2 <= lend + 1)
        load_block<NI>(P.x, sIO, true, ns, th, sm + C::O_IP + ((l + 2) % 3) * C::PLANE, l + 2, zdir(g, l + 2));
#endif
      cp_commit();
      // publication of step l-1 (its stores were issued before the barrier that ended step l-1):
      // the GPU-scope fence overlaps this step's load wait
      if (tid == 0 && l >= lfin0 + 1) {
#if !(defined(SC_EXP) && SC_EXP == 26)
        __threadfence();
#endif
        prog_release(flag_me, ((unsigned long long)(unsigned)epoch << 32) | (unsigned)l);   // steps <= l-1
      }
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
            if (r < NZE) { eo_reduce<NI>(in.ze(r / (TX + 1), r % (TX + 1)), 1, sA0, rq + C::R_ZE + r * 2); continue; }
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
#if !(defined(SC_EXP) && SC_EXP == 21)
        if constexpr (C::PER_ELEM)
          vol_elem<NI>(sCf, in, inb, intp, ac, acb, actp, rq, tid % TX, tid / TX, tw, th);
        else
          vol_class<NI>(kWarpClass[warp], sCf, in, inb, intp, ac, acb, actp, rq, vix, viy, tw, th, ph_t0);
#endif
        __syncthreads();
        SC_PHASE(2);
        // ============ primary part Htilde_BB of the edges / vertices, entity-centric ============
        // (Mtilde = diag(w0, 1..1, w0); Ktilde arrowhead: row 0 = (K00, a0, K0p),
        //  row p = (K0p, ap, K00), interior row m = (a0_m @0, Lam_m @m, ap_m @p).)
        // Edges: lane groups of n_I per edge; vertices: a lane each.  Each accumulator entry is
        // owned by exactly one lane, which sums the contributions of the tile's adjacent elements.
        // All results of a thread are computed first and added to the accumulators at the end
        // (no shared-memory read-after-write chain between entities).
#if !(defined(SC_EXP) && SC_EXP == 22)
        {
          auto present = [&](int ix, int iy) { return ix >= 0 && iy >= 0 && ix < tw && iy < th; };
          constexpr int NZE = (TY + 1) * (TX + 1), NXE = 2 * (TY + 1) * TX, NYE = 2 * TY * (TX + 1);
          constexpr int SZ = (NZE + NW * EPW - 1) / (NW * EPW), SX = (NXE + NW * EPW - 1) / (NW * EPW);
          constexpr int SY = (NYE + NW * EPW - 1) / (NW * EPW), SV = (2 * NZE + NT - 1) / NT;
          constexpr int SN = SZ + SX + SY + SV;
          double res[SN];
          int dsto[SN];
          const double w02d0 = dA * w02;
#pragma unroll
          for (int s = 0; s < SN; ++s) { res[s] = 0.0; dsto[s] = -1; }
          // ---- z-edges (fx = ix, fy = iy), coord k = c
#pragma unroll
          for (int s = 0; s < SZ; ++s) {
            const int e = (s * NW + warp) * EPW + esub, ix = e % (TX + 1), iy = e / (TX + 1), c = ec;
            if (!evalid || e >= NZE || ix > tw || iy > th) continue;
            const double u = in.ze(iy, ix)[c];
            const double tz = sA0[c] * (*inb.vv(iy, ix) + ((c & 1) ? -*intp.vv(iy, ix) : *intp.vv(iy, ix))) + sLam[c] * u;
            // the x-line term depends on ib only, the y-line term on jb only: each is evaluated
            // once and weighted by the number of present elements sharing it
            const int p00 = present(ix, iy), p10 = present(ix - 1, iy), p01 = present(ix, iy - 1),
                      p11 = present(ix - 1, iy - 1);
            double y = (p00 + p10 + p01 + p11) * (w02d0 * u + dD * w02 * tz);
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const int nxb = b ? p10 + p11 : p00 + p01, nyb = b ? p01 + p11 : p00 + p10;
              if (nxb) {
                const int ex = ix - b;
                const double txl = (b ? K0p : K00) * in.ze(iy, ex)[c] + (b ? K00 : K0p) * in.ze(iy, ex + 1)[c] +
                                   eo_row(rq + C::R_YI + (iy * TX + ex) * 2 * NI + 2 * c, b);
                y = fma(nxb * dB * w0, txl, y);
              }
              if (nyb) {
                const int ey = iy - b;
                const double tyl = (b ? K0p : K00) * in.ze(ey, ix)[c] + (b ? K00 : K0p) * in.ze(ey + 1, ix)[c] +
                                   eo_row(rq + C::R_XJ + (ey * (TX + 1) + ix) * 2 * NI + 2 * c, b);
                y = fma(nyb * dC * w0, tyl, y);
              }
            }
            res[s] = y;
            dsto[s] = (int)(ac.ze(iy, ix) + c - sm);
          }
          // ---- x-edges (ex = ix, fy = iy) of planes l, l+1, coord i = c
#pragma unroll
          for (int s = 0; s < SX; ++s) {
            const int e = (s * NW + warp) * EPW + esub, kb = e / ((TY + 1) * TX), ff = e % ((TY + 1) * TX);
            const int ix = ff % TX, iy = ff / TX, c = ec;
            if (!evalid || e >= NXE || ix >= tw || iy > th) continue;
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
              y += w02d0 * u + dB * w02 * txl + dC * w0 * tyl + dD * w0 * tzl;
            }
            res[SZ + s] = y;
            dsto[SZ + s] = (int)((kb ? actp : acb).xe(iy, ix) + c - sm);
          }
          // ---- y-edges (fx = ix, ey = iy) of planes l, l+1, coord j = c
#pragma unroll
          for (int s = 0; s < SY; ++s) {
            const int e = (s * NW + warp) * EPW + esub, kb = e / (TY * (TX + 1)), ff = e % (TY * (TX + 1));
            const int ix = ff % (TX + 1), iy = ff / (TX + 1), c = ec;
            if (!evalid || e >= NYE || ix > tw || iy >= th) continue;
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
              y += w02d0 * u + dB * w0 * txl + dC * w02 * tyl + dD * w0 * tzl;
            }
            res[SZ + SX + s] = y;
            dsto[SZ + SX + s] = (int)((kb ? actp : acb).ye(iy, ix) + c - sm);
          }
          // ---- vertices (fx = ix, fy = iy) of planes l, l+1
#pragma unroll
          for (int s = 0; s < SV; ++s) {
            const int v = s * NT + tid, kb = v / NZE, ff = v % NZE, ix = ff % (TX + 1), iy = ff / (TX + 1);
            if (v >= 2 * NZE || ix > tw || iy > th) continue;
            const Plane<NI> pk = kb ? intp : inb;
            const double u = *pk.vv(iy, ix);
            const double tzl = (kb ? K0p : K00) * *inb.vv(iy, ix) + (kb ? K00 : K0p) * *intp.vv(iy, ix) +
                               eo_row(rq + C::R_ZE + (iy * (TX + 1) + ix) * 2, kb);
            const int p00 = present(ix, iy), p10 = present(ix - 1, iy), p01 = present(ix, iy - 1),
                      p11 = present(ix - 1, iy - 1);
            double y = (p00 + p10 + p01 + p11) * (w02d0 * w0 * u + w02 * dD * tzl);
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const int nxb = b ? p10 + p11 : p00 + p01, nyb = b ? p01 + p11 : p00 + p10;
              if (nxb) {
                const int ex = ix - b;
                const double txl = (b ? K0p : K00) * *pk.vv(iy, ex) + (b ? K00 : K0p) * *pk.vv(iy, ex + 1) +
                                   eo_row(rq + C::R_XE + (kb * (TY + 1) * TX + iy * TX + ex) * 2, b);
                y = fma(nxb * w02 * dB, txl, y);
              }
              if (nyb) {
                const int ey = iy - b;
                const double tyl = (b ? K0p : K00) * *pk.vv(ey, ix) + (b ? K00 : K0p) * *pk.vv(ey + 1, ix) +
                                   eo_row(rq + C::R_YE + (kb * TY * (TX + 1) + ey * (TX + 1) + ix) * 2, b);
                y = fma(nyb * w02 * dC, tyl, y);
              }
            }
            res[SZ + SX + SY + s] = y;
            dsto[SZ + SX + SY + s] = (int)((kb ? actp : acb).vv(iy, ix) - sm);
          }
          double old[SN];
#pragma unroll
          for (int s = 0; s < SN; ++s) old[s] = dsto[s] >= 0 ? sm[dsto[s]] : 0.0;
#pragma unroll
          for (int s = 0; s < SN; ++s)
            if (dsto[s] >= 0) sm[dsto[s]] = old[s] + res[s];
        }
#endif
        __syncthreads();
        SC_PHASE(6);
      }
      if (l < lfin0) continue;               // warm-up step of an upper z-segment: no output
      // finish the W / S boundary entities of step l - LB: gather (flags, pending + neighbour
      // partials) before this step's finalize, so the loads overlap it; store after
      constexpr int MAXE = (C::PEND + NT - 1) / NT;
      double fval[MAXE];
      double* fdst[MAXE];
#pragma unroll
      for (int k = 0; k < MAXE; ++k) { fval[k] = 0.0; fdst[k] = nullptr; }
#if !(defined(SC_EXP) && SC_EXP == 24)
      if (l >= lfin0 + kLB)
        finish_gather<NI>(P, item, l - kLB, x0, y0, tw, th, flag_w, flag_s, flag_sw, epoch, sRow, sIO, sKnown, fval, fdst);
#endif
#if !(defined(SC_EXP) && SC_EXP == 23)
      finalize_step<NI>(P, item, l, x0, y0, tw, th, ac, acb, in, inb, sIO, ns, !last, dot);
#endif
      finish_scatter<NI>(P, fval, fdst, dot);
      SC_PHASE(7);
      __syncthreads();
      SC_PHASE(8);
    }
    // end of the column: publish the last step, finish the last LB steps
    if (tid == 0) {
      __threadfence();
      prog_release(flag_me, ((unsigned long long)(unsigned)epoch << 32) | (unsigned)(lend + 1));
    }
    for (int ls = max(lfin0, lend - kLB + 1); ls <= lend; ++ls) {
      finish_boundary<NI>(P, item, ls, x0, y0, tw, th, flag_w, flag_s, flag_sw, epoch, sRow, sIO, sKnown, dot);
      __syncthreads();
    }
    // per-tile partial of x . y (fixed order: deterministic)
    if (P.dotp) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      __syncthreads();
      if (lane == 0) sRow[warp] = __double_as_longlong(dot);
      __syncthreads();
      if (tid == 0) {
        double t = 0.0;
        for (int w = 0; w < NW; ++w) t += __longlong_as_double(sRow[w]);
        P.dotp[item] = t;
      }
    }
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
  static int max_active_d[kMaxDev], nsm_d[kMaxDev];   // per device (0 = not queried yet)
  const int dv = dev_slot();
  int& max_active = max_active_d[dv];
  int& nsm = nsm_d[dv];
  if (max_active < 1) {
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
  return (int)cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(unsigned long long) * 8 * 16);
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

// Load balance of the persistent kernel: ntiles tile columns on nsm CTAs take
// ceil(ntiles / nsm) rounds of nz + 1 steps; splitting each column into S z-segments gives
// ceil(S ntiles / nsm) rounds of ceil(nz / S) + 1 (+ 1 recomputed layer) steps.  Model cost per
// round: the steps plus ~2 steps of look-back pipeline fill.  SC_ZSEG overrides S.
int col_slots() { return kSlots; }

void col_choose_segments(int ntiles, int nz, int nsm, int* nseg, int* zseg) {
  int best = 1;
  double bcost = 1e300;
  const char* env = getenv("SC_ZSEG");
  const int forced = env ? atoi(env) : 0;
  for (int S = 1; S <= 8 && S <= nz; ++S) {
    const int zs = (nz + S - 1) / S;
    if ((long long)zs * (S - 1) >= nz) continue;           // every segment non-empty
    const double rounds = (double)(((long long)ntiles * S + nsm - 1) / nsm);
    const double cost = rounds * (zs + 1 + (S > 1 ? 1 : 0) + 2);
    if (forced ? S == forced : cost < bcost * 0.97) { bcost = cost; best = S; }
  }
  *nseg = best;
  *zseg = (nz + best - 1) / best;
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

int launch_apply_col_raw(const Geom& g, const double* x, double* y, const double* done, void* state, void* flags,
                         double* corner, double* pending, int ntx, int nty, int nseg, int zseg, const void* coef,
                         double* dotp, void* stream, int* nl, void* events) {
  ColParams P;
  P.g = g; P.x = x; P.y = y; P.done = done; P.st = (ColState*)state; P.prog = (unsigned long long*)flags; P.corner = corner;
  P.pending = pending;
  P.ntx = ntx; P.nty = nty; P.nitems = ntx * nty * nseg;
  P.nseg = nseg; P.zseg = zseg;
  P.dotp = dotp;
  memcpy(&P.cf, coef, sizeof(ColCoef));
  int grid = 0;
  return launch_apply_col(P, stream, nl, &grid, events);
}

}  // namespace sc
