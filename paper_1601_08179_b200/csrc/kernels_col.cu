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
  int ntx, nty, nitems;
};

template <int NI>
struct CS {
  static constexpr int N2 = NI * NI;
  static constexpr int LPE = NI <= 1 ? 1 : (NI <= 2 ? 2 : (NI <= 4 ? 4 : 8));
  static constexpr int NT = 128;
  static constexpr int NE = NT / LPE;
  static constexpr int TX = NE == 128 ? 16 : (NE >= 32 ? 8 : 4);
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
  static constexpr int DINV = NI * NI * NI;
  static constexpr int O_IS = 0;
  static constexpr int O_IP = O_IS + SIDE;
  static constexpr int O_AS = O_IP + 2 * PLANE;
  static constexpr int O_AP = O_AS + SIDE;
  static constexpr int O_QZ = O_AP + 2 * PLANE;
  static constexpr int O_DINV = O_QZ + QZ;
  static constexpr int O_D = O_DINV + DINV;          // per-element d: NE x 4
  static constexpr int O_TAB = O_D + 4 * NE;         // a0, ap, lam (3 x 32)
  static constexpr int TOTAL = O_TAB + 3 * 32;
  static constexpr int NSH = 6 * N2 + 12 * NI + 8;   // element shell nodes
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

// Load one z-plane (fz) of the tile into smem (Dirichlet entities read as 0).
template <int NI>
__device__ void load_plane(const ColParams& P, Plane<NI> pl, int x0, int y0, int tw, int th, int fz) {
  using C = CS<NI>;
  const Geom& g = P.g;
  Addr A{g};
  const bool zd = zdir(g, fz);
  const int tid = threadIdx.x;
  // z-faces: TY rows x TX faces (contiguous tw*N2 per row)
  for (int t = tid; t < C::TY * C::TX * C::N2; t += C::NT) {
    int q = t % C::N2, ix = (t / C::N2) % C::TX, iy = t / (C::N2 * C::TX);
    double v = 0.0;
    if (ix < tw && iy < th && !zd) v = P.x[A.zf(x0 + ix, y0 + iy, fz) + q];
    pl.zf(iy, ix)[q] = v;
  }
  for (int t = tid; t < (C::TY + 1) * C::TX * NI; t += C::NT) {   // x-edges (ex, fy)
    int c = t % NI, ix = (t / NI) % C::TX, iy = t / (NI * C::TX);
    int fy = y0 + iy;
    double v = 0.0;
    if (ix < tw && iy <= th && !zd && fy != 0 && fy != g.ny) v = P.x[A.xe(x0 + ix, fy, fz) + c];
    pl.xe(iy, ix)[c] = v;
  }
  for (int t = tid; t < C::TY * (C::TX + 1) * NI; t += C::NT) {   // y-edges (fx, ey)
    int c = t % NI, ix = (t / NI) % (C::TX + 1), iy = t / (NI * (C::TX + 1));
    int fx = x0 + ix;
    double v = 0.0;
    if (ix <= tw && iy < th && !zd && fx != 0 && fx != g.nx) v = P.x[A.ye(fx, y0 + iy, fz) + c];
    pl.ye(iy, ix)[c] = v;
  }
  for (int t = tid; t < (C::TY + 1) * (C::TX + 1); t += C::NT) {   // vertices
    int ix = t % (C::TX + 1), iy = t / (C::TX + 1);
    int fx = x0 + ix, fy = y0 + iy;
    double v = 0.0;
    if (ix <= tw && iy <= th && !zd && fx != 0 && fx != g.nx && fy != 0 && fy != g.ny) v = P.x[A.vv(fx, fy, fz)];
    *pl.vv(iy, ix) = v;
  }
}

template <int NI>
__device__ void load_side(const ColParams& P, Side<NI> sd, int x0, int y0, int tw, int th, int ez) {
  using C = CS<NI>;
  const Geom& g = P.g;
  Addr A{g};
  const int tid = threadIdx.x;
  for (int t = tid; t < C::TY * (C::TX + 1) * C::N2; t += C::NT) {   // x-faces (fx, ey)
    int q = t % C::N2, ix = (t / C::N2) % (C::TX + 1), iy = t / (C::N2 * (C::TX + 1));
    int fx = x0 + ix;
    double v = 0.0;
    if (ix <= tw && iy < th && fx != 0 && fx != g.nx) v = P.x[A.xf(fx, y0 + iy, ez) + q];
    sd.xf(iy, ix)[q] = v;
  }
  for (int t = tid; t < (C::TY + 1) * C::TX * C::N2; t += C::NT) {   // y-faces (ex, fy)
    int q = t % C::N2, ix = (t / C::N2) % C::TX, iy = t / (C::N2 * C::TX);
    int fy = y0 + iy;
    double v = 0.0;
    if (ix < tw && iy <= th && fy != 0 && fy != g.ny) v = P.x[A.yf(x0 + ix, fy, ez) + q];
    sd.yf(iy, ix)[q] = v;
  }
  for (int t = tid; t < (C::TY + 1) * (C::TX + 1) * NI; t += C::NT) {   // z-edges (fx, fy)
    int c = t % NI, ix = (t / NI) % (C::TX + 1), iy = t / (NI * (C::TX + 1));
    int fx = x0 + ix, fy = y0 + iy;
    double v = 0.0;
    if (ix <= tw && iy <= th && fx != 0 && fx != g.nx && fy != 0 && fy != g.ny) v = P.x[A.ze(fx, fy, ez) + c];
    sd.ze(iy, ix)[c] = v;
  }
}

// Primary part (Htilde_BB) contribution of element (ix, iy) at its shell node s, accumulated
// into the tile accumulators (arrowhead Ktilde rows: 0 = (K00, a0, K0p),
// p = (K0p, ap, K00), interior m = (a0_m @0, Lam_m @m, ap_m @p)).
template <int NI>
__device__ void primary_node(int s, int ix, int iy, const double* d, Side<NI> in, Plane<NI> inb, Plane<NI> intp,
                             Side<NI> ac, Plane<NI> acb, Plane<NI> actp, const double* a0, const double* ap,
                             const double* lam, double K00, double K0p, double w0) {
  using C = CS<NI>;
  constexpr int N2 = C::N2;
  const double w02 = w0 * w0;
  if (s < 6 * N2) {
    const int f = s / N2, q = s % N2, a = q % NI, b = q / NI;
    double u, opp, diag, e1, e2;
    double* out;
    if (f < 2) {            // x-face: coords (a = j, b = k)
      const int ib = f;
      u = in.xf(iy, ix + ib)[q];
      opp = in.xf(iy, ix + 1 - ib)[q];
      diag = d[0] * w0 + d[1] * K00 + d[2] * w0 * lam[a] + d[3] * w0 * lam[b];
      // d2 term: z-edges (ib, jb=0/1) along k; d3 term: y-edges (ib, kb=0/1) along j
      e1 = d[2] * w0 * (a0[a] * in.ze(iy, ix + ib)[b] + ap[a] * in.ze(iy + 1, ix + ib)[b]);
      e2 = d[3] * w0 * (a0[b] * inb.ye(iy, ix + ib)[a] + ap[b] * intp.ye(iy, ix + ib)[a]);
      out = ac.xf(iy, ix + ib) + q;
      *out += diag * u + d[1] * K0p * opp + e1 + e2;
    } else if (f < 4) {     // y-face: coords (a = i, b = k)
      const int jb = f - 2;
      u = in.yf(iy + jb, ix)[q];
      opp = in.yf(iy + 1 - jb, ix)[q];
      diag = d[0] * w0 + d[1] * w0 * lam[a] + d[2] * K00 + d[3] * w0 * lam[b];
      e1 = d[1] * w0 * (a0[a] * in.ze(iy + jb, ix)[b] + ap[a] * in.ze(iy + jb, ix + 1)[b]);
      e2 = d[3] * w0 * (a0[b] * inb.xe(iy + jb, ix)[a] + ap[b] * intp.xe(iy + jb, ix)[a]);
      out = ac.yf(iy + jb, ix) + q;
      *out += diag * u + d[2] * K0p * opp + e1 + e2;
    } else {                // z-face: coords (a = i, b = j)
      const int kb = f - 4;
      Plane<NI> pu = kb ? intp : inb, po = kb ? inb : intp;
      u = pu.zf(iy, ix)[q];
      opp = po.zf(iy, ix)[q];
      diag = d[0] * w0 + d[1] * w0 * lam[a] + d[2] * w0 * lam[b] + d[3] * K00;
      e1 = d[1] * w0 * (a0[a] * pu.ye(iy, ix)[b] + ap[a] * pu.ye(iy, ix + 1)[b]);
      e2 = d[2] * w0 * (a0[b] * pu.xe(iy, ix)[a] + ap[b] * pu.xe(iy + 1, ix)[a]);
      out = (kb ? actp : acb).zf(iy, ix) + q;
      *out += diag * u + d[3] * K0p * opp + e1 + e2;
    }
    return;
  }
  s -= 6 * N2;
  if (s < 12 * NI) {
    const int e = s / NI, c = s % NI, grp = e >> 2, b0 = e & 1, b1 = (e >> 1) & 1;
    if (grp == 0) {         // x-edge (jb = b0, kb = b1), coord i = c
      const int jb = b0, kb = b1;
      Plane<NI> pk = kb ? intp : inb;
      const double u = pk.xe(iy + jb, ix)[c];
      // along x: vertices (ib = 0/1, jb, kb)
      double tx = a0[c] * *pk.vv(iy + jb, ix) + lam[c] * u + ap[c] * *pk.vv(iy + jb, ix + 1);
      // y-line at (i = c, k = kb p): x-edges (jb'=0/1, kb) ends, z-face (kb) interior (i = c, j = a)
      const double* fz = pk.zf(iy, ix);
      const double* ry = jb ? ap : a0;
      double ty = (jb ? K0p : K00) * pk.xe(iy, ix)[c] + (jb ? K00 : K0p) * pk.xe(iy + 1, ix)[c];
#pragma unroll
      for (int a = 0; a < NI; ++a) ty += ry[a] * fz[c + NI * a];
      // z-line at (i = c, j = jb p): x-edges (jb, kb'=0/1) ends, y-face (jb) interior (i = c, k = a)
      const double* fy = in.yf(iy + jb, ix);
      const double* rz = kb ? ap : a0;
      double tz = (kb ? K0p : K00) * inb.xe(iy + jb, ix)[c] + (kb ? K00 : K0p) * intp.xe(iy + jb, ix)[c];
#pragma unroll
      for (int a = 0; a < NI; ++a) tz += rz[a] * fy[c + NI * a];
      (kb ? actp : acb).xe(iy + jb, ix)[c] += d[0] * w02 * u + d[1] * w02 * tx + d[2] * w0 * ty + d[3] * w0 * tz;
    } else if (grp == 1) {  // y-edge (ib = b0, kb = b1), coord j = c
      const int ib = b0, kb = b1;
      Plane<NI> pk = kb ? intp : inb;
      const double u = pk.ye(iy, ix + ib)[c];
      // x-line at (j = c, k = kb p): y-edges (ib'=0/1, kb), z-face (kb) interior (i = a, j = c)
      const double* fz = pk.zf(iy, ix);
      const double* rx = ib ? ap : a0;
      double tx = (ib ? K0p : K00) * pk.ye(iy, ix)[c] + (ib ? K00 : K0p) * pk.ye(iy, ix + 1)[c];
#pragma unroll
      for (int a = 0; a < NI; ++a) tx += rx[a] * fz[a + NI * c];
      double ty = a0[c] * *pk.vv(iy, ix + ib) + lam[c] * u + ap[c] * *pk.vv(iy + 1, ix + ib);
      // z-line at (i = ib p, j = c): y-edges (ib, kb'=0/1), x-face (ib) interior (j = c, k = a)
      const double* fx = in.xf(iy, ix + ib);
      const double* rz = kb ? ap : a0;
      double tz = (kb ? K0p : K00) * inb.ye(iy, ix + ib)[c] + (kb ? K00 : K0p) * intp.ye(iy, ix + ib)[c];
#pragma unroll
      for (int a = 0; a < NI; ++a) tz += rz[a] * fx[c + NI * a];
      (kb ? actp : acb).ye(iy, ix + ib)[c] += d[0] * w02 * u + d[1] * w0 * tx + d[2] * w02 * ty + d[3] * w0 * tz;
    } else {                // z-edge (ib = b0, jb = b1), coord k = c
      const int ib = b0, jb = b1;
      const double u = in.ze(iy + jb, ix + ib)[c];
      // x-line at (j = jb p, k = c): z-edges (ib'=0/1, jb), y-face (jb) interior (i = a, k = c)
      const double* fy = in.yf(iy + jb, ix);
      const double* rx = ib ? ap : a0;
      double tx = (ib ? K0p : K00) * in.ze(iy + jb, ix)[c] + (ib ? K00 : K0p) * in.ze(iy + jb, ix + 1)[c];
#pragma unroll
      for (int a = 0; a < NI; ++a) tx += rx[a] * fy[a + NI * c];
      // y-line at (i = ib p, k = c): z-edges (ib, jb'=0/1), x-face (ib) interior (j = a, k = c)
      const double* fx = in.xf(iy, ix + ib);
      const double* ry = jb ? ap : a0;
      double ty = (jb ? K0p : K00) * in.ze(iy, ix + ib)[c] + (jb ? K00 : K0p) * in.ze(iy + 1, ix + ib)[c];
#pragma unroll
      for (int a = 0; a < NI; ++a) ty += ry[a] * fx[a + NI * c];
      double tz = a0[c] * *inb.vv(iy + jb, ix + ib) + lam[c] * u + ap[c] * *intp.vv(iy + jb, ix + ib);
      ac.ze(iy + jb, ix + ib)[c] += d[0] * w02 * u + d[1] * w0 * tx + d[2] * w0 * ty + d[3] * w02 * tz;
    }
    return;
  }
  s -= 12 * NI;
  {                         // vertex (ib, jb, kb)
    const int ib = s & 1, jb = (s >> 1) & 1, kb = (s >> 2) & 1;
    Plane<NI> pk = kb ? intp : inb;
    const double u = *pk.vv(iy + jb, ix + ib);
    const double* rx = ib ? ap : a0;
    const double* ry = jb ? ap : a0;
    const double* rz = kb ? ap : a0;
    double tx = (ib ? K0p : K00) * *pk.vv(iy + jb, ix) + (ib ? K00 : K0p) * *pk.vv(iy + jb, ix + 1);
    double ty = (jb ? K0p : K00) * *pk.vv(iy, ix + ib) + (jb ? K00 : K0p) * *pk.vv(iy + 1, ix + ib);
    double tz = (kb ? K0p : K00) * *inb.vv(iy + jb, ix + ib) + (kb ? K00 : K0p) * *intp.vv(iy + jb, ix + ib);
    const double* ex = pk.xe(iy + jb, ix);
    const double* ey = pk.ye(iy, ix + ib);
    const double* ez = in.ze(iy + jb, ix + ib);
#pragma unroll
    for (int a = 0; a < NI; ++a) {
      tx += rx[a] * ex[a];
      ty += ry[a] * ey[a];
      tz += rz[a] * ez[a];
    }
    *(kb ? actp : acb).vv(iy + jb, ix + ib) += d[0] * w02 * w0 * u + w02 * (d[1] * tx + d[2] * ty + d[3] * tz);
  }
}

// ---- finalize helpers: write / publish / consume one entity vector ----------------------
// Corner record address: corner point (cx, cy) of the tile grid, step l, slot (0 SW, 1 S, 2 W).
__device__ __forceinline__ double* corner_rec(const ColParams& P, int cx, int cy, int l, int slot) {
  const int ni = P.g.ni;
  return P.corner + ((((long long)cy * (P.ntx + 1) + cx) * (P.g.nz + 1) + l) * 3 + slot) * (ni + 1);
}

template <int NI>
__global__ void __launch_bounds__(128) k_apply_col(ColParams P) {
  using C = CS<NI>;
  constexpr int N2 = C::N2, TX = C::TX, TY = C::TY, NT = C::NT, LPE = C::LPE;
  if (P.done != nullptr && *P.done != 0.0) return;
  const Geom& g = P.g;
  extern __shared__ double sm[];
  double* sDinv = sm + C::O_DINV;
  double* sD = sm + C::O_D;
  double* sA0 = sm + C::O_TAB;
  double* sAp = sA0 + 32;
  double* sLam = sAp + 32;
  __shared__ unsigned long long sTicket;
  __shared__ int sEpoch;
  const int tid = threadIdx.x;
  if (tid == 0) sEpoch = *(volatile int*)&P.st->epoch + 1;
  Addr A{g};
  const double K00 = g.tab[TAB_SCAL + 0], K0p = g.tab[TAB_SCAL + 1], w0 = g.tab[TAB_SCAL + 2];
  for (int t = tid; t < NI; t += NT) {
    sA0[t] = g.tab[TAB_A0 + t];
    sAp[t] = g.tab[TAB_AP + t];
    sLam[t] = g.tab[TAB_LAM + t];
  }
  if (g.dinv)
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
  Side<NI> in{sm + C::O_IS}, ac{sm + C::O_AS};
  double* const qz = sm + C::O_QZ;
  // ---- per-thread constants of the volume phase: thread (e, k)
  const int ve = tid / LPE, vk = tid % LPE;
  const bool vact = vk < NI;
  const int vix = ve % TX, viy = ve / TX;
  const double sk = (vk & 1) ? -1.0 : 1.0;

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

    // plane 0: input + accumulator
    load_plane<NI>(P, Plane<NI>{sm + C::O_IP}, x0, y0, tw, th, 0);
    for (int t = tid; t < C::PLANE; t += NT) sm[C::O_AP + t] = 0.0;

    for (int l = 0; l <= g.nz; ++l) {
      const bool last = (l == g.nz);         // final step: only plane nz remains
      Plane<NI> inb{sm + C::O_IP + (l & 1) * C::PLANE}, intp{sm + C::O_IP + ((l + 1) & 1) * C::PLANE};
      Plane<NI> acb{sm + C::O_AP + (l & 1) * C::PLANE}, actp{sm + C::O_AP + ((l + 1) & 1) * C::PLANE};
      if (!last) {
        load_side<NI>(P, in, x0, y0, tw, th, l);
        load_plane<NI>(P, intp, x0, y0, tw, th, l + 1);
        for (int t = tid; t < C::SIDE; t += NT) sm[C::O_AS + t] = 0.0;
        for (int t = tid; t < C::PLANE; t += NT) actp.b[t] = 0.0;
        for (int t = tid; t < C::NE; t += NT) {
          int ex = x0 + min(t % TX, tw - 1), ey = y0 + min(t / TX, th - 1);
          double d[4];
          metric(g, ex, ey, l, d);
          for (int q = 0; q < 4; ++q) sD[t * 4 + q] = d[q];
        }
        __syncthreads();
        // ================= volume phase: faces-in, D^{-1}, faces-out (even/odd) ==============
        {
          const bool eact = vact && vix < tw && viy < th;
          const double* d = sD + ve * 4;
          const double d1 = d[1], d2 = d[2], d3 = d[3];
          const int kk = vact ? vk : 0;
          const double ak = eact ? sA0[kk] : 0.0;
          double pxp[NI], pxm[NI], pyp[NI], pym[NI];
          double qxp[NI], qxm[NI], qyp[NI], qym[NI];
          const double* W = in.xf(viy, vix);
          const double* E = in.xf(viy, vix + 1);
          const double* S = in.yf(viy, vix);
          const double* N = in.yf(viy + 1, vix);
          const double* B = inb.zf(viy, vix);
          const double* T = intp.zf(viy, vix);
#pragma unroll
          for (int j = 0; j < NI; ++j) {
            double w = eact ? W[j + NI * kk] : 0.0, e = eact ? E[j + NI * kk] : 0.0;
            pxp[j] = d1 * (w + e);
            pxm[j] = d1 * (w - e);
            double s = eact ? S[j + NI * kk] : 0.0, n = eact ? N[j + NI * kk] : 0.0;
            pyp[j] = d2 * (s + n);
            pym[j] = d2 * (s - n);
            qxp[j] = qxm[j] = qyp[j] = qym[j] = 0.0;
          }
          const double d0 = d[0];
#pragma unroll
          for (int j = 0; j < NI; ++j) {
#pragma unroll
            for (int i = 0; i < NI; ++i) {
              const int q = i + NI * j;
              const double pz = d3 * (B[q] + sk * T[q]);
              const double u = sA0[i] * ((i & 1) ? pxm[j] : pxp[j]) + sA0[j] * ((j & 1) ? pym[i] : pyp[i]) + ak * pz;
              const double dinv = g.dinv ? sDinv[q + N2 * kk]
                                         : 1.0 / (d0 + d1 * sLam[i] + d2 * sLam[j] + d3 * sLam[kk]);
              const double v = u * dinv;
              if (i & 1) qxm[j] += sA0[i] * v; else qxp[j] += sA0[i] * v;
              if (j & 1) qym[i] += sA0[j] * v; else qyp[i] += sA0[j] * v;
              double c = ak * v;
              if (LPE >= 4) c += __shfl_xor_sync(0xffffffffu, c, 2);
              if (LPE >= 8) c += __shfl_xor_sync(0xffffffffu, c, 4);
              if (vk < 2 && eact) qz[(ve * 2 + vk) * N2 + q] = c;
            }
          }
          // x / y outputs: low faces first, high faces after a barrier (race-free accumulation)
          if (eact) {
            double* aW = ac.xf(viy, vix);
            double* aS = ac.yf(viy, vix);
#pragma unroll
            for (int j = 0; j < NI; ++j) {
              aW[j + NI * kk] -= d1 * (qxp[j] + qxm[j]);
              aS[j + NI * kk] -= d2 * (qyp[j] + qym[j]);
            }
          }
          __syncthreads();
          if (eact) {
            double* aE = ac.xf(viy, vix + 1);
            double* aN = ac.yf(viy + 1, vix);
#pragma unroll
            for (int j = 0; j < NI; ++j) {
              aE[j + NI * kk] -= d1 * (qxp[j] - qxm[j]);
              aN[j + NI * kk] -= d2 * (qyp[j] - qym[j]);
            }
          }
        }
        __syncthreads();
        // z outputs from the parity sums
        for (int t = tid; t < C::NE * N2; t += NT) {
          const int e = t / N2, q = t % N2, ix = e % TX, iy = e / TX;
          if (ix >= tw || iy >= th) continue;
          const double d3 = sD[e * 4 + 3];
          const double qp = qz[(e * 2) * N2 + q], qm = NI > 1 ? qz[(e * 2 + 1) * N2 + q] : 0.0;
          acb.zf(iy, ix)[q] -= d3 * (qp + qm);
          actp.zf(iy, ix)[q] -= d3 * (qp - qm);
        }
        __syncthreads();
        // ================= primary part, four colour phases ==================================
        for (int col = 0; col < 4; ++col) {
          const int cx = col & 1, cy = col >> 1;
          constexpr int NPC = ((TX + 1) / 2) * ((TY + 1) / 2);   // elements per colour
          for (int t = tid; t < NPC * C::NSH; t += NT) {
            const int ec = t / C::NSH, s = t % C::NSH;
            const int ix = cx + 2 * (ec % ((TX + 1) / 2)), iy = cy + 2 * (ec / ((TX + 1) / 2));
            if (ix >= tw || iy >= th) continue;
            primary_node<NI>(s, ix, iy, sD + (iy * TX + ix) * 4, in, inb, intp, ac, acb, actp, sA0, sAp, sLam, K00, K0p,
                             w0);
          }
          __syncthreads();
        }
      }
      // ================= finalize: publish, write owned, look-back, write boundary ==========
      // Entities finished at this step: side entities of layer l (if !last) and plane l.
      const bool pzd = zdir(g, l);
      // (a) publish partials of entities owned by a higher-ticket tile
      if (!last) {
        for (int t = tid; t < th * N2; t += NT) {          // x-faces at fx = x0 + tw (E boundary)
          const int iy = t / N2, q = t % N2, fx = x0 + tw;
          if (fx < g.nx) P.y[A.xf(fx, y0 + iy, l) + q] = ac.xf(iy, tw)[q];
        }
        for (int t = tid; t < tw * N2; t += NT) {          // y-faces at fy = y0 + th (N boundary)
          const int ix = t / N2, q = t % N2, fy = y0 + th;
          if (fy < g.ny) P.y[A.yf(x0 + ix, fy, l) + q] = ac.yf(th, ix)[q];
        }
      }
      // z-edges (layer l) + vertices (plane l) on the tile boundary lines; x-edges / y-edges (plane l)
      for (int t = tid; t < (TX + 1) * (TY + 1) * (NI + 1); t += NT) {
        const int c = t % (NI + 1), ix = (t / (NI + 1)) % (TX + 1), iy = t / ((NI + 1) * (TX + 1));
        if (ix > tw || iy > th) continue;
        const int fx = x0 + ix, fy = y0 + iy;
        const bool ex_ = (ix == tw && fx < g.nx), ny_ = (iy == th && fy < g.ny);
        const bool wx = (ix == 0 && fx > 0), sy = (iy == 0 && fy > 0);
        if (!ex_ && !ny_) continue;                         // owned here
        const bool isv = (c == NI);
        if (!isv && last) continue;
        if (isv ? (pzd || fx == 0 || fx == g.nx || fy == 0 || fy == g.ny)
                : (fx == 0 || fx == g.nx || fy == 0 || fy == g.ny))
          continue;                                         // Dirichlet: nothing to publish
        const double v = isv ? *acb.vv(iy, ix) : ac.ze(iy, ix)[c];
        if (ex_ && ny_) {
          corner_rec(P, (fx) / TX, (fy) / TY, l, 0)[c] = v;         // I am SW of the owner
        } else if (ex_ && sy) {
          corner_rec(P, fx / TX, fy / TY, l, 2)[c] = v;             // I am W of the owner
        } else if (ny_ && wx) {
          corner_rec(P, fx / TX, fy / TY, l, 1)[c] = v;             // I am S of the owner
        } else {
          if (isv) P.y[A.vv(fx, fy, l)] = v;
          else P.y[A.ze(fx, fy, l) + c] = v;
        }
      }
      for (int t = tid; t < tw * NI; t += NT) {            // x-edges at fy = y0 + th, plane l
        const int ix = t / NI, c = t % NI, fy = y0 + th;
        if (fy < g.ny && !pzd) P.y[A.xe(x0 + ix, fy, l) + c] = acb.xe(th, ix)[c];
      }
      for (int t = tid; t < th * NI; t += NT) {            // y-edges at fx = x0 + tw, plane l
        const int iy = t / NI, c = t % NI, fx = x0 + tw;
        if (fx < g.nx && !pzd) P.y[A.ye(fx, y0 + iy, l) + c] = acb.ye(iy, tw)[c];
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) flag_release(flag_me + l, epoch);
      // (b) owned entities without a lower-ticket contributor
      if (!last) {
        for (int t = tid; t < th * (TX + 1) * N2; t += NT) {   // x-faces
          const int q = t % N2, ix = (t / N2) % (TX + 1), iy = t / (N2 * (TX + 1));
          const int fx = x0 + ix;
          if (ix > tw) continue;
          if (ix == tw && fx < g.nx) continue;                 // published
          if (ix == 0 && fx > 0) continue;                     // needs W
          P.y[A.xf(fx, y0 + iy, l) + q] = (fx == 0 || fx == g.nx) ? 0.0 : ac.xf(iy, ix)[q];
        }
        for (int t = tid; t < (TY + 1) * tw * N2; t += NT) {   // y-faces
          const int q = t % N2, ix = (t / N2) % tw, iy = t / (N2 * tw);
          const int fy = y0 + iy;
          if (iy > th) continue;
          if (iy == th && fy < g.ny) continue;
          if (iy == 0 && fy > 0) continue;
          P.y[A.yf(x0 + ix, fy, l) + q] = (fy == 0 || fy == g.ny) ? 0.0 : ac.yf(iy, ix)[q];
        }
      }
      for (int t = tid; t < th * tw * N2; t += NT) {           // z-faces of plane l
        const int q = t % N2, ix = (t / N2) % tw, iy = t / (N2 * tw);
        P.y[A.zf(x0 + ix, y0 + iy, l) + q] = pzd ? 0.0 : acb.zf(iy, ix)[q];
      }
      for (int t = tid; t < (TX + 1) * (TY + 1) * (NI + 1); t += NT) {   // z-edges + vertices
        const int c = t % (NI + 1), ix = (t / (NI + 1)) % (TX + 1), iy = t / ((NI + 1) * (TX + 1));
        if (ix > tw || iy > th) continue;
        const bool isv = (c == NI);
        if (!isv && last) continue;
        const int fx = x0 + ix, fy = y0 + iy;
        const bool ex_ = (ix == tw && fx < g.nx), ny_ = (iy == th && fy < g.ny);
        const bool wx = (ix == 0 && fx > 0), sy = (iy == 0 && fy > 0);
        if (ex_ || ny_) continue;
        const bool dr = (fx == 0 || fx == g.nx || fy == 0 || fy == g.ny) || (isv && pzd);
        if (!dr && (wx || sy)) continue;                       // needs look-back
        const double v = dr ? 0.0 : (isv ? *acb.vv(iy, ix) : ac.ze(iy, ix)[c]);
        if (isv) P.y[A.vv(fx, fy, l)] = v;
        else P.y[A.ze(fx, fy, l) + c] = v;
      }
      for (int t = tid; t < (TY + 1) * tw * NI; t += NT) {     // x-edges of plane l
        const int c = t % NI, ix = (t / NI) % tw, iy = t / (NI * tw);
        if (iy > th) continue;
        const int fy = y0 + iy;
        if (iy == th && fy < g.ny) continue;
        const bool dr = pzd || fy == 0 || fy == g.ny;
        if (!dr && iy == 0 && fy > 0) continue;
        P.y[A.xe(x0 + ix, fy, l) + c] = dr ? 0.0 : acb.xe(iy, ix)[c];
      }
      for (int t = tid; t < th * (TX + 1) * NI; t += NT) {     // y-edges of plane l
        const int c = t % NI, ix = (t / NI) % (TX + 1), iy = t / (NI * (TX + 1));
        if (ix > tw) continue;
        const int fx = x0 + ix;
        if (ix == tw && fx < g.nx) continue;
        const bool dr = pzd || fx == 0 || fx == g.nx;
        if (!dr && ix == 0 && fx > 0) continue;
        P.y[A.ye(fx, y0 + iy, l) + c] = dr ? 0.0 : acb.ye(iy, ix)[c];
      }
      // (c) look-back: wait for the W, S, SW tiles of this step
      if (tid == 0) {
        if (flag_w) while (flag_acquire(flag_w + l) != epoch) __nanosleep(64);
        if (flag_s) while (flag_acquire(flag_s + l) != epoch) __nanosleep(64);
        if (flag_sw) while (flag_acquire(flag_sw + l) != epoch) __nanosleep(64);
      }
      __syncthreads();
      if (!last) {
        if (x0 > 0)
          for (int t = tid; t < th * N2; t += NT) {            // x-faces at fx = x0
            const int iy = t / N2, q = t % N2;
            const long long a = A.xf(x0, y0 + iy, l) + q;
            P.y[a] = ac.xf(iy, 0)[q] + ld_cg(P.y + a);
          }
        if (y0 > 0)
          for (int t = tid; t < tw * N2; t += NT) {            // y-faces at fy = y0
            const int ix = t / N2, q = t % N2;
            const long long a = A.yf(x0 + ix, y0, l) + q;
            P.y[a] = ac.yf(0, ix)[q] + ld_cg(P.y + a);
          }
      }
      for (int t = tid; t < (TX + 1) * (TY + 1) * (NI + 1); t += NT) {
        const int c = t % (NI + 1), ix = (t / (NI + 1)) % (TX + 1), iy = t / ((NI + 1) * (TX + 1));
        if (ix > tw || iy > th) continue;
        const bool isv = (c == NI);
        if (!isv && last) continue;
        const int fx = x0 + ix, fy = y0 + iy;
        const bool ex_ = (ix == tw && fx < g.nx), ny_ = (iy == th && fy < g.ny);
        const bool wx = (ix == 0 && fx > 0), sy = (iy == 0 && fy > 0);
        if (ex_ || ny_) continue;
        const bool dr = (fx == 0 || fx == g.nx || fy == 0 || fy == g.ny) || (isv && pzd);
        if (dr || !(wx || sy)) continue;
        double v = isv ? *acb.vv(iy, ix) : ac.ze(iy, ix)[c];
        const long long a = isv ? A.vv(fx, fy, l) : A.ze(fx, fy, l) + c;
        if (wx && sy) {
          const int cx = fx / TX, cy = fy / TY;
          v += ld_cg(corner_rec(P, cx, cy, l, 0) + c) + ld_cg(corner_rec(P, cx, cy, l, 1) + c) +
               ld_cg(corner_rec(P, cx, cy, l, 2) + c);
        } else {
          v += ld_cg(P.y + a);
        }
        P.y[a] = v;
      }
      if (!pzd) {
        if (y0 > 0)
          for (int t = tid; t < tw * NI; t += NT) {            // x-edges at fy = y0, plane l
            const int ix = t / NI, c = t % NI;
            const long long a = A.xe(x0 + ix, y0, l) + c;
            P.y[a] = acb.xe(0, ix)[c] + ld_cg(P.y + a);
          }
        if (x0 > 0)
          for (int t = tid; t < th * NI; t += NT) {            // y-edges at fx = x0, plane l
            const int iy = t / NI, c = t % NI;
            const long long a = A.ye(x0, y0 + iy, l) + c;
            P.y[a] = acb.ye(iy, 0)[c] + ld_cg(P.y + a);
          }
      }
      __syncthreads();
    }
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

bool col_supported(int ni) { return ni >= 1 && ni <= 8; }

void col_tile(int ni, int* tx, int* ty) {
  switch (ni) {
#define TCASE(N) case N: *tx = CS<N>::TX; *ty = CS<N>::TY; return;
    TCASE(1) TCASE(2) TCASE(3) TCASE(4) TCASE(5) TCASE(6) TCASE(7) TCASE(8)
#undef TCASE
    default: *tx = *ty = 0;
  }
}

int launch_apply_col(const ColParams& P, void* stream, int* nl, int* grid_out, void* events);

int launch_apply_col_raw(const Geom& g, const double* x, double* y, const double* done, void* state, int* flags,
                         double* corner, int ntx, int nty, void* stream, int* nl, void* events) {
  ColParams P;
  P.g = g; P.x = x; P.y = y; P.done = done; P.st = (ColState*)state; P.flags = flags; P.corner = corner;
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
