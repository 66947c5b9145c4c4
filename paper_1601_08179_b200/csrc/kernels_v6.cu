// Condensed operator v6 (rows a3-a8 of SURVEY §8(a)) for 2 <= n_I <= 7 (p = 3..8), uniform
// geometry: tile columns with a recomputed halo, bulk-copy (TMA) row loads, uniform class lanes.
//
// Work decomposition.  A CTA owns the skeleton entities of an xy-tile of 7 x (H - 1) elements over a
// z-segment of element layers: x-faces fx in [x0, x0+7), y-faces fy in [y0, y0+H-1), z-faces /
// edges / vertices of the same index ranges, element layers [lfin0, lend] and planes [lfin0, lend]
// (+ plane nz for the top segment).  It computes the 8 x H elements ex in [x0-1, x0+7),
// ey in [y0-1, y0+H-1): the extra column / row (the "halo") are the neighbours whose condensed
// parts reach the owned W / S faces.  Every owned entity is then complete inside the CTA: no
// inter-CTA communication (no look-back, flags or atomics), each skeleton entry is written by
// exactly one CTA, and the result is independent of scheduling.  Edges and vertices have no
// condensed part (c13), so their values are primary-part stencils of the input, computed
// entity-centrically by their owner.  H = 4 (two CTAs of 8 warps per SM) or 8 (one CTA of 16 warps,
// halo overhead 64/49 instead of 32/21).
//
// The CTA marches up its column one element layer per step.  Per step l warp 0 bulk-loads
// (cp.async.bulk + one mbarrier transaction) the rows of layer l (x-faces, y-faces, z-edges) and
// plane l+1 (z-faces, x-edges, y-edges, vertices); plane l stays from the previous step.  Each
// entity row of the tile is one contiguous skeleton range; a row is copied as the
// 16-byte aligned superset of its valid range into a slot whose base has the same 8-byte phase,
// so the row sits at slot + (global index & 1).
//
// Condensed part (Table 2, Eq. 26) in the even / odd form: with ap = sigma .* a0 the
// interior points split into 8 parity classes (s_i, s_j, s_k); lane = (element, class), a warp
// holds a 2 x 2 block of elements x 8 classes and every warp runs the same code (see k_apply_v6).
//
// An earlier design of this file (v5, git history) ran one class per warp with fully
// specialised code; measured instruction-fetch bound (8 distinct code streams per CTA) and slower.
//
// Fused p . q (PCG): x . A x = sum over owned entities of x * (primary part) - sum over owned
// elements of the condensed energy uhat . D^{-1} uhat (uhat = faces-in of the element), so
// each CTA returns its partial without re-reading x.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include "sc_device.cuh"

namespace sc {

struct V5Coef {
  double c[3][8];        // c[d][m] = d_{d+1} a0_m                        (condensed faces in / out)
  double dinv[343];      // D^{-1}(i,j,k) = 1/(d0 + d1 Lam_i + d2 Lam_j + d3 Lam_k), i fastest
  double fdx[49];        // x-face self (2 elements): 2 (d0 w0 + d1 K00 + d2 w0 Lam_j + d3 w0 Lam_k) at j + NI k
  double fdy[49];        // y-face self: 2 (d0 w0 + d2 K00 + d1 w0 Lam_i + d3 w0 Lam_k) at i + NI k
  double fdz[49];        // z-face self per layer: d0 w0 + d3 K00 + d1 w0 Lam_i + d2 w0 Lam_j at i + NI j
  double k0p[3];         // d_{d+1} K0p                                   (opposite face)
  double ef2[3][8];      // 2 d_{d+1} w0 a0_m    (x- / y-face <- bounding edges, 2 elements)
  double ef1[3][8];      // d_{d+1} w0 a0_m      (z-face <- bounding edges, one layer)
  double czu[8], cxu[8], cyu[8];   // edge self terms (see the edge phase)
  double sc[16];         // scalars of the edge / vertex stencils (see v6_make_coef)
  double a0[8], sig[8];
};

struct V5Params {
  Geom g;
  const double* x;
  double* y;
  const double* done;
  double* dotp;          // per-CTA partials of x . (A x) (fused PCG p . q), or null
  int ntx, nty, nseg, zseg, nitems;
  V5Coef cf;
};

namespace v5 {

constexpr int TX = 8, OX = 7;   // compute / owned tile width in x

// tile of height H (compute H rows of elements, own H - 1): derived constants and the row kinds of
// the per-item descriptor table (side rows of layer l: x-faces, y-faces, z-edges; plane rows of
// plane q: z-faces, x-edges, y-edges, vertices)
template <int H>
struct TC {
  static constexpr int TY = H, OY = H - 1, NO = OX * OY, NT = 64 * H;
  static constexpr int R_XF = 0, R_YF = H, R_ZE = 2 * H + 1, R_ZF = 3 * H + 2, R_XE = 4 * H + 2, R_YE = 5 * H + 3,
                       R_V = 6 * H + 3, NROWS = 7 * H + 4, NSIDE = 3 * H + 2;
};

// slot of a row of len doubles: >= len + 2 (the 16-byte rounding of the copy), even, and for long
// rows (res >= 0) the stride residue res mod 16 doubles (bank-pair placement of neighbouring rows)
constexpr int slot_len(int len, int res) {
  int v = len + 2;
  if (v & 1) ++v;
  if (len >= 16 && res >= 0)
    while (v % 16 != res) v += 2;
  return v;
}
constexpr int even(int v) { return v + (v & 1); }

// shared-memory layout of the input rows: face rows with a stride of 4 mod 16 doubles (the two rows
// a half-warp reads fall on disjoint bank pairs), edge / vertex rows unpadded
template <int NI, int H>
struct L {
  using C = TC<H>;
  static constexpr int TY = H;
  static constexpr int N2 = NI * NI;
  static constexpr int XS = slot_len((TX + 1) * N2, 4), YS = slot_len(TX * N2, 4), ZS = slot_len(TX * N2, 4);
  static constexpr int ZES = slot_len((TX + 1) * NI, -1), XES = slot_len(TX * NI, -1), YES = slot_len((TX + 1) * NI, -1);
  static constexpr int VS = slot_len(TX + 1, -1);
  static constexpr int O_XF = 0;
  static constexpr int O_YF = O_XF + TY * XS;
  static constexpr int O_ZE = O_YF + (TY + 1) * YS;
  static constexpr int O_ZF = O_ZE + (TY + 1) * ZES;       // 2 planes (plane q in q & 1)
  static constexpr int PZ = TY * ZS;
  static constexpr int O_PL = O_ZF + 2 * PZ;                // 2 planes of edges / vertices
  static constexpr int PLX = 0, PLY = (TY + 1) * XES, PLV = PLY + TY * YES, PLS = PLV + (TY + 1) * VS;
  static constexpr int END = O_PL + 2 * PLS;                // first double after the input rows
};

struct Row {
  long long g0, gs;   // skeleton index of the row start at layer / plane 0, per-layer stride
  int slot, len;      // smem slot offset (doubles), row length (entries)
  int a, b;           // valid, non-Dirichlet entries [a, b) (a >= b: nothing to copy)
  int plane;          // plane row (Dirichlet when its plane is)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* m, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* m, unsigned bytes) {
  unsigned long long state;
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 %0, [%1], %2;"
               : "=l"(state)
               : "r"(smem_u32(m)), "r"(bytes)
               : "memory");
  (void)state;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(smem_u32(m)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* m) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(m))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ---- per-item row descriptors ------------------------------------------------------------
template <int NI, int H>
__device__ void make_row(const Geom& g, int r, int cx0, int cy0, Row& d) {
  using LL = L<NI, H>;
  constexpr int R_YF = TC<H>::R_YF, R_ZE = TC<H>::R_ZE, R_ZF = TC<H>::R_ZF, R_XE = TC<H>::R_XE, R_YE = TC<H>::R_YE,
                R_V = TC<H>::R_V;
  constexpr int N2 = NI * NI;
  const int nx = g.nx, ny = g.ny;
  auto clampx = [&](int lo_ok, int hi_ok, int per) {   // valid index range [lo_ok, hi_ok] of the row's entities
    const int lo = max(cx0, lo_ok), hi = min(cx0 + TX - (per == 0 ? 1 : 0), hi_ok);
    d.a = (lo - cx0) * (per ? per : 1);
    d.b = (hi - cx0 + 1) * (per ? per : 1);
  };
  (void)clampx;
  d.plane = 0;
  if (r < R_YF) {                                   // x-faces (fx in [cx0, cx0+8], ey = cy0 + r)
    const int ey = cy0 + r;
    d.g0 = g.off_f[0] + ((long long)cx0 + (long long)(nx + 1) * ey) * N2;
    d.gs = (long long)(nx + 1) * ny * N2;
    d.slot = LL::O_XF + r * LL::XS; d.len = (TX + 1) * N2;
    const int lo = max(cx0, 1), hi = min(cx0 + TX, nx - 1);
    d.a = (lo - cx0) * N2; d.b = (hi - cx0 + 1) * N2;
    if (ey < 0 || ey >= ny) d.b = d.a;
  } else if (r < R_ZE) {                            // y-faces (ex in [cx0, cx0+8), fy = cy0 + q)
    const int fy = cy0 + (r - R_YF);
    d.g0 = g.off_f[1] + ((long long)cx0 + (long long)nx * fy) * N2;
    d.gs = (long long)nx * (ny + 1) * N2;
    d.slot = LL::O_YF + (r - R_YF) * LL::YS; d.len = TX * N2;
    const int lo = max(cx0, 0), hi = min(cx0 + TX - 1, nx - 1);
    d.a = (lo - cx0) * N2; d.b = (hi - cx0 + 1) * N2;
    if (fy < 1 || fy > ny - 1) d.b = d.a;
  } else if (r < R_ZF) {                            // z-edges (fx in [cx0, cx0+8], fy = cy0 + q)
    const int fy = cy0 + (r - R_ZE);
    d.g0 = g.off_e[2] + ((long long)cx0 + (long long)(nx + 1) * fy) * NI;
    d.gs = (long long)(nx + 1) * (ny + 1) * NI;
    d.slot = LL::O_ZE + (r - R_ZE) * LL::ZES; d.len = (TX + 1) * NI;
    const int lo = max(cx0, 1), hi = min(cx0 + TX, nx - 1);
    d.a = (lo - cx0) * NI; d.b = (hi - cx0 + 1) * NI;
    if (fy < 1 || fy > ny - 1) d.b = d.a;
  } else if (r < R_XE) {                            // z-faces (ex in [cx0, cx0+8), ey = cy0 + q), plane rows
    const int ey = cy0 + (r - R_ZF);
    d.g0 = g.off_f[2] + ((long long)cx0 + (long long)nx * ey) * N2;
    d.gs = (long long)nx * ny * N2;
    d.slot = LL::O_ZF + (r - R_ZF) * LL::ZS; d.len = TX * N2;
    const int lo = max(cx0, 0), hi = min(cx0 + TX - 1, nx - 1);
    d.a = (lo - cx0) * N2; d.b = (hi - cx0 + 1) * N2;
    if (ey < 0 || ey >= ny) d.b = d.a;
    d.plane = 1;
  } else if (r < R_YE) {                            // x-edges (ex in [cx0, cx0+8), fy = cy0 + q)
    const int fy = cy0 + (r - R_XE);
    d.g0 = g.off_e[0] + ((long long)cx0 + (long long)nx * fy) * NI;
    d.gs = (long long)nx * (ny + 1) * NI;
    d.slot = LL::O_PL + LL::PLX + (r - R_XE) * LL::XES; d.len = TX * NI;
    const int lo = max(cx0, 0), hi = min(cx0 + TX - 1, nx - 1);
    d.a = (lo - cx0) * NI; d.b = (hi - cx0 + 1) * NI;
    if (fy < 1 || fy > ny - 1) d.b = d.a;
    d.plane = 1;
  } else if (r < R_V) {                             // y-edges (fx in [cx0, cx0+8], ey = cy0 + q)
    const int ey = cy0 + (r - R_YE);
    d.g0 = g.off_e[1] + ((long long)cx0 + (long long)(nx + 1) * ey) * NI;
    d.gs = (long long)(nx + 1) * ny * NI;
    d.slot = LL::O_PL + LL::PLY + (r - R_YE) * LL::YES; d.len = (TX + 1) * NI;
    const int lo = max(cx0, 1), hi = min(cx0 + TX, nx - 1);
    d.a = (lo - cx0) * NI; d.b = (hi - cx0 + 1) * NI;
    if (ey < 0 || ey >= ny) d.b = d.a;
    d.plane = 1;
  } else {                                          // vertices (fx in [cx0, cx0+8], fy = cy0 + q)
    const int fy = cy0 + (r - R_V);
    d.g0 = g.off_v + (long long)cx0 + (long long)(nx + 1) * fy;
    d.gs = (long long)(nx + 1) * (ny + 1);
    d.slot = LL::O_PL + LL::PLV + (r - R_V) * LL::VS; d.len = TX + 1;
    const int lo = max(cx0, 1), hi = min(cx0 + TX, nx - 1);
    d.a = lo - cx0; d.b = hi - cx0 + 1;
    if (fy < 1 || fy > ny - 1) d.b = d.a;
    d.plane = 1;
  }
  if (d.b < d.a) d.b = d.a;
}

// smem offset of row r for layer / plane q (its slot, plane slots alternating with q)
template <int NI, int H>
__device__ __forceinline__ int row_off(const Row& d, int r, int q) {
  using LL = L<NI, H>;
  constexpr int R_ZF = TC<H>::R_ZF, R_XE = TC<H>::R_XE;
  int s = d.slot;
  if (r >= R_ZF) s += (q & 1) * (r < R_XE ? LL::PZ : LL::PLS);
  return s + (int)((d.g0 + (long long)q * d.gs) & 1);
}

// Bulk loads of one step, issued by warp 0 as one mbarrier transaction: the side rows of layer qs
// (if side), the plane rows of plane qa (if pa) and of plane qb (if pb); copy c = lane + 32 h over
// the list [side rows | plane rows of qa | plane rows of qb].
template <int NI, int H>
__device__ void issue_step(const V5Params& P, double* sm, const Row* rows, bool side, int qs, bool pa, int qa, bool za,
                           bool pb, int qb, bool zb, unsigned long long* mbar) {
  constexpr int NSIDE = TC<H>::NSIDE, NROWS = TC<H>::NROWS, NC = (NSIDE + 2 * (NROWS - NSIDE) + 31) / 32;
  const int lane = threadIdx.x & 31;
  unsigned bytes[NC];
  long long src[NC];
  int dst[NC];
#pragma unroll
  for (int h = 0; h < NC; ++h) {
    bytes[h] = 0u;
    src[h] = 0;
    dst[h] = 0;
    const int c = lane + 32 * h;
    if (c >= NSIDE + 2 * (NROWS - NSIDE)) continue;
    int r, q;
    bool on;
    if (c < NSIDE) { r = c; q = qs; on = side; }
    else if (c < NROWS) { r = c; q = qa; on = pa && !za; }
    else { r = c - (NROWS - NSIDE); q = qb; on = pb && !zb; }
    const Row& d = rows[r];
    if (!on || d.a >= d.b) continue;
    const long long gq = d.g0 + (long long)q * d.gs;
    const long long ga = gq + d.a, gb = gq + d.b;
    src[h] = ga & ~1LL;
    bytes[h] = (unsigned)(((gb + 1) & ~1LL) - src[h]) * 8u;
    dst[h] = row_off<NI, H>(d, r, q) + d.a - (int)(ga & 1);
  }
  unsigned tot = 0u;
#pragma unroll
  for (int h = 0; h < NC; ++h) tot += bytes[h];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  if (lane == 0) mbar_arrive_tx(mbar, tot);
  __syncwarp();
#pragma unroll
  for (int h = 0; h < NC; ++h)
    if (bytes[h]) bulk_g2s(sm + dst[h], P.x + src[h], bytes[h], mbar);
}

// zero the invalid / Dirichlet parts of rows [r0, r1) for layer / plane q (after the wait)
template <int NI, int H>
__device__ __noinline__ void fix_rows(double* sm, const Row* rows, int r0, int r1, int q, bool zplane) {
#pragma unroll 1
  for (int r = r0 + (threadIdx.x >> 5); r < r1; r += TC<H>::NT / 32) {
    const Row& d = rows[r];
    double* b = sm + row_off<NI, H>(d, r, q);
    const bool none = d.a >= d.b || (d.plane && zplane);
    const int a = none ? d.len : d.a, e = none ? d.len : d.b;
    for (int t = threadIdx.x & 31; t < a; t += 32) b[t] = 0.0;
    for (int t = e + (threadIdx.x & 31); t < d.len; t += 32) b[t] = 0.0;
  }
}

__device__ __forceinline__ bool rows_complete(const Row* rows, int r0, int r1) {
#pragma unroll 1
  for (int r = r0; r < r1; ++r)
    if (rows[r].a != 0 || rows[r].b != rows[r].len) return false;
  return true;
}

// ---- per-step view of the tile in shared memory --------------------------------------------
// Row r of a kind starts at sm + offset table entry (offsets of the step's layer / planes, in
// shared memory: lane-dependent rows are then one shared load, not local-memory pointer arrays).
template <int H>
struct View {
  using C = TC<H>;
  const double* sm;
  const int* rs;   // side rows, layer l
  const int* rb;   // plane rows, plane l
  const int* rt;   // plane rows, plane l + 1
  __device__ __forceinline__ const double* xf(int r) const { return sm + rs[C::R_XF + r]; }   // x-faces (fx in [cx0, cx0+8])
  __device__ __forceinline__ const double* yf(int r) const { return sm + rs[C::R_YF + r]; }   // y-faces (ex in [cx0, cx0+8))
  __device__ __forceinline__ const double* ze(int r) const { return sm + rs[C::R_ZE + r]; }   // z-edges (fx)
  __device__ __forceinline__ const double* zf(int kb, int r) const { return sm + (kb ? rt : rb)[C::R_ZF + r]; }
  __device__ __forceinline__ const double* xe(int kb, int r) const { return sm + (kb ? rt : rb)[C::R_XE + r]; }
  __device__ __forceinline__ const double* ye(int kb, int r) const { return sm + (kb ? rt : rb)[C::R_YE + r]; }
  __device__ __forceinline__ const double* vv(int kb, int r) const { return sm + (kb ? rt : rb)[C::R_V + r]; }
};

// ---- edge / vertex primary parts (entity-centric, owned entities) -----------------------------
// x-edge (ex, fy) at plane P = l + kb, node i: layer l's two elements (ey = fy - 1, fy) contribute
//   2 [d0 w0^2 + d1 w0^2 Lam_i + (d2 + d3) w0 K00] u + 2 d1 w0^2 (a0_i V(ex) + ap_i V(ex + 1))
//   + d2 w0 [sum_j ap_j Fz(ex, fy - 1)(i, j) + sum_j a0_j Fz(ex, fy)(i, j) + K0p (u(fy - 1) + u(fy + 1))]
//   + 2 d3 w0 [sum_k at_k Fy(ex, fy, l)(i, k) + K0p u(other plane)],  at = a0 (kb = 0) or ap (kb = 1)
// (K~ rows 0 / p = (K00, a0, K0p) / (K0p, ap, K00), interior rows (a0_m, Lam_m, ap_m); M~ = diag(w0, 1..1, w0),
// P:381-405).  y-edges by x <-> y symmetry; vertices and z-edges likewise (see v6_make_coef).
template <int NI>
struct Edge {
  // line sum over m of w_m f[m * stride]
  __device__ static __forceinline__ double lsum(const double* w, const double* f, int stride) {
    double s = 0.0;
#pragma unroll
    for (int m = 0; m < NI; ++m) s = fma(w[m], f[m * stride], s);
    return s;
  }
};

// ---- edge / vertex stencils of one step (entity-centric; owned (ix, iy) in [1, 8) x [1, 4)) ----
// x-edges, y-edges and vertices of plane l are final (aeb: the partial sums of layer l - 1) and
// those of plane l + 1 get layer l's part (aet); z-edges of layer l are final.  One loop per entity
// kind (item t -> owned entity e = t / NI, node c = t % NI; consecutive t are consecutive skeleton
// entries of a row, so the stores coalesce).  Shared by the v5 and v6 kernels.
template <int NI, bool DOT, int H>
__device__ __forceinline__ void edge_phase(const V5Params& P, const View<H>& V, const double* sa0, const double* sap,
                                           const double* czu, const double* cxu, const double* cyu, double* aeb,
                                           double* aet, int cx0, int cy0, int l, bool lay, bool fin_l, bool fin_t,
                                           double& dot) {
  constexpr int N2 = NI * NI;
  const Geom& g = P.g;
  const V5Coef& cf = P.cf;
  const int tid = threadIdx.x, nthreads = blockDim.x;
  constexpr int NO = TC<H>::NO;
    {
      constexpr int NE1 = NO * NI;
      const int nx = g.nx, ny = g.ny;
      const double k0p = cf.sc[15];
      // z-edges (fx, fy) of layer l, node k (final)
      if (lay) {
        for (int t = tid; t < NE1; t += nthreads) {
          const int e = t / NI, c = t - e * NI, jx = e % OX + 1, jy = e / OX + 1;
          const int fx = cx0 + jx, fy = cy0 + jy;
          const double* Z = V.ze(jy) + jx * NI;
          const double u = Z[c];
          const double* Fy0 = V.yf(jy) + (jx - 1) * N2 + c * NI;    // y-face (fx - 1, fy), (i, k) at fixed k
          const double* Fx0 = V.xf(jy - 1) + jx * N2 + c * NI;     // x-face (fx, fy - 1), (j, k) at fixed k
          const double* Fx1 = V.xf(jy) + jx * N2 + c * NI;         // x-face (fx, fy)
          const double ly = Edge<NI>::lsum(sap, Fy0, 1) + Edge<NI>::lsum(sa0, Fy0 + N2, 1);
          const double lx = Edge<NI>::lsum(sap, Fx0, 1) + Edge<NI>::lsum(sa0, Fx1, 1);
          const double nxs = Z[c - NI] + Z[c + NI];
          const double nys = V.ze(jy - 1)[jx * NI + c] + V.ze(jy + 1)[jx * NI + c];
          const double vb = V.vv(0, jy)[jx], vt = V.vv(1, jy)[jx];
          // 4 [d0 w0^2 + (d1 + d2) w0 K00 + d3 w0^2 Lam_k] u + 4 d3 w0^2 (a0_k V_b + ap_k V_t)
          // + 2 d1 w0 [y-face i-lines + K0p (u(fx-1) + u(fx+1))] + 2 d2 w0 [x-face j-lines + K0p (u(fy-1) + u(fy+1))]
          double val = czu[c] * u + cf.sc[0] * fma(sa0[c], vb, sap[c] * vt) + cf.sc[1] * fma(k0p, nxs, ly) +
                       cf.sc[2] * fma(k0p, nys, lx);
          if (DOT && fin_l) dot = fma(u, val, dot);
          if (fin_l && fx <= nx && fy <= ny) {
            if (fx == 0 || fx == nx || fy == 0 || fy == ny) val = 0.0;
            P.y[g.off_e[2] + ((long long)fx + (long long)(nx + 1) * (fy + (long long)(ny + 1) * l)) * NI + c] = val;
          }
        }
      }
      // x-edges (ex, fy) and y-edges (fx, ey) of planes l (final) and l + 1 (partial), node c
      for (int t = tid; t < 2 * NE1; t += nthreads) {
        const bool xk = t < NE1;
        const int tt = xk ? t : t - NE1;
        const int e = tt / NI, c = tt - e * NI, jx = e % OX + 1, jy = e / OX + 1;
        const int fx = cx0 + jx, fy = cy0 + jy;
        double* const ab = aeb + (xk ? 0 : NE1) + tt;
        double* const at = aet + (xk ? 0 : NE1) + tt;
        double p0 = 0.0, p1 = 0.0;
        if (lay) {
          const double* U0 = (xk ? V.xe(0, jy) : V.ye(0, jy)) + jx * NI;
          const double* U1 = (xk ? V.xe(1, jy) : V.ye(1, jy)) + jx * NI;
          // the layer's face along k: y-face (ex, fy) (x-edge, entries (i, k)) / x-face (fx, ey) (y-edge, (j, k))
          const double* Fl = (xk ? V.yf(jy) : V.xf(jy)) + jx * N2 + c;
          const double lk0 = Edge<NI>::lsum(sa0, Fl, NI), lk1 = Edge<NI>::lsum(sap, Fl, NI);
          const double cu = xk ? cxu[c] : cyu[c];
          // x-edge: 2 d1 w0^2, d2 w0, 2 d3 w0;  y-edge: 2 d2 w0^2, d1 w0, 2 d3 w0
          const double sv = xk ? cf.sc[3] : cf.sc[6], sl = xk ? cf.sc[4] : cf.sc[7], sk = xk ? cf.sc[5] : cf.sc[8];
#pragma unroll
          for (int kb = 0; kb < 2; ++kb) {
            const double* U = kb ? U1 : U0;
            const double* Uo = kb ? U0 : U1;
            // z-faces of plane l + kb across the edge: x-edge (ex, fy-1) / (ex, fy), j-line at i = c;
            // y-edge (fx-1, ey) / (fx, ey), i-line at j = c
            const double* Fa = xk ? V.zf(kb, jy - 1) + jx * N2 + c : V.zf(kb, jy) + (jx - 1) * N2 + c * NI;
            const double* Fb = xk ? V.zf(kb, jy) + jx * N2 + c : Fa + N2;
            const int st = xk ? NI : 1;
            const double lz = Edge<NI>::lsum(sap, Fa, st) + Edge<NI>::lsum(sa0, Fb, st);
            const double nb = xk ? V.xe(kb, jy - 1)[jx * NI + c] + V.xe(kb, jy + 1)[jx * NI + c] : U[c - NI] + U[c + NI];
            const double v1 = xk ? V.vv(kb, jy)[jx + 1] : V.vv(kb, jy + 1)[jx];
            const double vc = fma(sa0[c], V.vv(kb, jy)[jx], sap[c] * v1);
            const double pv = cu * U[c] + sv * vc + sl * fma(k0p, nb, lz) + sk * fma(k0p, Uo[c], kb ? lk1 : lk0);
            if (kb == 0) p0 = pv; else p1 = pv;
          }
          if (DOT) {
            if (fin_l) dot = fma(U0[c], p0, dot);
            if (fin_t) dot = fma(U1[c], p1, dot);
          }
        }
        double val = *ab + p0;
        *at = p1;
        if (fin_l) {
          const bool zd = zdir(g, l);
          if (xk && fx < nx && fy <= ny) {
            if (zd || fy == 0 || fy == ny) val = 0.0;
            P.y[g.off_e[0] + ((long long)fx + (long long)nx * (fy + (long long)(ny + 1) * l)) * NI + c] = val;
          } else if (!xk && fx <= nx && fy < ny) {
            if (zd || fx == 0 || fx == nx) val = 0.0;
            P.y[g.off_e[1] + ((long long)fx + (long long)(nx + 1) * (fy + (long long)ny * l)) * NI + c] = val;
          }
        }
      }
      // vertices (fx, fy) of planes l (final) and l + 1 (partial)
      for (int e = tid; e < NO; e += nthreads) {
        const int jx = e % OX + 1, jy = e / OX + 1;
        const int fx = cx0 + jx, fy = cy0 + jy;
        double* const ab = aeb + 2 * NE1 + e;
        double* const at = aet + 2 * NE1 + e;
        double p0 = 0.0, p1 = 0.0;
        if (lay) {
          const double* Z = V.ze(jy) + jx * NI;    // z-edge (fx, fy) of layer l
          const double lk0 = Edge<NI>::lsum(sa0, Z, 1), lk1 = Edge<NI>::lsum(sap, Z, 1);
#pragma unroll
          for (int kb = 0; kb < 2; ++kb) {
            const double* Vr = V.vv(kb, jy);
            const double u = Vr[jx], uo = V.vv(1 - kb, jy)[jx];
            const double lx = Edge<NI>::lsum(sap, V.xe(kb, jy) + (jx - 1) * NI, 1) + Edge<NI>::lsum(sa0, V.xe(kb, jy) + jx * NI, 1);
            const double ly = Edge<NI>::lsum(sap, V.ye(kb, jy - 1) + jx * NI, 1) + Edge<NI>::lsum(sa0, V.ye(kb, jy) + jx * NI, 1);
            const double nxs = Vr[jx - 1] + Vr[jx + 1], nys = V.vv(kb, jy - 1)[jx] + V.vv(kb, jy + 1)[jx];
            // 4 (d0 w0^3 + (d1 + d2 + d3) w0^2 K00) u + 2 d1 w0^2 [x-edge lines + K0p (u(fx-1) + u(fx+1))]
            // + 2 d2 w0^2 [y-edge lines + K0p (...)] + 4 d3 w0^2 [z-edge line + K0p u(other plane)]
            const double pv = cf.sc[9] * u + cf.sc[10] * fma(k0p, nxs, lx) + cf.sc[11] * fma(k0p, nys, ly) +
                              cf.sc[12] * fma(k0p, uo, kb ? lk1 : lk0);
            if (kb == 0) p0 = pv; else p1 = pv;
            if (DOT && (kb == 0 ? fin_l : fin_t)) dot = fma(u, pv, dot);
          }
        }
        double val = *ab + p0;
        *at = p1;
        if (fin_l && fx <= nx && fy <= ny) {
          if (zdir(g, l) || fx == 0 || fx == nx || fy == 0 || fy == ny) val = 0.0;
          P.y[g.off_v + (long long)fx + (long long)(nx + 1) * (fy + (long long)(ny + 1) * l)] = val;
        }
      }
    }
}

// =============================================================================================
// Operator v6 (same tiles, rows, loads and edge stencils as v5): uniform class lanes.
//
// v5 runs one parity class per warp: eight different instruction streams per CTA (16 per SM),
// which measured instruction-fetch bound (ncu: no_instruction 8 stall cycles per issue), plus the
// pair coupling of the hand-over.  v6 maps lane = (element, class): a warp holds a 2 x 2 block of
// elements x 8 classes, every warp runs the same code (classes padded to n0^3 points with zero
// coefficients, so the padded points add exact zeros), and the three pair exchanges of a class are
// warp shuffles (xor 4 / 2 / 1).  Faces shared by the two elements of a block are assembled with
// a lane shuffle; the W / S faces whose other element is in the neighbour block take that part
// from a small shared buffer (XB / YB) in the store pass.  z-faces are assembled in global memory:
// step l stores plane l + 1 as (primary + condensed) of layer l, and step l + 1 adds layer l + 1's
// part to it (the value is written and re-read by the same thread ~one step later, so it stays in
// L2 and costs no DRAM traffic).  The x- / y-face primaries are computed entity-centrically into
// the owned accumulators before the class phase.
// =============================================================================================
// smallest k stride >= pj * p1 such that {si + pj sj + pk sk} (si, sj, sk in {0, 1}) are distinct mod 16
constexpr bool di_ok(int pj, int pk) {
  int o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int c = 0; c < 8; ++c) o[c] = ((c & 1) + pj * ((c >> 1) & 1) + pk * (c >> 2)) % 16;
  for (int a = 0; a < 8; ++a)
    for (int b = a + 1; b < 8; ++b)
      if (o[a] == o[b]) return false;
  return true;
}
constexpr int di_pk(int pj, int p1) {
  for (int pk = pj * p1; pk < pj * p1 + 16; ++pk)
    if (di_ok(pj, pk)) return pk;
  return pj * p1;
}

template <int NI, int H>
struct L6 {
  using B = L<NI, H>;
  using C = TC<H>;
  static constexpr int N2 = NI * NI;
  static constexpr int M = (NI + 1) / 2;                   // padded class extent
  static constexpr int ACC = even(C::NO * N2);
  static constexpr int O_AX = B::END;                      // owned x-faces of the layer
  static constexpr int O_AY = O_AX + ACC;                  // owned y-faces of the layer
  static constexpr int O_XB = O_AY + ACC;                  // [OY][3][N2]: E parts of elements ix = 1, 3, 5, rows >= 1
  static constexpr int NYB = H / 2 - 1;                    // rows iy = 1, 3, .., H - 3 send N parts across blocks
  static constexpr int O_YB = O_XB + even(C::OY * 3 * N2); // [NYB][OX][N2]
  static constexpr int O_AE = O_YB + even(NYB * OX * N2);  // edge accumulators, 2 planes
  static constexpr int AES = even(2 * C::NO * NI + C::NO); // per plane: x-edges | y-edges | vertices
  static constexpr int O_TAB = O_AE + 2 * AES;             // a0, ap, czu, cxu, cyu (8 each)
  static constexpr int O_CT = O_TAB + 40;                  // class tables (see k_apply_v6)
  static constexpr int CT_C = 0, CT_FDZ = 24, CT_EF1 = CT_FDZ + even(N2), CT_FDX = CT_EF1 + 16,
                       CT_FDY = CT_FDX + even(N2), CT_EF2 = CT_FDY + even(N2), CT_N = CT_EF2 + 24;
  // D^{-1}(i, j, k) at i + P1 (j + P1 k), P1 = NI + 1: padded class points (index NI in some
  // direction) read a 0 there, so they contribute exact zeros to every sum and to the energy
  // (with the unpadded stride NI they would alias real entries)
  static constexpr int P1 = NI + 1;
  // j / k strides of the table: the 8 class bases si + PJ sj + PK sk of a warp's lanes fall on 8
  // distinct 8-byte bank pairs (distinct mod 16 doubles), so a class-phase D^{-1} load is one
  // wavefront (with PK = P1^2 the s_k = 0 / 1 classes collided: 2-way conflicts, r2s ncu)
  static constexpr int PJ = P1;
  static constexpr int PK = di_pk(P1, P1);
  static constexpr int DIN = even(PK * P1);
  static constexpr int O_DI = O_CT + CT_N;
  static constexpr int O_SCR = O_DI + DIN;                 // scratch row of stores that own nothing
  static constexpr int O_AZ = O_SCR + even(N2);            // owned z-faces of plane l
  static constexpr int TOTAL = O_AZ + ACC;
  static constexpr int CTAS = H == 4 ? 2 : 1;              // CTAs per SM the layout is sized for
  // per SM: CTAS x (dynamic + ~2 KB static + 1 KB reserved) <= 228 KB
  static_assert(CTAS * (TOTAL * 8 + 2048 + 1024) <= 228 * 1024, "v6 shared memory");
};

template <int NI, bool DOT, int H>
__global__ void __launch_bounds__(64 * H, H == 4 ? 2 : 1) k_apply_v6(const __grid_constant__ V5Params P) {
  using LL = L<NI, H>;
  using L6T = L6<NI, H>;
  using C = TC<H>;
  constexpr int N2 = NI * NI, M = L6T::M;
  constexpr int OY = C::OY, NO = C::NO, NT = C::NT, NROWS = C::NROWS, NSIDE = C::NSIDE;
  if (P.done != nullptr && *P.done != 0.0) return;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ Row rows[NROWS];
  __shared__ int rofs[2][NROWS];
  __shared__ double sred[NT / 32];
  const Geom& g = P.g;
  const V5Coef& cf = P.cf;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int item = blockIdx.x;
  const int ntile = P.ntx * P.nty;
  const int seg = item / ntile, tile = item - seg * ntile;
  const int tx = tile % P.ntx, ty = tile / P.ntx;
  const int x0 = tx * OX, y0 = ty * OY, cx0 = x0 - 1, cy0 = y0 - 1;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int lfin0 = seg * P.zseg;
  const int lbeg = seg > 0 ? lfin0 - 1 : 0;
  const int lend = seg == P.nseg - 1 ? nz : min(nz, lfin0 + P.zseg) - 1;

  if (item == 0) {   // padding entries of y are written as 0 by the first CTA
    const long long ends[7] = {g.off_f[0] + g.n_f[0] * N2, g.off_f[1] + g.n_f[1] * N2, g.off_f[2] + g.n_f[2] * N2,
                               g.off_e[0] + g.n_e[0] * NI, g.off_e[1] + g.n_e[1] * NI, g.off_e[2] + g.n_e[2] * NI,
                               g.off_v + g.n_v};
    const long long nexts[7] = {g.off_f[1], g.off_f[2], g.off_e[0], g.off_e[1], g.off_e[2], g.off_v, g.n_total};
#pragma unroll 1
    for (int q = 0; q < 7; ++q)
      for (long long i = ends[q] + tid; i < nexts[q]; i += NT) P.y[i] = 0.0;
  }
  // the input rows are read beyond their valid ends by padded class points (times a zero
  // coefficient): every slot starts as finite zeros
  for (int t = tid; t < LL::END; t += NT) sm[t] = 0.0;
  double* const sa0 = sm + L6T::O_TAB;
  double* const sap = sa0 + 8;
  double* const czu = sa0 + 16;
  double* const cxu = sa0 + 24;
  double* const cyu = sa0 + 32;
  double* const ct = sm + L6T::O_CT;
  double* const sdi = sm + L6T::O_DI;
  if (tid < 8) {
    const bool in = tid < NI;
    sa0[tid] = cf.a0[tid];
    sap[tid] = cf.a0[tid] * cf.sig[tid];
    czu[tid] = cf.czu[tid];
    cxu[tid] = cf.cxu[tid];
    cyu[tid] = cf.cyu[tid];
    for (int d = 0; d < 3; ++d) {
      ct[L6T::CT_C + 8 * d + tid] = in ? cf.c[d][tid] : 0.0;
      ct[L6T::CT_EF2 + 8 * d + tid] = in ? cf.ef2[d][tid] : 0.0;
    }
    for (int d = 0; d < 2; ++d) ct[L6T::CT_EF1 + 8 * d + tid] = in ? cf.ef1[d][tid] : 0.0;
  }
  for (int t = tid; t < N2; t += NT) {
    ct[L6T::CT_FDZ + t] = cf.fdz[t];
    ct[L6T::CT_FDX + t] = cf.fdx[t];
    ct[L6T::CT_FDY + t] = cf.fdy[t];
  }
  for (int t = tid; t < L6T::DIN; t += NT) {
    const int k = t / L6T::PK, r = t - k * L6T::PK, j = r / L6T::PJ, i = r - j * L6T::PJ;
    sdi[t] = (i < NI && j < NI && k < NI) ? cf.dinv[i + NI * (j + NI * k)] : 0.0;
  }
  if (tid < NROWS) make_row<NI, H>(g, tid, cx0, cy0, rows[tid]);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = tid; t < L6T::AES; t += NT) sm[L6T::O_AE + (lbeg & 1) * L6T::AES + t] = 0.0;
  __syncthreads();
  const bool side_ok = rows_complete(rows, 0, NSIDE);
  const bool plane_ok = rows_complete(rows, NSIDE, NROWS);
  if (tid < NROWS) {
    rofs[lbeg & 1][tid] = row_off<NI, H>(rows[tid], tid, lbeg);
    if (tid >= NSIDE) rofs[(lbeg + 1) & 1][tid] = row_off<NI, H>(rows[tid], tid, lbeg + 1);
  }
  fence_proxy_async();   // the zero fill above precedes the bulk copies into the same rows
  __syncthreads();
  if (warp == 0)
    issue_step<NI, H>(P, sm, rows, lbeg < nz, lbeg, true, lbeg, zdir(g, lbeg), lbeg < nz, lbeg + 1, zdir(g, lbeg + 1),
                   &mbar);
  __syncthreads();
  unsigned phase = 0;
  bool pending = true;
  bool first_fix = !plane_ok || zdir(g, lbeg);
  double dot = 0.0;

  // ---- lane = (element of the warp's 2 x 2 block, parity class)
  const int cls = lane & 7, si = cls >> 2, sj = (cls >> 1) & 1, sk = cls & 1;
  // half-warp = one column of the block (dy = 0, 1): with row strides = 4 mod 16 doubles its 8
  // distinct face addresses (2 elements x 4 (s_a, s_b)) fall on disjoint bank pairs
  const int dy = (lane >> 3) & 1, dx = lane >> 4, bx = warp & 3, by = warp >> 2;
  const int ix = 2 * bx + dx, iy = 2 * by + dy;
  const int CI = (NI - si + 1) >> 1, CJ = (NI - sj + 1) >> 1, CK = (NI - sk + 1) >> 1;
  const double gi = si ? -1.0 : 1.0, gj = sj ? -1.0 : 1.0, gk = sk ? -1.0 : 1.0;
  const int ex = cx0 + ix, ey = cy0 + iy;
  const bool own = ix >= 1 && iy >= 1 && ex < nx && ey < ny;   // owned element (its W / S / B faces)
  const int o_lane = (iy - 1) * OX + (ix - 1);
  double c1r[M];
#pragma unroll
  for (int ii = 0; ii < M; ++ii) c1r[ii] = ct[L6T::CT_C + si + 2 * ii];

  for (int l = lbeg; l <= lend; ++l) {
    const bool lay = l < nz;
    if (pending) {
      mbar_wait(&mbar, phase);
      phase ^= 1;
      pending = false;
    }
    const bool fix = first_fix || (lay && (!side_ok || !plane_ok || zdir(g, l + 1)));
    if (fix) {
      if (first_fix) fix_rows<NI, H>(sm, rows, NSIDE, NROWS, l, zdir(g, l));
      if (lay) {
        fix_rows<NI, H>(sm, rows, 0, NSIDE, l, false);
        fix_rows<NI, H>(sm, rows, NSIDE, NROWS, l + 1, zdir(g, l + 1));
      }
      __syncthreads();
    }
    first_fix = false;
    View<H> V{sm, rofs[l & 1], rofs[l & 1], rofs[(l + 1) & 1]};
    const bool fin_l = l >= lfin0;
    const bool fin_t = l + 1 <= lend;
    double* const aeb = sm + L6T::O_AE + (l & 1) * L6T::AES;
    double* const aet = sm + L6T::O_AE + ((l + 1) & 1) * L6T::AES;
    edge_phase<NI, DOT, H>(P, V, sa0, sap, czu, cxu, cyu, aeb, aet, cx0, cy0, l, lay, fin_l, fin_t, dot);
    double* const AX = sm + L6T::O_AX;
    double* const AY = sm + L6T::O_AY;
    double* const XB = sm + L6T::O_XB;
    double* const YB = sm + L6T::O_YB;
    double* const scr = sm + L6T::O_SCR;
    double* const AZ = sm + L6T::O_AZ;
    // plane l's owned z-faces start from what step l - 1 stored there (layer l - 1's part; nothing
    // below a segment's first plane): one warp per row, coalesced, so their L2 latency overlaps
    if (lay && fin_l) {
      for (int oy = warp; oy < OY; oy += NT / 32) {
        const int eyz = y0 + oy;
        const bool below = l > lbeg && eyz < ny;
        const int cnt = below ? min(OX, nx - x0) : 0;
        const double* src = P.y + g.off_f[2] + ((long long)x0 + (long long)nx * (eyz + (long long)ny * l)) * N2;
        double* dst = AZ + oy * OX * N2;
        for (int t = lane; t < OX * N2; t += 32) dst[t] = t < cnt * N2 ? src[t] : 0.0;
      }
    }
    __syncthreads();   // plane-l accumulator initialised (and every edge line read)
    if (lay) {
      // ======== condensed part: this lane's class of its element (padded to M^3 points)
      const double* W = V.xf(iy) + ix * N2 + sj + NI * sk;    // x-face entries (j, k) = (sj + 2jj, sk + 2kk)
      const double* E = W + N2;
      const double* S = V.yf(iy) + ix * N2 + si + NI * sk;    // y-face entries (i, k)
      const double* Nn = V.yf(iy + 1) + ix * N2 + si + NI * sk;
      const double* Bf = V.zf(0, iy) + ix * N2 + si + NI * sj;   // z-face entries (i, j)
      const double* Tf = V.zf(1, iy) + ix * N2 + si + NI * sj;
      const double* Dc = sdi + si + L6T::PJ * sj + L6T::PK * sk;   // D^{-1}(si + 2ii, sj + 2jj, sk + 2kk)
      // primaries (Eq. 26 generalised) of the faces this lane stores: x (s_i = 0 lanes, entries (j, k)),
      // y (s_j = 0, entries (i, k)), plane-l z-face (s_k = 0) / plane-(l+1) z-face (s_k = 1) entries (i, j)
      const double* Wm = W - N2;                                  // x-face fx - 1 (same entries)
      const double* Sm = V.yf(iy > 0 ? iy - 1 : 0) + ix * N2 + si + NI * sk;   // y-face fy - 1
      const double* zsx = V.ze(iy) + ix * NI + sk;                // z-edge (fx, ey), (fx, ey + 1): k = sk + 2kk
      const double* znx = V.ze(iy + 1) + ix * NI + sk;
      const double* ybx = V.ye(0, iy) + ix * NI + sj;             // y-edge (fx, ey) at planes l, l + 1: j
      const double* ytx = V.ye(1, iy) + ix * NI + sj;
      const double* xby = V.xe(0, iy) + ix * NI + si;             // x-edge (ex, fy) at planes l, l + 1: i
      const double* xty = V.xe(1, iy) + ix * NI + si;
      const double* fdxl = ct + L6T::CT_FDX + sj + NI * sk;
      const double* fdyl = ct + L6T::CT_FDY + si + NI * sk;
      const double* e2x = ct + L6T::CT_EF2 + 8 + sj;              // 2 d2 w0 a0_j
      const double* e3x = ct + L6T::CT_EF2 + 16 + sk;             // 2 d3 w0 a0_k
      const double* e1y = ct + L6T::CT_EF2 + si;                  // 2 d1 w0 a0_i
      const bool pd = DOT && own && fin_l;                        // this lane's primaries count in x . A x
      // accumulator rows of this lane's stores (scratch for the lanes / entries that own nothing)
      double* const axr = (si == 0 && own) ? AX + o_lane * N2 + sj + NI * sk
                          : ((si == 1 && dx == 1 && bx < 3 && iy >= 1) ? XB + ((iy - 1) * 3 + bx) * N2 + sj + NI * sk : scr);
      double* const ayr = (sj == 0 && own) ? AY + o_lane * N2 + si + NI * sk
                          : ((sj == 1 && dy == 1 && by < L6T::NYB && ix >= 1) ? YB + (by * OX + ix - 1) * N2 + si + NI * sk
                                                                                : scr);
      double zin[M][M], qz[M][M];
#pragma unroll
      for (int ii = 0; ii < M; ++ii)
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
          zin[ii][jj] = fma(gk, Tf[2 * ii + 2 * NI * jj], Bf[2 * ii + 2 * NI * jj]);
          qz[ii][jj] = 0.0;
        }
      double en = 0.0;
#pragma unroll
      for (int kk = 0; kk < M; ++kk) {
        const double c3 = ct[L6T::CT_C + 16 + sk + 2 * kk];
        const double zx = fma(gj, znx[2 * kk], zsx[2 * kk]);      // x primaries: Zs + s_j Zn at k
        const double zy = fma(gi, zsx[NI + 2 * kk], zsx[2 * kk]); // y primaries: Zw + s_i Ze at k
        double yin[M], qy[M];
#pragma unroll
        for (int ii = 0; ii < M; ++ii) {
          yin[ii] = fma(gj, Nn[2 * ii + 2 * NI * kk], S[2 * ii + 2 * NI * kk]);
          qy[ii] = 0.0;
        }
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
          const double c2 = ct[L6T::CT_C + 8 + sj + 2 * jj];
          const int ox = 2 * jj + 2 * NI * kk;
          const double wv = W[ox], evv = E[ox];
          const double xin = fma(gi, evv, wv);
          double qx = 0.0;
#pragma unroll
          for (int ii = 0; ii < M; ++ii) {
            const double u = fma(c1r[ii], xin, fma(c2, yin[ii], c3 * zin[ii][jj]));
            const double v = u * Dc[2 * ii + 2 * L6T::PJ * jj + 2 * L6T::PK * kk];
            if (DOT) en = fma(u, v, en);
            qx = fma(c1r[ii], v, qx);
            qy[ii] = fma(c2, v, qy[ii]);
            qz[ii][jj] = fma(c3, v, qz[ii][jj]);
          }
          // x pair (s_i = 0 / 1, lane ^ 4): W part -(Q0 + Q1), E part -(Q0 - Q1); the owned W face of
          // element ix gets W(ix) + E(ix - 1) (lane - 16 inside the block, XB across blocks)
          const double qp = __shfl_xor_sync(0xffffffffu, qx, 4);
          const double wpart = -(qx + qp);
          const double ep = si ? qx - qp : qp - qx;        // -(Q0 - Q1), Q0 on the s_i = 0 lane
          const double em = __shfl_up_sync(0xffffffffu, ep, 16);   // element ix - 1
          const bool valid = jj < CJ && kk < CK;
          // x primary of entry (j, k): self (2 elements), opposite faces fx -/+ 1, bounding edges
          const double yx = fma(gk, ytx[2 * jj], ybx[2 * jj]);
          const double pr = fma(fdxl[ox], wv, fma(cf.k0p[0], Wm[ox] + evv, fma(e2x[2 * jj], zx, e3x[2 * kk] * yx)));
          if (pd && si == 0 && valid) dot = fma(wv, pr, dot);
          double* const dst = valid ? axr + ox : scr;
          *dst = si == 0 ? pr + wpart + (dx ? em : 0.0) : ep;
        }
        // y pair (s_j = 0 / 1, lane ^ 2): S part -(Q0 + Q1), N part -(Q0 - Q1); the owned S face of
        // element iy gets S(iy) + N(iy - 1) (lane - 8 inside the block, YB across blocks)
#pragma unroll
        for (int ii = 0; ii < M; ++ii) {
          const double qp = __shfl_xor_sync(0xffffffffu, qy[ii], 2);
          const double spart = -(qy[ii] + qp);
          const double np = sj ? qy[ii] - qp : qp - qy[ii];    // -(Q0 - Q1)
          const double nm = __shfl_up_sync(0xffffffffu, np, 8);     // element iy - 1
          const bool valid = ii < CI && kk < CK;
          const int oy = 2 * ii + 2 * NI * kk;
          const double sv = S[oy];
          const double xy = fma(gk, xty[2 * ii], xby[2 * ii]);
          const double pr = fma(fdyl[oy], sv, fma(cf.k0p[1], Sm[oy] + Nn[oy], fma(e1y[2 * ii], zy, e3x[2 * kk] * xy)));
          if (pd && sj == 0 && valid) dot = fma(sv, pr, dot);
          double* const dst = valid ? ayr + oy : scr;
          *dst = sj == 0 ? pr + spart + (dy ? nm : 0.0) : np;
        }
      }
      // z pair (s_k = 0 / 1, lane ^ 1): B part -(Q0 + Q1) on plane l, T part -(Q0 - Q1) on plane l + 1.
      // Lane s_k = 0 adds its primary + B part to the owned plane-l accumulator; lane s_k = 1 stores
      // plane l + 1 as its primary + T part (step l + 1 adds layer l + 1's part to it).
      {
        const int kb = sk;
        double* const azr = (sk == 0 && own) ? AZ + o_lane * N2 + si + NI * sj : scr;
        const bool st = sk == 1 && own && fin_t;
        const bool zd = zdir(g, l + kb);
        const bool cnt = DOT && own && (kb ? fin_t : fin_l) && !zd;
        const double* Yw = V.ye(kb, iy) + ix * NI + sj;   // y-edges (ex, ey), (ex + 1, ey) at plane l + kb: j
        const double* Xs = V.xe(kb, iy) + ix * NI + si;   // x-edges (ex, fy = ey), (ex, ey + 1): i
        const double* Xn = V.xe(kb, iy + 1) + ix * NI + si;
        const double* U = kb ? Tf : Bf;
        const double* Uo = kb ? Bf : Tf;
        const double* fdzl = ct + L6T::CT_FDZ + si + NI * sj;
        const double* e1z = ct + L6T::CT_EF1 + si;
        const double* e2z = ct + L6T::CT_EF1 + 8 + sj;
        double* const yrow = P.y + g.off_f[2] + ((long long)ex + (long long)nx * (ey + (long long)ny * (l + 1))) * N2 +
                             si + NI * sj;
#pragma unroll
        for (int ii = 0; ii < M; ++ii)
#pragma unroll
          for (int jj = 0; jj < M; ++jj) {
            const double qp = __shfl_xor_sync(0xffffffffu, qz[ii][jj], 1);
            const bool valid = ii < CI && jj < CJ;
            const int oz = 2 * ii + 2 * NI * jj;
            const double u = U[oz];
            const double pr = fma(fdzl[oz], u, fma(cf.k0p[2], Uo[oz], fma(e1z[2 * ii], fma(gi, Yw[NI + 2 * jj], Yw[2 * jj]),
                                                                       e2z[2 * jj] * fma(gj, Xn[2 * ii], Xs[2 * ii]))));
            if (cnt && valid) dot = fma(u, pr, dot);
            if (sk == 0) {
              double* const d = valid ? azr + oz : scr;
              *d = *d + pr - (qz[ii][jj] + qp);
            } else if (st && valid) {
              yrow[oz] = zd ? 0.0 : pr + (qz[ii][jj] - qp);   // T: -(Q0 - Q1), Q0 on the s_k = 0 lane
            }
          }
      }
      if (DOT && own && fin_l) dot -= en;
    }
    __syncthreads();   // accumulators final; every input row of step l dead
    if (l + 1 <= lend && l + 1 < nz) {
      if (tid < NROWS) {
        if (tid < NSIDE) rofs[(l + 1) & 1][tid] = row_off<NI, H>(rows[tid], tid, l + 1);
        else rofs[(l + 2) & 1][tid] = row_off<NI, H>(rows[tid], tid, l + 2);
      }
      fence_proxy_async();
      if (warp == 0) issue_step<NI, H>(P, sm, rows, true, l + 1, false, 0, false, true, l + 2, zdir(g, l + 2), &mbar);
      pending = true;
    }
    // cross-block parts: x-faces jx = 2, 4, 6 of rows >= 1 (XB), y-faces of rows jy = 2, 4, .. (YB)
    if (lay && fin_l) {
      for (int t = tid; t < (OY * 3 + L6T::NYB * OX) * N2; t += NT) {
        const int f = t / N2, ent = t - f * N2;
        if (f < OY * 3) {
          const int oy = f / 3, jx = 2 * (f - oy * 3) + 2;
          AX[(oy * OX + jx - 1) * N2 + ent] += XB[t];
        } else {
          const int q = f - OY * 3, b = q / OX, jx = q - b * OX + 1, jy = 2 * b + 2;
          AY[((jy - 1) * OX + jx - 1) * N2 + ent] += YB[t - OY * 3 * N2];
        }
      }
    }
    __syncthreads();
    // ======== store the owned x- and y-faces of layer l, z-faces of plane l
    if (fin_l) {
      for (int rr = warp; rr < 3 * OY; rr += NT / 32) {
        const int kind = rr / OY, oy = rr - kind * OY;
        const int e0 = x0, er = y0 + oy;
        int cnt, z0 = 0, z1 = 0, za = 0;
        long long gb;
        if (kind == 0) {
          if (!lay || er >= ny) continue;
          cnt = min(OX, nx + 1 - e0);
          z0 = e0 == 0;
          z1 = e0 + cnt - 1 == nx;
          gb = g.off_f[0] + ((long long)e0 + (long long)(nx + 1) * (er + (long long)ny * l)) * N2;
        } else if (kind == 1) {
          if (!lay || er > ny) continue;
          cnt = min(OX, nx - e0);
          za = (er == 0 || er == ny);
          gb = g.off_f[1] + ((long long)e0 + (long long)nx * (er + (long long)(ny + 1) * l)) * N2;
        } else {   // (after the last layer, step l = nz: plane nz was completed by step nz - 1)
          if (!lay || er >= ny) continue;
          cnt = min(OX, nx - e0);
          za = zdir(g, l);
          gb = g.off_f[2] + ((long long)e0 + (long long)nx * (er + (long long)ny * l)) * N2;
        }
        if (cnt <= 0) continue;
        const double* src = (kind == 0 ? AX : (kind == 1 ? AY : AZ)) + oy * OX * N2;
        double* dst = P.y + gb;
        const int n = cnt * N2, lo = za ? n : (z0 ? N2 : 0), hi = z1 ? n - N2 : n;
        for (int t = lane; t < n; t += 32) dst[t] = (t >= lo && t < hi) ? src[t] : 0.0;
      }
    }
    __syncthreads();
  }
  if (DOT && P.dotp != nullptr) {
    double s = dot;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sred[warp] = s;
    __syncthreads();
    if (tid == 0) {
      double tsum = 0.0;
      for (int w = 0; w < NT / 32; ++w) tsum += sred[w];
      P.dotp[item] = tsum;
    }
  }
}

}  // namespace v5

bool v6_supported(int ni) { return ni >= 2 && ni <= 7; }

// tiles own 7 x 3 elements; the entity index ranges fx in [0, nx], fy in [0, ny] are covered
void v6_tiles(int nx, int ny, int h, int* ntx, int* nty) {
  *ntx = (nx + 1 + v5::OX - 1) / v5::OX;
  *nty = (ny + 1 + (h - 1) - 1) / (h - 1);
}

// z-segments: ntiles columns of nz layers on nsm SMs x 2 CTAs; a segment above the first recomputes
// the layer below its first plane, so more segments cost compute: pick the count that minimises
// (waves rounded up) x (layers + 1) per column
void v6_segments(int ntiles, int nz, int nslots, int* nseg, int* zseg) {
  double best = 1e300;
  int bs = 1;
  for (int s = 1; s <= nz && s <= 64; ++s) {
    const int zs = (nz + s - 1) / s;
    const int segs = (nz + zs - 1) / zs;
    const long long items = (long long)ntiles * segs;
    const long long waves = (items + nslots - 1) / nslots;
    const double cost = (double)waves * (zs + (segs > 1 ? 1 : 0));
    if (cost < best - 1e-9) { best = cost; bs = s; }
  }
  const int zs = (nz + bs - 1) / bs;
  *zseg = zs;
  *nseg = (nz + zs - 1) / zs;
}

void v6_make_coef(int ni, const double* d, const double* a0, const double* lam, double K00, double K0p, double w0,
                  std::vector<unsigned char>& out) {
  V5Coef c;
  memset(&c, 0, sizeof(c));
  const double w02 = w0 * w0, w03 = w02 * w0;
  for (int m = 0; m < ni; ++m) {
    for (int q = 0; q < 3; ++q) {
      c.c[q][m] = d[q + 1] * a0[m];
      c.ef2[q][m] = 2.0 * d[q + 1] * w0 * a0[m];
      c.ef1[q][m] = d[q + 1] * w0 * a0[m];
    }
    c.a0[m] = a0[m];
    c.sig[m] = (m & 1) ? -1.0 : 1.0;
    // z-edge self: 4 [d0 w0^2 + (d1 + d2) w0 K00 + d3 w0^2 Lam_k]
    c.czu[m] = 4.0 * (d[0] * w02 + (d[1] + d[2]) * w0 * K00 + d[3] * w02 * lam[m]);
    // x-edge self (per layer): 2 [d0 w0^2 + d1 w0^2 Lam_i + (d2 + d3) w0 K00]; y-edge likewise
    c.cxu[m] = 2.0 * (d[0] * w02 + d[1] * w02 * lam[m] + (d[2] + d[3]) * w0 * K00);
    c.cyu[m] = 2.0 * (d[0] * w02 + d[2] * w02 * lam[m] + (d[1] + d[3]) * w0 * K00);
  }
  for (int k = 0; k < ni; ++k)
    for (int j = 0; j < ni; ++j)
      for (int i = 0; i < ni; ++i) c.dinv[i + ni * (j + ni * k)] = 1.0 / (d[0] + d[1] * lam[i] + d[2] * lam[j] + d[3] * lam[k]);
  for (int b = 0; b < ni; ++b)
    for (int a = 0; a < ni; ++a) {
      c.fdx[a + ni * b] = 2.0 * (d[0] * w0 + d[1] * K00 + d[2] * w0 * lam[a] + d[3] * w0 * lam[b]);
      c.fdy[a + ni * b] = 2.0 * (d[0] * w0 + d[2] * K00 + d[1] * w0 * lam[a] + d[3] * w0 * lam[b]);
      c.fdz[a + ni * b] = d[0] * w0 + d[3] * K00 + d[1] * w0 * lam[a] + d[2] * w0 * lam[b];
    }
  for (int q = 0; q < 3; ++q) c.k0p[q] = d[q + 1] * K0p;
  // z-edge: 4 d3 w0^2 (vertex coupling), 2 d1 w0, 2 d2 w0 (line sums + K0p neighbours)
  c.sc[0] = 4.0 * d[3] * w02;
  c.sc[1] = 2.0 * d[1] * w0;
  c.sc[2] = 2.0 * d[2] * w0;
  // x-edge: 2 d1 w0^2, d2 w0, 2 d3 w0;  y-edge: 2 d2 w0^2, d1 w0, 2 d3 w0
  c.sc[3] = 2.0 * d[1] * w02; c.sc[4] = d[2] * w0; c.sc[5] = 2.0 * d[3] * w0;
  c.sc[6] = 2.0 * d[2] * w02; c.sc[7] = d[1] * w0; c.sc[8] = 2.0 * d[3] * w0;
  // vertex: 4 (d0 w0^3 + (d1 + d2 + d3) w0^2 K00), 2 d1 w0^2, 2 d2 w0^2, 4 d3 w0^2
  c.sc[9] = 4.0 * (d[0] * w03 + (d[1] + d[2] + d[3]) * w02 * K00);
  c.sc[10] = 2.0 * d[1] * w02; c.sc[11] = 2.0 * d[2] * w02; c.sc[12] = 4.0 * d[3] * w02;
  c.sc[15] = K0p;
  out.resize(sizeof(c));
  memcpy(out.data(), &c, sizeof(c));
}

template <int NI, bool DOT, int H>
static int launch_v6_t(const V5Params& P, cudaStream_t st, int* nl) {
  const size_t smem = sizeof(double) * v5::L6<NI, H>::TOTAL;
  static bool attr[kMaxDev];
  const int dv = dev_slot();
  if (!attr[dv]) {
    cudaFuncSetAttribute(v5::k_apply_v6<NI, DOT, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr[dv] = true;
  }
  v5::k_apply_v6<NI, DOT, H><<<P.nitems, 64 * H, smem, st>>>(P);
  (*nl)++;
  return cudaGetLastError();
}

int launch_apply_v6(const Geom& g, const double* x, double* y, const double* done, int ntx, int nty, int nseg,
                    int zseg, const void* coef, double* dotp, void* stream, int* nl, void* events, int h) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  V5Params P;
  P.g = g; P.x = x; P.y = y; P.done = done; P.dotp = dotp;
  P.ntx = ntx; P.nty = nty; P.nseg = nseg; P.zseg = zseg; P.nitems = ntx * nty * nseg;
  memcpy(&P.cf, coef, sizeof(V5Coef));
  if (ev) cudaEventRecord(ev[0], st);
  int e = 0;
  const bool dot = dotp != nullptr;
  switch (g.ni) {
#define SC_V5_CASE(N) \
    case N:                                                                                     \
      if (h == 8) e = dot ? launch_v6_t<N, true, 8>(P, st, nl) : launch_v6_t<N, false, 8>(P, st, nl); \
      else e = dot ? launch_v6_t<N, true, 4>(P, st, nl) : launch_v6_t<N, false, 4>(P, st, nl);           \
      break;
    SC_V5_CASE(2) SC_V5_CASE(3) SC_V5_CASE(4) SC_V5_CASE(5) SC_V5_CASE(6) SC_V5_CASE(7)
#undef SC_V5_CASE
    default: return (int)cudaErrorInvalidValue;
  }
  if (ev) cudaEventRecord(ev[1], st);
  return e;
}

}  // namespace sc
