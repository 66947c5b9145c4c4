// Condensed operator v7 for 2 <= n_I <= 7 (p = 3..8), uniform geometry, one rank: two passes,
// condensed part element by element, then assembly + primary part entity by entity
// (SURVEY §8(a) rows a3-a8).
//
// The tile-column kernels (v3, v6) move the algorithmic 16 N_c bytes but spend 1300-1600 warp
// instructions per element on assembling the shared entities on chip (look-back / halo
// recompute, barrier phases): they run at ~11 % of the HBM roofline.  v7 trades
// bytes for simplicity:
//  * pass A (k_v7_cond): the condensed part -H~_FI D^{-1} H~_IF of every element (Table 2, P:425-440,
//    faces-in / D^{-1} / faces-out, 7 FP64 operations per interior point in the even / odd form)
//    is written unassembled, side by side: for each face the part of the element on its high side
//    (the face is that element's w / s / b face) in U0, the part of the element on its low side in
//    U1.  U0 and U1 have the layout of the skeleton's face arrays, so a CTA's 16-element x-run
//    writes contiguous rows.  lane = (element, parity class) as in v6, pair exchanges by shuffles.
//  * pass B (k_v7_assemble): every skeleton entry (one thread each) = the primary part
//    (Eq. eq:east_east_primary_part_transformed generalised: diagonal face self terms,
//    opposite faces, rank-1 face <-> edge couplings, arrowhead rows of K~ for edges / vertices),
//    summed over all elements containing the entry, + U0 + U1 for faces.  Each entry is written
//    once, in a fixed order; the p . q partials of PCG are formed here (fused dot).
// On one rank every free entry's elements lie inside the domain, so the primary coefficients are the
// uniform-grid constants; Dirichlet entries are written as 0 and read as 0.  On z-slab ranks the
// operator returns local partial sums on the interface planes (the halo exchange adds the neighbour's):
// the condensed parts and edge line sums of pass A are local by construction (written by the local
// elements only; U0 / U1 entries no local element writes stay 0), pass B forms the local half of the
// interface entities' symmetric primary terms.  An interface edge's face-line sums are split between
// the ranks by element (each line belongs to one element), not halved: only the halo sum is the
// operator's value there.
#include <cuda_runtime.h>
#include <string.h>
#include <vector>
#include "sc_device.cuh"

namespace sc {

constexpr int V7_MAXNI = 23;   // v7 covers 2 <= n_I <= 23 (p = 3..24; n_I^3 uhat of an element in shared memory)

// pass B block size: 256 threads, or one face (n_I^2 entries, warp-rounded) when that is larger
template <int NI>
struct V7B {
  static constexpr int BT = NI * NI > 256 ? ((NI * NI + 31) / 32) * 32 : 256;
};

struct V7Coef {
  double c[3][24];        // d_{d+1} a0_m  (faces in / out, parity form)
  const double* dinv;     // device table D^{-1}(i,j,k), i fastest (n_I^3 doubles, owned by the context)
  double a0[24], ap[24], lam[24];
  double fd[3][529];      // face self: 2 (d0 w0 + d_n K00 + d_a w0 Lam_a + d_b w0 Lam_b), in-plane (a, b)
  double kf[3];           // d_n K0p (opposite faces)
  double ef[3][3];        // face <- edge: 2 d w0 (per direction d, for the face normal n)
  double eself[3][24];    // edge self: 4 d0 w0^2 + 4 d_e w0^2 Lam_m + 4 (d_o1 + d_o2) w0 K00
  double ev[3];           // edge <- vertex: 4 d_e w0^2
  double el[3][3];        // edge line sums: 2 d w0 for the transverse directions
  double vself;           // vertex: 8 d0 w0^3 + 8 (d1 + d2 + d3) w0^2 K00
  double vl[3];           // vertex line sums: 4 d w0^2
  double K0p;
};

struct V7Params {
  Geom g;
  const double* x;
  double* y;
  double* u0;             // face-part vectors (skeleton face layout), pass A -> pass B
  double* u1;
  const double* done;
  double* dotp;           // per-block partials of x . y (PCG p . q), or null
  int runx;               // pass A x-run length R: x-faces with fx % R == 0 carry a second part in U1
  int zseg;               // pass A z-segment length Z: z-faces with fz % Z == 0 carry a second part in U1
  V7Coef cf;
};

namespace v7 {


// smallest k stride >= pj * p1 with the 8 class bases si + pj sj + pk sk on distinct bank pairs
__host__ __device__ constexpr bool di_ok(int pj, int pk) {
  int o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int c = 0; c < 8; ++c) o[c] = ((c >> 2) + pj * ((c >> 1) & 1) + pk * (c & 1)) % 16;
  for (int a = 0; a < 8; ++a)
    for (int b = a + 1; b < 8; ++b)
      if (o[a] == o[b]) return false;
  return true;
}
__host__ __device__ constexpr int di_pk(int pj, int p1) {
  for (int pk = pj * p1; pk < pj * p1 + 16; ++pk)
    if (di_ok(pj, pk)) return pk;
  return pj * p1;
}

// ------------------------------------------------------------------------------------ pass A
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
      "W7: mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W7;\n}\n" ::"r"(smem_u32(m)),
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

// A work item is an x-run of R elements (ex0 .. ex0 + cnt - 1, ey, ez).  Its inputs are five
// contiguous skeleton ranges: the x-faces ex0 .. ex0 + cnt (one row), the y-faces of rows ey, ey + 1 and
// the z-faces of planes ez, ez + 1 (cnt faces each).  Each range is bulk-copied (cp.async.bulk, one
// mbarrier transaction per item) as its 16-byte aligned superset into a slot, so the range starts at
// slot + (start & 1).  Dirichlet rows are not copied: the lanes read a zero row instead (as they do for
// the Dirichlet x-faces fx = 0, nx).
struct __align__(16) Item {
  int ex0, cnt, ey, ez;
  int step, zc, col, pad;   // step in the column, column length, column
  int par, dirm;    // bit r: range r starts at an odd index / is a Dirichlet row
  long long s[5];   // range starts: x row, y rows ey / ey + 1, z planes ez / ez + 1
  bool dir[5];      // Dirichlet row (not copied)
};

// Column c = (rx, ey, zs) = rx + nruns (ey + ny zs), step s: the item (x-run rx, row ey, layer zs Z + s).
template <int NI, int R>
__device__ __forceinline__ Item decode(const Geom& g, int c, int step, int nruns, int Z) {
  constexpr int N2 = NI * NI;
  Item it;
  const int rx = c % nruns, rest = c / nruns;
  it.ey = rest % g.ny;
  it.ez = (rest / g.ny) * Z + step;
  it.step = step;
  it.col = c;
  it.ex0 = rx * R;
  it.cnt = min(R, g.nx - it.ex0);
  const long long nx = g.nx, ny = g.ny;
  it.s[0] = g.off_f[0] + (it.ex0 + (nx + 1) * (it.ey + ny * it.ez)) * N2;
  it.dir[0] = false;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int fy = it.ey + s, fz = it.ez + s;
    it.s[1 + s] = g.off_f[1] + (it.ex0 + nx * (fy + (ny + 1) * it.ez)) * N2;
    it.dir[1 + s] = !(fy > 0 && fy < g.ny);
    it.s[3 + s] = g.off_f[2] + (it.ex0 + nx * (it.ey + ny * fz)) * N2;
    it.dir[3 + s] = zdir(g, fz);
  }
  it.par = 0;
  it.dirm = 0;
  for (int r = 0; r < 5; ++r) {
    it.par |= (int)(it.s[r] & 1) << r;
    it.dirm |= (int)it.dir[r] << r;
  }
  return it;
}

template <int NI, int SX, int SR>
__device__ __forceinline__ void issue_item(const V7Params& P, const Item& it, double* stage, unsigned long long* mb) {
  constexpr int N2 = NI * NI;
  unsigned total = 0;
  long long a[5];
  unsigned by[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    const long long len = (long long)(r == 0 ? it.cnt + 1 : it.cnt) * N2;
    a[r] = it.s[r] & ~1LL;
    by[r] = it.dir[r] ? 0u : (unsigned)((((it.s[r] + len + 1) & ~1LL) - a[r]) * 8);
    total += by[r];
  }
  mbar_arrive_tx(mb, total);
#pragma unroll
  for (int r = 0; r < 5; ++r)
    if (by[r]) bulk_g2s(stage + (r == 0 ? 0 : SX + (r - 1) * SR), P.x + a[r], by[r], mb);
}

// ------------------------------------------------------------------------------------ pass A
// Pass A: lane = (element, x-line (j, k)), three phases per item (an x-run of R elements):
//  X: faces-in + D^{-1} along the lane's x-line (the y / z inputs of the line's points are the face
//     values (S +- N)(i, k), (B +- T)(i, j); the sign is the parity of the lane's j / k, P:302 sigma), the
//     x faces-out as the two parity sums Q_even / Q_odd of the line (W part -(Qe + Qo), E part -(Qe - Qo)),
//     uhat = D^{-1} (...) stored to shared memory;
//  Y: lane = (i, k): y faces-out = parity sums over j of c2_j uhat(i, j, k);
//  Z: lane = (i, j): z faces-out over k; then the edge line sums (U0 / U1 at the edges).
// Per-lane constants (D^{-1}(., j, k), the y / z coefficients and signs) stay in registers.
// Assembly on chip: the x-faces inside a run (E part of element e + W part of element e + 1, through
// shared memory) and the z-faces inside a column (a persistent CTA marches a column of Z items up z; the
// T part of layer ez stays in the lane's registers and is added to the B part of layer ez + 1).  Only the
// run-boundary x-faces (fx % R == 0) and segment-boundary z-faces (fz % Z == 0) keep a second part in
// U1; y-faces are written as U0 (S part) + U1 (N part).  Every output row is a contiguous range.
template <int NI, int STAGES>
struct V8A {
  static constexpr int N2 = NI * NI, N3 = N2 * NI;
  // elements per item (x-run) and per thread group; one stage: G N2 <= 256 threads and NG groups per
  // item; two stages (the next item's loads in flight while this one computes): one group per item
  // n_I >= 8: one group per item, the largest power of two G with G n_I^2 <= 256 (R must be a power of
  // two: pass B tests the run-boundary x-faces with fx & (R - 1))
  static constexpr int GB = N2 <= 64 ? 4 : (N2 <= 128 ? 2 : 1);   // n_I >= 16: one element, one lane per line
  static constexpr int R = NI >= 8 ? GB : (NI == 7 ? 10 : (NI >= 6 ? 8 : (NI >= 4 ? 16 : 32)));
  static constexpr int G = NI >= 8 ? GB : (STAGES == 2 ? R : (NI == 7 ? 5 : (NI >= 6 ? 4 : (NI == 5 ? 8 : (NI == 4 ? 16 : (NI == 3 ? 16 : 32))))));
  static constexpr int NG = R / G;
  static constexpr int NT = ((G * N2 + 31) / 32) * 32;       // threads per CTA
  static constexpr int EWF = ((R * 2 * NI + 31) / 32) * 32;  // edge-phase slots per family (warp-rounded)
  static constexpr int MINB = NI >= 16 ? 1 : NI >= 7 ? 3 : (STAGES == 2 ? (NT > 256 ? 2 : 4) : (NT <= 128 ? 8 : (NT <= 160 ? 6 : 4)));
  static constexpr int SX = ((R + 1) * N2 + 1 + 1) & ~1;     // slot >= len + 1 (the 8-byte phase), even
  static constexpr int SR = (R * N2 + 1 + 1) & ~1;
  static constexpr int STAGE = SX + 4 * SR;
  static constexpr int VS = N3 + (N3 % 2 == 0 ? 1 : 0);      // uhat per element (odd stride)
  static constexpr int SMEM = (STAGES * STAGE + R * VS + R * N2) * 8;   // inputs, uhat, E parts
};

// Edge line sums of one element family (see the header): F = 0 x-edges, 1 y-edges, 2 z-edges; hi = 0: the
// a0-weighted lines of the element's low faces (U0 at its low edge), hi = 1: the ap = sigma a0 weighted
// lines of its high faces (U1 at its high edge).  An interior edge's four face lines (the K~ rows of the
// primary part couple it to the face interiors along lines) belong to exactly these two elements.
template <int NI, int F>
__device__ __forceinline__ double edge_line(const V7Coef& cf, const double* zb, const double* zt, const double* ys,
                                            const double* yn, const double* w, const double* e, int hi, int m) {
  // F = 0: z-face (m, q) over j + y-face (m, q) over k; F = 1: z-face (q, m) over i + x-face (m, q) over k;
  // F = 2: y-face (q, m) over i + x-face (q, m) over j
  const double* p1 = F == 0 ? (hi ? zt : zb) + m : (F == 1 ? (hi ? zt : zb) + NI * m : (hi ? yn : ys) + NI * m);
  const double* p2 = F == 0 ? (hi ? yn : ys) + m : (F == 1 ? (hi ? e : w) + m : (hi ? e : w) + NI * m);
  constexpr int S1 = F == 0 ? NI : 1, S2 = F == 2 ? 1 : NI;
  const double e1 = F == 0 ? cf.el[0][1] : (F == 1 ? cf.el[1][0] : cf.el[2][0]);
  const double e2 = F == 0 ? cf.el[0][2] : (F == 1 ? cf.el[1][2] : cf.el[2][1]);
  double se = 0.0, so = 0.0;
#pragma unroll
  for (int q = 0; q < NI; ++q) {
    const double t = fma(e1, p1[S1 * q], e2 * p2[S2 * q]);
    if (q & 1) so = fma(cf.a0[q], t, so);
    else se = fma(cf.a0[q], t, se);
  }
  return hi ? se - so : se + so;
}

template <int NI, int STAGES>
__global__ void __launch_bounds__(V8A<NI, STAGES>::NT, V8A<NI, STAGES>::MINB) k_v7_lines(const __grid_constant__ V7Params P,
                                                                                       int ncols, int nruns) {
  if (P.done != nullptr && *P.done != 0.0) return;
  using A = V8A<NI, STAGES>;
  constexpr int N2 = NI * NI, G = A::G, R = A::R, NG = A::NG;
  constexpr int EWF = A::EWF;
  const Geom& g = P.g;
  const V7Coef& cf = P.cf;
  const int nx = g.nx, ny = g.ny, nz = g.nz, Z = P.zseg;
  const long long nx1 = nx + 1, ny1 = ny + 1;
  extern __shared__ __align__(16) double smem[];
  double* const sv = smem + STAGES * A::STAGE;
  double* const sE = sv + R * A::VS;   // E parts of phase X (x-faces assembled inside the run)
  __shared__ unsigned long long mbar[2];
  __shared__ Item sit[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // this CTA's columns: blockIdx.x, + gridDim.x, ...; column length zc = min(Z, nz - zs Z); thread 0
  // walks the items it issues (ic, is, izc) STAGES ahead of the computation
  auto col_len = [&](int c) { const int zs = (c / nruns) / ny; return min(Z, nz - zs * Z); };
  int ic = blockIdx.x, is = 0, izc = ic < ncols ? col_len(ic) : 0;
  if (tid == 0)
    for (int q = 0; q < STAGES && ic < ncols; ++q) {
      sit[q] = decode<NI, R>(g, ic, is, nruns, Z);
      sit[q].zc = izc;
      issue_item<NI, A::SX, A::SR>(P, sit[q], smem + q * A::STAGE, &mbar[q]);
      if (++is >= izc) {
        ic += gridDim.x;
        is = 0;
        izc = ic < ncols ? col_len(ic) : 0;
      }
    }
  // lane constants: line l = a + NI b of the element (phase X: (j, k) = (a, b); Y: (i, k); Z: (i, j))
  const bool lane_on = tid < G * N2;
  const int eg = tid / N2, l = tid - eg * N2, la = l % NI, lb = l / NI;
  double Dl[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) Dl[i] = lane_on ? cf.dinv[i + NI * l] : 0.0;
  const double c2j = cf.c[1][la], c3k = cf.c[2][lb];
  const double gj = (la & 1) ? -1.0 : 1.0, gk = (lb & 1) ? -1.0 : 1.0;
  const double kf0 = cf.kf[0], kf1 = cf.kf[1], kf2 = cf.kf[2];
  double wpart[NG], tcarry[NG];
#pragma unroll
  for (int r = 0; r < NG; ++r) tcarry[r] = 0.0;
  const long long d01 = P.u1 - P.u0;
  for (int n = 0;; ++n) {
    if ((int)blockIdx.x >= ncols) break;
    const int b = STAGES == 2 ? (n & 1) : 0;
    double* const stage = smem + b * A::STAGE;
    mbar_wait(&mbar[b], (unsigned)((STAGES == 2 ? (n >> 1) : n) & 1));
    const int4 ih = *reinterpret_cast<const int4*>(&sit[b]);          // ex0, cnt, ey, ez
    const int4 icq = *reinterpret_cast<const int4*>(&sit[b].step);    // step, zc, column
    const int par = sit[b].par, dirm = sit[b].dirm;
    const int ex0 = ih.x, cnt = ih.y, ey = ih.z, ez = ih.w;
    const int s = icq.x, zc = icq.y;
    double* const X = stage + (par & 1);
    // the Dirichlet x-faces fx = 0, nx of a boundary run and the Dirichlet y / z rows (not copied) read as
    // zero (block-uniform branch)
    if (ex0 == 0 || ex0 + cnt == nx || (dirm & 0x1e)) {
      if (tid < N2) {
        if (ex0 == 0) X[tid] = 0.0;
        if (ex0 + cnt == nx) X[cnt * N2 + tid] = 0.0;
      }
      for (int q = 1; q < 5; ++q)
        if ((dirm >> q) & 1)
          for (int t = tid; t < A::SR; t += A::NT) stage[A::SX + (q - 1) * A::SR + t] = 0.0;
      __syncthreads();
    }
    const double* Yr[2];
    const double* Zr[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      Yr[q] = stage + A::SX + q * A::SR + ((par >> (1 + q)) & 1);
      Zr[q] = stage + A::SX + (2 + q) * A::SR + ((par >> (3 + q)) & 1);
    }
    // output bases of the item's first element (face rows are contiguous along x)
    double* const ux = P.u0 + g.off_f[0] + (ex0 + nx1 * (ey + (long long)ny * ez)) * N2 + l;
    double* const uy = P.u0 + g.off_f[1] + (ex0 + (long long)nx * (ey + ny1 * ez)) * N2 + l;
    double* const uz = P.u0 + g.off_f[2] + (ex0 + (long long)nx * (ey + (long long)ny * ez)) * N2 + l;
    // ---- phase X (+ the face values the lane's Y / Z outputs couple to, kept in registers)
    double kfy[NG][2], kfz[NG][2];
    if (lane_on) {
#pragma unroll
      for (int gr = 0; gr < NG; ++gr) {
        const int el = gr * G + eg;
        const double w = X[el * N2 + l], e = X[(el + 1) * N2 + l];
        const double xs = w + e, xd = w - e;
        const double* S = Yr[0] + el * N2 + NI * lb;   // S(i, k), i = 0..NI-1
        const double* Nn = Yr[1] + el * N2 + NI * lb;
        const double* B = Zr[0] + el * N2 + NI * la;   // B(i, j)
        const double* T = Zr[1] + el * N2 + NI * la;
        double qe = 0.0, qo = 0.0;
        double* const v = sv + el * A::VS + NI * l;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const double yin = fma(gj, Nn[i], S[i]);
          const double zin = fma(gk, T[i], B[i]);
          const double c1 = cf.c[0][i];
          const double u = fma(c1, (i & 1) ? xd : xs, fma(c2j, yin, c3k * zin));
          const double vv = u * Dl[i];
          if (i & 1) qo = fma(c1, vv, qo);
          else qe = fma(c1, vv, qe);
          v[i] = vv;
        }
        // the element's W / E face parts: condensed part + the element's opposite-face coupling of the
        // primary part (d1 K0p times the element's other x-face; the two elements of a face
        // give d1 K0p (u_{fx-1} + u_{fx+1}))
        wpart[gr] = fma(kf0, e, -(qe + qo));            // the element's W face
        sE[el * N2 + l] = fma(kf0, w, qo - qe);         // its E face (added to the W part of element el + 1)
        // the same coupling for the y / z faces (entry l = (i, k) / (i, j) of the Y / Z phases)
        kfy[gr][0] = kf1 * Yr[1][el * N2 + l];   // into S: the element's N face
        kfy[gr][1] = kf1 * Yr[0][el * N2 + l];   // into N: its S face
        kfz[gr][0] = kf2 * Zr[1][el * N2 + l];   // into B: its T face
        kfz[gr][1] = kf2 * Zr[0][el * N2 + l];   // into T: its B face
      }
    }
    // ---- edge line sums: slot -> (family, element, high side, entry); a warp's slots share the family
#pragma unroll 1
    for (int sl = tid; sl < 3 * EWF; sl += A::NT) {
      const int ef = sl / EWF, er = sl - ef * EWF;
      const int el = er / (2 * NI), eo = er - el * (2 * NI), ehi = eo / NI, em = eo - ehi * NI;
      if (el < cnt) {
        const int ex = ex0 + el;
        const double* zb = Zr[0] + el * N2;
        const double* zt = Zr[1] + el * N2;
        const double* ys = Yr[0] + el * N2;
        const double* yn = Yr[1] + el * N2;
        const double* w = X + el * N2;
        const double* e = X + (el + 1) * N2;
        double sum;
        long long dst;
        if (ef == 0) {
          sum = edge_line<NI, 0>(cf, zb, zt, ys, yn, w, e, ehi, em);
          dst = g.off_e[0] + (ex + (long long)nx * (ey + ehi + ny1 * (ez + ehi))) * NI + em;
        } else if (ef == 1) {
          sum = edge_line<NI, 1>(cf, zb, zt, ys, yn, w, e, ehi, em);
          dst = g.off_e[1] + (ex + ehi + nx1 * (ey + (long long)ny * (ez + ehi))) * NI + em;
        } else {
          sum = edge_line<NI, 2>(cf, zb, zt, ys, yn, w, e, ehi, em);
          dst = g.off_e[2] + (ex + ehi + nx1 * (ey + ehi + ny1 * ez)) * NI + em;
        }
        __stcs((ehi ? P.u1 : P.u0) + dst, sum);
      }
    }
    // the stage is no longer read (the Y / Z phases use uhat, the E parts and registers): release it and
    // issue the item STAGES ahead into it, so its loads overlap the Y / Z phases
    fence_proxy_async();
    __syncthreads();
    const bool more = (s + 1 < zc || (int)(icq.z + gridDim.x) < ncols);
    if (tid == 0 && ic < ncols) {
      sit[b] = decode<NI, R>(g, ic, is, nruns, Z);
      sit[b].zc = izc;
      issue_item<NI, A::SX, A::SR>(P, sit[b], stage, &mbar[b]);
      if (++is >= izc) {
        ic += gridDim.x;
        is = 0;
        izc = ic < ncols ? col_len(ic) : 0;
      }
    }
    // ---- x-faces, phases Y, Z
    if (lane_on) {
#pragma unroll
      for (int gr = 0; gr < NG; ++gr) {
        const int el = gr * G + eg;
        if (el < cnt) {
          // x-face ex0 + el: W part + the E part of element el - 1 (inside the run); the run's first
          // face keeps the previous run's E part in U1, the run's last E part goes to U1
          __stcs(ux + el * N2, el > 0 ? wpart[gr] + sE[(el - 1) * N2 + l] : wpart[gr]);
          if (el == cnt - 1) __stcs(ux + d01 + (el + 1) * N2, sE[el * N2 + l]);
          const double* const v = sv + el * A::VS;
          double qe = 0.0, qo = 0.0;
#pragma unroll
          for (int j = 0; j < NI; ++j) {   // lane (i, k) = (la, lb)
            const double t = cf.c[1][j] * v[la + NI * (j + NI * lb)];
            if (j & 1) qo += t;
            else qe += t;
          }
          __stcs(uy + el * N2, kfy[gr][0] - (qe + qo));                                // S face (ey) in U0
          __stcs(uy + d01 + (long long)nx * N2 + el * N2, kfy[gr][1] + (qo - qe));     // N face (ey + 1) in U1
          qe = 0.0; qo = 0.0;
#pragma unroll
          for (int k = 0; k < NI; ++k) {   // lane (i, j) = (la, lb)
            const double t = cf.c[2][k] * v[l + N2 * k];
            if (k & 1) qo += t;
            else qe += t;
          }
          // z-face ez: B part + the T part of layer ez - 1 of this column (the column's first face keeps
          // the previous segment's T part in U1); the column's last T part goes to U1 at ez + 1
          const double bp = kfz[gr][0] - (qe + qo), tp = kfz[gr][1] + (qo - qe);
          __stcs(uz + el * N2, s > 0 ? bp + tcarry[gr] : bp);
          if (s == zc - 1) __stcs(uz + d01 + (long long)nx * ny * N2 + el * N2, tp);
          tcarry[gr] = tp;
        }
      }
    }
    // uhat and the E parts are rewritten by the next item's phase X
    __syncthreads();
    if (!more) break;
  }
}

// ------------------------------------------------------------------------------------ pass B
// One CTA per cell row (cy, cz) of the vertex lattice, 0 <= cy <= ny, 0 <= cz <= nz.  The cell
// (c_x, cy, cz) owns the x-face (c_x, cy, cz), y-face (c_x, cy, cz), z-face (c_x, cy, cz), x-edge,
// y-edge, z-edge and vertex with the same indices (those that exist), so the cell rows partition the
// skeleton and each CTA writes seven contiguous skeleton ranges (one per entity kind), one thread per
// entry, consecutive threads on consecutive entries (coalesced loads of x / U0 / U1, coalesced
// stores of y).  The values of the neighbouring rows (opposite faces, edge line sums over faces of
// the rows (cy - 1, cz), (cy, cz - 1)) are read through L2 while they are still resident: rows run
// in cy-fastest order, so the reuse distance is one row (cy) or one plane of rows (cz).  U0 / U1 are
// read once (evict-first), y is written once (streaming stores): the resident set stays x.
// Every entry is a sum in a fixed order; the p . q partial of the CTA is formed in a fixed order.
__device__ __forceinline__ bool in_f(int v, int n) { return v > 0 && v < n; }

__device__ __forceinline__ double ldv(const double* __restrict__ x, long long i, bool ok) {
  const double v = __ldg(x + (ok ? i : 0));   // always a valid address: the load is not predicated
  return ok ? v : 0.0;
}

// Face rows.  Thread t < FPI N2 keeps one in-face entry e = (ea, eb) = t % N2 (its coefficients in
// registers) and walks the row's faces f = t / N2 + FPI it, so a warp's accesses are contiguous.  One face
// entry: y = fd u + wA (a0_ea A0[eb] + ap_ea A1[eb]) + wB (a0_eb B0[ea] + ap_eb B1[ea]) + U0 (+ U1)
// (the primary part of Eq. eq:east_east_primary_part_transformed summed over the face's two elements,
// P:415-424; its opposite-face term kf (u_lo + u_hi) is added per element in pass A, which has both
// parallel faces of the element on chip, together with the condensed parts).  CLS 0 / 1 / 2: x- / y- /
// z-face row of the cell row.
template <int NI, bool DOT, int CLS>
__device__ __forceinline__ void face_row(const V7Params& P, int cy, int cz, double& dot) {
  constexpr int N2 = NI * NI, FPI = V7B<NI>::BT / N2;
  const int t = threadIdx.x;
  if (t >= FPI * N2) return;
  const Geom& g = P.g;
  const V7Coef& cf = P.cf;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long nx1 = nx + 1, ny1 = ny + 1;
  const int f0 = t / N2, e = t - f0 * N2, eb = e / NI, ea = e - eb * NI;
  // a z-slab interface plane (cz = 0 / nz not Dirichlet): this rank holds one of the plane's two element
  // layers, so it forms the local half of the symmetric primary-part terms; the halo exchange adds the
  // neighbour's half (the condensed parts in U0 / U1 are local by construction)
  const bool ifc = (cz == 0 && !g.dir_bot) || (cz == g.nz && !g.dir_top);
  const double hf = (CLS == 2 && ifc) ? 0.5 : 1.0;
  const double fd = hf * cf.fd[CLS][e];
  const double a0a = cf.a0[ea], apa = cf.ap[ea], a0b = cf.a0[eb], apb = cf.ap[eb];
  const bool zb0 = !zdir(g, cz), zb1 = !zdir(g, cz + 1);
  int nf;
  long long base, so, A0, A1, B0, B1, astep, bstep;
  bool rowfree, olo_r = true, ohi_r = true, oka0 = true, oka1 = true, okb0, okb1, u1r = true;
  double wA, wB, kf;
  if (CLS == 0) {          // x-faces (fx, cy, cz): A = z-edges (fx, cy / cy + 1, cz), B = y-edges (fx, cy, cz / cz + 1)
    nf = nx + 1;
    base = g.off_f[0] + nx1 * (cy + (long long)ny * cz) * N2;
    so = N2;
    rowfree = true;
    A0 = g.off_e[2] + nx1 * (cy + ny1 * cz) * NI; A1 = A0 + nx1 * NI; astep = NI;
    oka0 = in_f(cy, ny); oka1 = in_f(cy + 1, ny);
    B0 = g.off_e[1] + nx1 * (cy + (long long)ny * cz) * NI; B1 = B0 + nx1 * ny * NI; bstep = NI;
    okb0 = zb0; okb1 = zb1;
    wA = cf.ef[0][1]; wB = cf.ef[0][2]; kf = cf.kf[0];
  } else if (CLS == 1) {   // y-faces (ex, cy, cz): A = z-edges (ex / ex + 1, cy, cz), B = x-edges (ex, cy, cz / cz + 1)
    nf = nx;
    base = g.off_f[1] + (long long)nx * (cy + ny1 * cz) * N2;
    so = (long long)nx * N2;
    rowfree = in_f(cy, ny);
    olo_r = cy - 1 > 0; ohi_r = cy + 1 < ny;
    A0 = g.off_e[2] + nx1 * (cy + ny1 * cz) * NI; A1 = A0 + NI; astep = NI;
    B0 = g.off_e[0] + (long long)nx * (cy + ny1 * cz) * NI; B1 = B0 + (long long)nx * ny1 * NI; bstep = NI;
    okb0 = zb0; okb1 = zb1;
    wA = cf.ef[1][0]; wB = cf.ef[1][2]; kf = cf.kf[1];
  } else {                 // z-faces (ex, cy, cz): A = y-edges (ex / ex + 1, cy, cz), B = x-edges (ex, cy / cy + 1, cz)
    nf = nx;
    base = g.off_f[2] + (long long)nx * (cy + (long long)ny * cz) * N2;
    so = (long long)nx * ny * N2;
    rowfree = zb0;
    olo_r = cz - 1 >= 0 && !zdir(g, cz - 1); ohi_r = cz + 1 <= nz && !zdir(g, cz + 1);
    A0 = g.off_e[1] + nx1 * (cy + (long long)ny * cz) * NI; A1 = A0 + NI; astep = NI;
    B0 = g.off_e[0] + (long long)nx * (cy + ny1 * cz) * NI; B1 = B0 + (long long)nx * NI; bstep = NI;
    okb0 = in_f(cy, ny); okb1 = in_f(cy + 1, ny);
    u1r = cz % P.zseg == 0 || cz == g.nz;
    wA = hf * cf.ef[2][0]; wB = hf * cf.ef[2][1]; kf = cf.kf[2];
  }
  const double* __restrict__ x = P.x;
  const double* xp = x + base + e;
  const double* u0p = P.u0 + base + e;
  const double* u1p = P.u1 + base + e;
  double* yp = P.y + base + e;
  const double* pa0 = x + A0 + eb;
  const double* pa1 = x + A1 + eb;
  const double* pb0 = x + B0 + ea;
  const double* pb1 = x + B1 + ea;
#pragma unroll 2
  for (int f = f0; f < nf; f += FPI) {
    const long long o = (long long)f * N2;
    bool fr = rowfree, olo = olo_r, ohi = ohi_r, ka0 = oka0, ka1 = oka1, u1 = u1r;
    if (CLS == 0) {
      fr = in_f(f, nx);
      olo = f - 1 > 0;
      ohi = f + 1 < nx;
      u1 = f % P.runx == 0;
    } else {
      ka0 = in_f(f, nx);
      ka1 = in_f(f + 1, nx);
    }
    double yv = 0.0;
    if (fr) {
      const double u = __ldg(xp + o);
      const long long oa = (long long)f * astep, ob = (long long)f * bstep;
      const double va0 = __ldg(pa0 + (ka0 ? oa : 0)), va1 = __ldg(pa1 + (ka1 ? oa : 0));
      const double vb0 = __ldg(pb0 + (okb0 ? ob : 0)), vb1 = __ldg(pb1 + (okb1 ? ob : 0));
      const double c0 = __ldcs(u0p + o);
      const double c1 = u1 ? __ldcs(u1p + o) : 0.0;
      const double ea_ = a0a * (ka0 ? va0 : 0.0) + apa * (ka1 ? va1 : 0.0);
      const double eb_ = a0b * (okb0 ? vb0 : 0.0) + apb * (okb1 ? vb1 : 0.0);
      yv = fd * u + wA * ea_ + wB * eb_ + c0 + c1;
      if (DOT) dot = fma(u, yv, dot);
    }
    __stcs(yp + o, yv);
  }
}

// Edge rows (entry m = t % NI fixed per thread, edges t / NI + EPI it).  The face-line sums come from
// pass A in U0 + U1 at the edge's entries; the rest is the K~ arrowhead: self, the two vertices, the
// K0p couplings to the neighbouring edges along the two transverse directions.
template <int NI, bool DOT, int DIR>
__device__ __forceinline__ void edge_row(const V7Params& P, int cy, int cz, double& dot) {
  constexpr int EPI = V7B<NI>::BT / NI;
  const int t = threadIdx.x;
  if (t >= EPI * NI) return;
  const Geom& g = P.g;
  const V7Coef& cf = P.cf;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long nx1 = nx + 1, ny1 = ny + 1;
  const int a0i = t / NI, m = t - a0i * NI;
  const bool ifc = DIR < 2 && ((cz == 0 && !g.dir_bot) || (cz == g.nz && !g.dir_top));
  const double hf = ifc ? 0.5 : 1.0;   // interface plane: the local half (see face_row)
  const double self = hf * cf.eself[DIR][m], va = cf.a0[m], vp = cf.ap[m];
  const bool zb0 = !zdir(g, cz), zb1 = !zdir(g, cz + 1);
  const bool zlo = cz - 1 >= 0 && !zdir(g, cz - 1), zhi = cz + 1 <= nz && !zdir(g, cz + 1);
  const double* __restrict__ x = P.x;
  int ne;
  long long base, vbase, vstep2, s1, s2;
  bool rowfree, lo1 = true, hi1 = true, lo2, hi2, vok1_r = true, vok2_r = true;
  double ev, c1, c2;
  if (DIR == 0) {          // x-edges (ex, cy, cz): vertices (ex / ex + 1, cy, cz); neighbours y (+- nx NI), z (+- nx ny1 NI)
    ne = nx;
    base = g.off_e[0] + (long long)nx * (cy + ny1 * cz) * NI;
    rowfree = in_f(cy, ny) && zb0;
    vbase = g.off_v + nx1 * (cy + ny1 * cz); vstep2 = 1;
    s1 = (long long)nx * NI; lo1 = cy - 1 > 0; hi1 = cy + 1 < ny;
    s2 = (long long)nx * ny1 * NI; lo2 = zlo; hi2 = zhi;
    ev = hf * cf.ev[0]; c1 = hf * cf.el[0][1] * cf.K0p; c2 = cf.el[0][2] * cf.K0p;
  } else if (DIR == 1) {   // y-edges (fx, cy, cz): vertices (fx, cy / cy + 1, cz); neighbours x (+- NI), z (+- nx1 ny NI)
    ne = nx + 1;
    base = g.off_e[1] + nx1 * (cy + (long long)ny * cz) * NI;
    rowfree = cy < ny && zb0;
    vbase = g.off_v + nx1 * (cy + ny1 * cz); vstep2 = nx1;
    vok1_r = in_f(cy, ny); vok2_r = in_f(cy + 1, ny);
    s1 = NI;
    s2 = nx1 * ny * NI; lo2 = zlo; hi2 = zhi;
    ev = hf * cf.ev[1]; c1 = hf * cf.el[1][0] * cf.K0p; c2 = cf.el[1][2] * cf.K0p;
  } else {                 // z-edges (fx, cy, cz): vertices (fx, cy, cz / cz + 1); neighbours x (+- NI), y (+- nx1 NI)
    ne = nx + 1;
    base = g.off_e[2] + nx1 * (cy + ny1 * cz) * NI;
    rowfree = in_f(cy, ny) && cz < nz;
    vbase = g.off_v + nx1 * (cy + ny1 * cz); vstep2 = nx1 * ny1;
    vok1_r = zb0; vok2_r = zb1;
    s1 = NI;
    s2 = nx1 * NI; lo2 = cy - 1 > 0; hi2 = cy + 1 < ny;
    ev = cf.ev[2]; c1 = cf.el[2][0] * cf.K0p; c2 = cf.el[2][1] * cf.K0p;
  }
  const double* xp = x + base + m;
  double* yp = P.y + base + m;
  const double* u0p = P.u0 + base + m;
  const double* u1p = P.u1 + base + m;
#pragma unroll 2
  for (int a = a0i; a < ne; a += EPI) {
    const long long o = (long long)a * NI;
    bool fr = rowfree, l1 = lo1, h1 = hi1, k1 = vok1_r, k2 = vok2_r;
    long long v1, v2;
    if (DIR == 0) {
      k1 = in_f(a, nx); k2 = in_f(a + 1, nx);
      v1 = vbase + a; v2 = v1 + 1;
    } else {
      fr = fr && in_f(a, nx);
      l1 = a - 1 > 0; h1 = a + 1 < nx;
      v1 = vbase + a; v2 = v1 + vstep2;
    }
    double yv = 0.0;
    if (fr) {
      const double u = __ldg(xp + o);
      const double w1 = ldv(x, v1, k1), w2 = ldv(x, v2, k2);
      const double n1 = ldv(xp, o - s1, l1) + ldv(xp, o + s1, h1);
      const double n2 = ldv(xp, o - s2, lo2) + ldv(xp, o + s2, hi2);
      yv = self * u + ev * (va * w1 + vp * w2) + c1 * n1 + c2 * n2 + __ldcs(u0p + o) + __ldcs(u1p + o);
      if (DOT) dot = fma(u, yv, dot);
    }
    __stcs(yp + o, yv);
  }
}

template <int NI, bool DOT>
__global__ void __launch_bounds__(V7B<NI>::BT, V7B<NI>::BT > 256 ? 2 : 4) k_v7_assemble(const __grid_constant__ V7Params P) {
  if (P.done != nullptr && *P.done != 0.0) return;
  const Geom& g = P.g;
  const V7Coef& cf = P.cf;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long nx1 = nx + 1, ny1 = ny + 1;
  const double* __restrict__ x = P.x;
  double* __restrict__ y = P.y;
  const int cy = blockIdx.x % (ny + 1), cz = blockIdx.x / (ny + 1);
  double dot = 0.0;
  if (cy < ny && cz < nz) face_row<NI, DOT, 0>(P, cy, cz, dot);
  if (cz < nz) face_row<NI, DOT, 1>(P, cy, cz, dot);
  if (cy < ny) face_row<NI, DOT, 2>(P, cy, cz, dot);
  edge_row<NI, DOT, 0>(P, cy, cz, dot);
  if (cy < ny) edge_row<NI, DOT, 1>(P, cy, cz, dot);
  if (cz < nz) edge_row<NI, DOT, 2>(P, cy, cz, dot);
  // ---------------- vertices (fx, cy, cz): lines along the 6 incident edges
  {
    const bool fr = in_f(cy, ny) && !zdir(g, cz);
    const bool zlo_ok = cz - 1 >= 0 && !zdir(g, cz - 1), zhi_ok = cz + 1 <= nz && !zdir(g, cz + 1);
    // interface plane: the in-plane terms are halved (two of the vertex's four element layers' worth
    // are local), the z-edge on the other rank's side is not local (see face_row)
    const bool ifc = (cz == 0 && !g.dir_bot) || (cz == nz && !g.dir_top);
    const double hf = ifc ? 0.5 : 1.0;
    const bool zbm = cz > 0, ztm = cz < nz;
    for (int fx = threadIdx.x; fx <= nx; fx += blockDim.x) {
      const long long i0 = g.off_v + fx + nx1 * (cy + ny1 * cz);
      double yv = 0.0;
      if (fr && in_f(fx, nx)) {
        constexpr int NI_ = NI;
        const double u = __ldg(x + i0);
        const long long xw = g.off_e[0] + (fx - 1 + (long long)nx * (cy + ny1 * cz)) * NI_, xe = xw + NI_;
        const long long ys = g.off_e[1] + (fx + nx1 * (cy - 1 + (long long)ny * cz)) * NI_, yn = ys + nx1 * NI_;
        const long long zb = g.off_e[2] + (fx + nx1 * (cy + ny1 * (cz - 1))) * NI_, zt = zb + nx1 * ny1 * NI_;
        double lx = 0.0, ly = 0.0, lz = 0.0;
#pragma unroll
        for (int q = 0; q < NI_; ++q) {
          lx = fma(cf.ap[q], __ldg(x + xw + q), fma(cf.a0[q], __ldg(x + xe + q), lx));
          ly = fma(cf.ap[q], __ldg(x + ys + q), fma(cf.a0[q], __ldg(x + yn + q), ly));
          lz = fma(cf.ap[q], ldv(x, zb + q, zbm), fma(cf.a0[q], ldv(x, zt + q, ztm), lz));
        }
        const double nbx = ldv(x, i0 - 1, fx - 1 > 0) + ldv(x, i0 + 1, fx + 1 < nx);
        const double nby = ldv(x, i0 - nx1, cy - 1 > 0) + ldv(x, i0 + nx1, cy + 1 < ny);
        const long long pl = nx1 * ny1;
        const double nbz = ldv(x, i0 - pl, zlo_ok) + ldv(x, i0 + pl, zhi_ok);
        yv = hf * (cf.vself * u + cf.vl[0] * fma(cf.K0p, nbx, lx) + cf.vl[1] * fma(cf.K0p, nby, ly)) +
             cf.vl[2] * fma(cf.K0p, nbz, lz);
        if (DOT) dot = fma(u, yv, dot);
      }
      __stcs(y + i0, yv);
    }
  }
  if (DOT) {
    // block partial of x . y in a fixed order (warp shuffles, then warps in order)
    __shared__ double red[V7B<NI>::BT / 32];
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < V7B<NI>::BT / 32; ++w) s += red[w];
      P.dotp[blockIdx.x] = s;
    }
  }
}

// padding entries of y between / after the entity arrays
__global__ void k_v7_padding(Geom g, double* __restrict__ y) {
  const long long N2 = (long long)g.ni * g.ni, NI = g.ni;
  const long long ends[7] = {g.off_f[0] + g.n_f[0] * N2, g.off_f[1] + g.n_f[1] * N2, g.off_f[2] + g.n_f[2] * N2,
                             g.off_e[0] + g.n_e[0] * NI, g.off_e[1] + g.n_e[1] * NI, g.off_e[2] + g.n_e[2] * NI,
                             g.off_v + g.n_v};
  const long long nexts[7] = {g.off_f[1], g.off_f[2], g.off_e[0], g.off_e[1], g.off_e[2], g.off_v, g.n_total};
  for (int q = 0; q < 7; ++q)
    for (long long i = ends[q] + threadIdx.x; i < nexts[q]; i += blockDim.x) y[i] = 0.0;
}

}  // namespace v7

bool v7_supported(int ni) { return ni >= 2 && ni <= V7_MAXNI; }

void v7_make_coef(int ni, const double* d, const double* a0, const double* ap, const double* lam, double K00,
                  double K0p, double w0, std::vector<unsigned char>& out, std::vector<double>& dinv) {
  V7Coef c;
  memset(&c, 0, sizeof(c));
  const double w02 = w0 * w0, w03 = w02 * w0;
  for (int m = 0; m < ni; ++m) {
    for (int q = 0; q < 3; ++q) c.c[q][m] = d[q + 1] * a0[m];
    c.a0[m] = a0[m];
    c.ap[m] = ap[m];
    c.lam[m] = lam[m];
    // edge along direction e, transverse o1, o2 (4 elements): 4 d0 w0^2 + 4 d_e w0^2 Lam_m + 4 (d_o1 + d_o2) w0 K00
    for (int e = 0; e < 3; ++e) {
      const int o1 = (e + 1) % 3, o2 = (e + 2) % 3;
      c.eself[e][m] = 4.0 * (d[0] * w02 + d[1 + e] * w02 * lam[m] + (d[1 + o1] + d[1 + o2]) * w0 * K00);
    }
  }
  dinv.assign((size_t)ni * ni * ni, 0.0);
  for (int k = 0; k < ni; ++k)
    for (int j = 0; j < ni; ++j)
      for (int i = 0; i < ni; ++i) dinv[i + ni * (j + ni * k)] = 1.0 / (d[0] + d[1] * lam[i] + d[2] * lam[j] + d[3] * lam[k]);
  c.dinv = nullptr;
  // face with normal n, in-plane directions (a, b) in increasing order: 2 (d0 w0 + d_n K00 + d_a w0 Lam_a + d_b w0 Lam_b)
  for (int n = 0; n < 3; ++n) {
    const int a = n == 0 ? 1 : 0, b = n == 2 ? 1 : 2;
    for (int eb = 0; eb < ni; ++eb)
      for (int ea = 0; ea < ni; ++ea)
        c.fd[n][ea + ni * eb] = 2.0 * (d[0] * w0 + d[1 + n] * K00 + d[1 + a] * w0 * lam[ea] + d[1 + b] * w0 * lam[eb]);
    c.kf[n] = d[1 + n] * K0p;
    for (int q = 0; q < 3; ++q) c.ef[n][q] = 2.0 * d[1 + q] * w0;
  }
  for (int e = 0; e < 3; ++e) {
    c.ev[e] = 4.0 * d[1 + e] * w02;
    for (int q = 0; q < 3; ++q) c.el[e][q] = 2.0 * d[1 + q] * w0;
    c.vl[e] = 4.0 * d[1 + e] * w02;
  }
  c.vself = 8.0 * d[0] * w03 + 8.0 * (d[1] + d[2] + d[3]) * w02 * K00;
  c.K0p = K0p;
  out.resize(sizeof(c));
  memcpy(out.data(), &c, sizeof(c));
}

void v7_set_dinv(std::vector<unsigned char>& coef, const double* d_dinv) {
  V7Coef c;
  memcpy(&c, coef.data(), sizeof(c));
  c.dinv = d_dinv;
  memcpy(coef.data(), &c, sizeof(c));
}

// Number of pass-B blocks (the p . q partials the PCG sums): one per cell row.
long long v7_dot_parts(const Geom& g) { return (long long)(g.ny + 1) * (g.nz + 1); }

template <int NI>
static int launch_v7_t(V7Params& P, cudaStream_t st, int* nl) {
  const Geom& g = P.g;
  static const char* sg = getenv("SC_V7_STAGES");
  const int two = sg && sg[0] == '2';
  int dev = 0;
  cudaGetDevice(&dev);
  // per device: dynamic shared memory opt-in and resident CTAs per SM of pass A
  static int attr_done[64][2] = {{0}}, per_sm[64][2] = {{0}}, nsm_c[64] = {0};
  const void* fn = two ? (const void*)v7::k_v7_lines<NI, 2> : (const void*)v7::k_v7_lines<NI, 1>;
  const int smem = two ? v7::V8A<NI, 2>::SMEM : v7::V8A<NI, 1>::SMEM;
  const int nthr = two ? v7::V8A<NI, 2>::NT : v7::V8A<NI, 1>::NT;
  const int R = v7::V8A<NI, 1>::R;
  if (dev < 64 && !attr_done[dev][two]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev][two], fn, nthr, smem);
    cudaDeviceGetAttribute(&nsm_c[dev], cudaDevAttrMultiProcessorCount, dev);
    attr_done[dev][two] = 1;
  }
  const int slots = (dev < 64 ? max(per_sm[dev][two], 1) * nsm_c[dev] : 148);
  const int nruns = (g.nx + R - 1) / R;
  // z-segment length Z: longer columns assemble more z-faces on chip (1 / Z of them keep a U1 part),
  // but the columns must still balance over the resident CTAs: minimise (waves) x (Z + 1)
  int Z = 1;
  long long best = -1;
  const int cand[6] = {32, 24, 16, 12, 8, 4};
  for (int q = 0; q < 6; ++q) {
    const int z = cand[q] < g.nz ? cand[q] : g.nz;
    const long long cols = (long long)nruns * g.ny * ((g.nz + z - 1) / z);
    const long long cost = ((cols + slots - 1) / slots) * (long long)(z + 1);
    if (best < 0 || cost < best) { best = cost; Z = z; }
  }
  const char* zs = getenv("SC_V7_Z");
  if (zs && atoi(zs) > 0) Z = atoi(zs) < g.nz ? atoi(zs) : g.nz;
  P.runx = R;
  P.zseg = Z;
  const int ncols = nruns * g.ny * ((g.nz + Z - 1) / Z);
  const int grid = ncols < slots ? ncols : slots;
  if (grid > 0) {
    if (two) v7::k_v7_lines<NI, 2><<<grid, nthr, smem, st>>>(P, ncols, nruns);
    else v7::k_v7_lines<NI, 1><<<grid, nthr, smem, st>>>(P, ncols, nruns);
  }
  (*nl)++;
  const unsigned rows = (unsigned)((g.ny + 1) * (g.nz + 1));
  if (P.dotp) v7::k_v7_assemble<NI, true><<<rows, V7B<NI>::BT, 0, st>>>(P);
  else v7::k_v7_assemble<NI, false><<<rows, V7B<NI>::BT, 0, st>>>(P);
  (*nl)++;
  v7::k_v7_padding<<<1, 256, 0, st>>>(g, P.y);
  (*nl)++;
  return cudaGetLastError();
}

int launch_apply_v7(const Geom& g, const double* x, double* y, double* u0, double* u1, const double* done,
                    const void* coef, double* dotp, void* stream, int* nl, void* events) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  V7Params P;
  memset(&P, 0, sizeof(P));
  P.g = g; P.x = x; P.y = y; P.u0 = u0; P.u1 = u1; P.done = done; P.dotp = dotp;
  memcpy(&P.cf, coef, sizeof(V7Coef));
  if (ev) cudaEventRecord(ev[0], st);
  int e = 0;
  switch (g.ni) {
    case 2: e = launch_v7_t<2>(P, st, nl); break;
    case 3: e = launch_v7_t<3>(P, st, nl); break;
    case 4: e = launch_v7_t<4>(P, st, nl); break;
    case 5: e = launch_v7_t<5>(P, st, nl); break;
    case 6: e = launch_v7_t<6>(P, st, nl); break;
    case 7: e = launch_v7_t<7>(P, st, nl); break;
    case 8: e = launch_v7_t<8>(P, st, nl); break;
    case 9: e = launch_v7_t<9>(P, st, nl); break;
    case 10: e = launch_v7_t<10>(P, st, nl); break;
    case 11: e = launch_v7_t<11>(P, st, nl); break;
    case 12: e = launch_v7_t<12>(P, st, nl); break;
    case 13: e = launch_v7_t<13>(P, st, nl); break;
    case 14: e = launch_v7_t<14>(P, st, nl); break;
    case 15: e = launch_v7_t<15>(P, st, nl); break;
    case 16: e = launch_v7_t<16>(P, st, nl); break;
    case 17: e = launch_v7_t<17>(P, st, nl); break;
    case 18: e = launch_v7_t<18>(P, st, nl); break;
    case 19: e = launch_v7_t<19>(P, st, nl); break;
    case 20: e = launch_v7_t<20>(P, st, nl); break;
    case 21: e = launch_v7_t<21>(P, st, nl); break;
    case 22: e = launch_v7_t<22>(P, st, nl); break;
    case 23: e = launch_v7_t<23>(P, st, nl); break;
    default: return (int)cudaErrorInvalidValue;
  }
  if (ev) cudaEventRecord(ev[1], st);
  return e;
}

}  // namespace sc
