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
// Every free entry's elements lie inside the domain on one rank, so the primary coefficients are
// the uniform-grid constants; Dirichlet entries are written as 0 and read as 0.
#include <cuda_runtime.h>
#include <string.h>
#include <vector>
#include "sc_device.cuh"

namespace sc {

struct V7Coef {
  double c[3][8];         // d_{d+1} a0_m  (faces in / out, parity form)
  double dinv[343];       // D^{-1}(i,j,k), i fastest (n_I^3 <= 343)
  double a0[8], ap[8], lam[8];
  double fd[3][49];       // face self: 2 (d0 w0 + d_n K00 + d_a w0 Lam_a + d_b w0 Lam_b), in-plane (a, b)
  double kf[3];           // d_n K0p (opposite faces)
  double ef[3][3];        // face <- edge: 2 d w0 (per direction d, for the face normal n)
  double eself[3][8];     // edge self: 4 d0 w0^2 + 4 d_e w0^2 Lam_m + 4 (d_o1 + d_o2) w0 K00
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
  V7Coef cf;
};

namespace v7 {

constexpr int RUN = 16;   // elements per CTA of pass A (a contiguous x-run)

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

// A work item is an x-run of RUN elements (ex0 .. ex0 + cnt - 1, ey, ez).  Its inputs are five
// contiguous skeleton ranges: the x-faces ex0 .. ex0 + cnt (one row), the y-faces of rows ey, ey + 1 and
// the z-faces of planes ez, ez + 1 (cnt faces each).  Each range is bulk-copied (cp.async.bulk, one
// mbarrier transaction per item) as its 16-byte aligned superset into a slot, so the range starts at
// slot + (start & 1).  Dirichlet rows are not copied: the lanes read a zero row instead (as they do for
// the Dirichlet x-faces fx = 0, nx).
template <int NI, int STAGES>
struct V7A {
  static constexpr int N2 = NI * NI;
  static constexpr int SX = ((RUN + 1) * N2 + 2 + 1) & ~1;   // x-face row slot (doubles, even)
  static constexpr int SR = (RUN * N2 + 2 + 1) & ~1;         // y / z row slot
  static constexpr int STAGE = SX + 4 * SR;
  static constexpr int PJ = NI + 1, PK = NI + 1;
  static constexpr int PKK = di_pk(PJ, PK);
  static constexpr int ND = ((PKK * PK + 2) + 1) & ~1;
  static constexpr int SMEM = (STAGES * STAGE + SR + ND) * 8;   // the stages, the zero row, D^{-1}
};

struct __align__(16) Item {
  int ex0, cnt, ey, ez;
  int par, dirm;    // bit r: range r starts at an odd index / is a Dirichlet row
  long long s[5];   // range starts: x row, y rows ey / ey + 1, z planes ez / ez + 1
  bool dir[5];      // Dirichlet row (not copied)
};

template <int NI, int R = RUN>
__device__ __forceinline__ Item decode(const Geom& g, int item, int nruns) {
  constexpr int N2 = NI * NI;
  Item it;
  // rows (ey, ez) in chunks of 8 layers, ez fastest inside a chunk: the rows that share a y-face are
  // nruns items apart, those that share a z-face 8 nruns (both inside the L2-resident window)
  const int rx = item % nruns, rest = item / nruns;
  const int zc = rest / (g.ny * 8), rr = rest - zc * g.ny * 8;
  const int nzc = min(8, g.nz - 8 * zc);
  it.ey = rr / nzc;
  it.ez = 8 * zc + (rr - it.ey * nzc);
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

// Pass A: persistent CTAs of 4 warps, items blockIdx.x + n gridDim.x, the loads of item n + 2 in flight
// while item n computes (two stages).  lane = (element of the run, parity class) as in v6.
template <int NI, int STAGES>
__global__ void __launch_bounds__(128, STAGES == 1 ? 4 : 3) k_v7_cond(const __grid_constant__ V7Params P, int nitems, int nruns) {
  if (P.done != nullptr && *P.done != 0.0) return;
  using A = V7A<NI, STAGES>;
  constexpr int N2 = NI * NI, M = (NI + 1) / 2;
  constexpr int PJ = A::PJ, PKK = A::PKK;
  const Geom& g = P.g;
  const V7Coef& cf = P.cf;
  const int nx = g.nx, ny = g.ny;
  extern __shared__ __align__(16) double smem[];
  double* const zrow = smem + STAGES * A::STAGE;
  double* const sD = zrow + A::SR;
  __shared__ double sC[3][8], sA0[8], sAP[8];
  __shared__ unsigned long long mbar[2];
  const int tid = threadIdx.x;
  for (int t = tid; t < A::SR; t += 128) zrow[t] = 0.0;
  // D^{-1} at i + PJ j + PKK k with the 8 class bases on distinct bank pairs (cf. kernels_v6.cu di_pk)
  for (int t = tid; t < A::ND; t += 128) {
    const int k = t / PKK, r = t - k * PKK, j = r / PJ, i = r - j * PJ;
    sD[t] = (i < NI && j < NI && k < NI) ? cf.dinv[i + NI * (j + NI * k)] : 0.0;
  }
  if (tid < 24) sC[tid / 8][tid % 8] = (tid % 8) < NI ? cf.c[tid / 8][tid % 8] : 0.0;
  if (tid < 8) {
    sA0[tid] = cf.a0[tid];
    sAP[tid] = cf.ap[tid];
  }
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      const int item = blockIdx.x + s * gridDim.x;
      if (item < nitems) issue_item<NI, A::SX, A::SR>(P, decode<NI>(g, item, nruns), smem + s * A::STAGE, &mbar[s]);
    }
  }
  const int warp = tid >> 5, lane = tid & 31;
  const int el = warp * 4 + (lane >> 3);          // element of the run
  const int cls = lane & 7, si = cls >> 2, sj = (cls >> 1) & 1, sk = cls & 1;
  const int CI = (NI - si + 1) >> 1, CJ = (NI - sj + 1) >> 1, CK = (NI - sk + 1) >> 1;
  const double gi = si ? -1.0 : 1.0, gj = sj ? -1.0 : 1.0, gk = sk ? -1.0 : 1.0;
  const double* const Dc = sD + si + PJ * sj + PKK * sk;
  for (int n = 0;; ++n) {
    const int item = blockIdx.x + n * gridDim.x;
    if (item >= nitems) break;
    const int b = STAGES == 1 ? 0 : (n & 1);
    const Item it = decode<NI>(g, item, nruns);
    double* const stage = smem + b * A::STAGE;
    mbar_wait(&mbar[b], (unsigned)((STAGES == 1 ? n : (n >> 1)) & 1));
    const bool act = el < it.cnt;
    const int ex = it.ex0 + el, ey = it.ey, ez = it.ez;
    // face rows of the element (entries (a, b) at a + NI b); Dirichlet faces / rows read the zero row
    const double* const X = stage + (it.s[0] & 1);
    const double* Wf = (ex > 0 && ex < nx) ? X + el * N2 : zrow;
    const double* Ef = (ex + 1 < nx) ? X + (el + 1) * N2 : zrow;
    const double* Yf[2];
    const double* Zf[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      Yf[s] = it.dir[1 + s] ? zrow : stage + A::SX + s * A::SR + (it.s[1 + s] & 1) + el * N2;
      Zf[s] = it.dir[3 + s] ? zrow : stage + A::SX + (2 + s) * A::SR + (it.s[3 + s] & 1) + el * N2;
    }
    {
      const double* W = Wf + sj + NI * sk;      // x-face entries (j, k)
      const double* E = Ef + sj + NI * sk;
      const double* S = Yf[0] + si + NI * sk;   // y-face entries (i, k)
      const double* Nn = Yf[1] + si + NI * sk;
      const double* B = Zf[0] + si + NI * sj;   // z-face entries (i, j)
      const double* T = Zf[1] + si + NI * sj;
      double c1[M];
#pragma unroll
      for (int ii = 0; ii < M; ++ii) c1[ii] = sC[0][si + 2 * ii];
      double zin[M][M], qz[M][M];
#pragma unroll
      for (int ii = 0; ii < M; ++ii)
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
          zin[ii][jj] = (ii < CI && jj < CJ) ? fma(gk, T[2 * ii + 2 * NI * jj], B[2 * ii + 2 * NI * jj]) : 0.0;
          qz[ii][jj] = 0.0;
        }
      // output rows (entries of the element's faces in U0 / U1)
      double* const uxw = P.u0 + g.off_f[0] + (ex + (long long)(nx + 1) * (ey + (long long)ny * ez)) * N2;   // face ex
      double* const uxe = P.u1 + g.off_f[0] + (ex + 1 + (long long)(nx + 1) * (ey + (long long)ny * ez)) * N2;
      double* const uys = P.u0 + g.off_f[1] + (ex + (long long)nx * (ey + (long long)(ny + 1) * ez)) * N2;
      double* const uyn = P.u1 + g.off_f[1] + (ex + (long long)nx * (ey + 1 + (long long)(ny + 1) * ez)) * N2;
      double* const uzb = P.u0 + g.off_f[2] + (ex + (long long)nx * (ey + (long long)ny * ez)) * N2;
      double* const uzt = P.u1 + g.off_f[2] + (ex + (long long)nx * (ey + (long long)ny * (ez + 1))) * N2;
#pragma unroll
      for (int kk = 0; kk < M; ++kk) {
        const double c3 = sC[2][sk + 2 * kk];
        double yin[M], qy[M];
#pragma unroll
        for (int ii = 0; ii < M; ++ii) {
          yin[ii] = (ii < CI && kk < CK) ? fma(gj, Nn[2 * ii + 2 * NI * kk], S[2 * ii + 2 * NI * kk]) : 0.0;
          qy[ii] = 0.0;
        }
        double qx[M];
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
          const double c2 = sC[1][sj + 2 * jj];
          const int ox = 2 * jj + 2 * NI * kk;
          const double xin = (jj < CJ && kk < CK) ? fma(gi, E[ox], W[ox]) : 0.0;
          qx[jj] = 0.0;
#pragma unroll
          for (int ii = 0; ii < M; ++ii) {
            const double u = fma(c1[ii], xin, fma(c2, yin[ii], c3 * zin[ii][jj]));
            const double v = u * Dc[2 * ii + 2 * PJ * jj + 2 * PKK * kk];
            qx[jj] = fma(c1[ii], v, qx[jj]);
            qy[ii] = fma(c2, v, qy[ii]);
            qz[ii][jj] = fma(c3, v, qz[ii][jj]);
          }
        }
        // x pair (s_i = 0 / 1: lane ^ 4): W part -(Q0 + Q1) (s_i = 0 lane), E part -(Q0 - Q1) (s_i = 1 lane)
        double qpx[M];
#pragma unroll
        for (int jj = 0; jj < M; ++jj) qpx[jj] = __shfl_xor_sync(0xffffffffu, qx[jj], 4);
#pragma unroll
        for (int jj = 0; jj < M; ++jj)
          if (act && jj < CJ && kk < CK) {
            if (si == 0) __stcs(uxw + sj + 2 * jj + NI * (sk + 2 * kk), -(qx[jj] + qpx[jj]));
            else __stcs(uxe + sj + 2 * jj + NI * (sk + 2 * kk), qx[jj] - qpx[jj]);
          }
        double qpy[M];   // y pair (lane ^ 2): S -(Q0 + Q1), N -(Q0 - Q1)
#pragma unroll
        for (int ii = 0; ii < M; ++ii) qpy[ii] = __shfl_xor_sync(0xffffffffu, qy[ii], 2);
#pragma unroll
        for (int ii = 0; ii < M; ++ii)
          if (act && ii < CI && kk < CK) {
            if (sj == 0) __stcs(uys + si + 2 * ii + NI * (sk + 2 * kk), -(qy[ii] + qpy[ii]));
            else __stcs(uyn + si + 2 * ii + NI * (sk + 2 * kk), qy[ii] - qpy[ii]);
          }
      }
#pragma unroll
      for (int ii = 0; ii < M; ++ii)   // z pair (lane ^ 1): B -(Q0 + Q1), T -(Q0 - Q1)
#pragma unroll
        for (int jj = 0; jj < M; ++jj) {
          const double qp = __shfl_xor_sync(0xffffffffu, qz[ii][jj], 1);
          if (act && ii < CI && jj < CJ) {
            if (sk == 0) __stcs(uzb + si + 2 * ii + NI * (sj + 2 * jj), -(qz[ii][jj] + qp));
            else __stcs(uzt + si + 2 * ii + NI * (sj + 2 * jj), qz[ii][jj] - qp);
          }
        }
    }
    // Edge line sums of the primary part (the K~ rows of an edge couple it to the face
    // interiors along lines).  An interior edge's four face lines belong to two of its elements: the
    // element on its high side in both transverse directions gives the a0-weighted lines of its low
    // faces (stored in U0 at the edge), the element on its low side gives the ap-weighted lines of its
    // high faces (stored in U1 at the edge).  lane cls = entry m of the edge (cls < NI).
    if (act && cls < NI) {
      const int m = cls;
      const long long nx1 = nx + 1, ny1 = ny + 1;
      double s0, s1;
      // x-edges: el01 sum_j w_j F_z(m, j) + el02 sum_k w_k F_y(m, k)
      s0 = 0.0; s1 = 0.0;
#pragma unroll
      for (int q = 0; q < NI; ++q) {
        s0 = fma(sA0[q], cf.el[0][1] * Zf[0][m + NI * q] + cf.el[0][2] * Yf[0][m + NI * q], s0);
        s1 = fma(sAP[q], cf.el[0][1] * Zf[1][m + NI * q] + cf.el[0][2] * Yf[1][m + NI * q], s1);
      }
      __stcs(P.u0 + g.off_e[0] + (ex + (long long)nx * (ey + ny1 * ez)) * NI + m, s0);
      __stcs(P.u1 + g.off_e[0] + (ex + (long long)nx * (ey + 1 + ny1 * (ez + 1))) * NI + m, s1);
      // y-edges: el10 sum_i w_i F_z(i, m) + el12 sum_k w_k F_x(m, k)
      s0 = 0.0; s1 = 0.0;
#pragma unroll
      for (int q = 0; q < NI; ++q) {
        s0 = fma(sA0[q], cf.el[1][0] * Zf[0][q + NI * m] + cf.el[1][2] * Wf[m + NI * q], s0);
        s1 = fma(sAP[q], cf.el[1][0] * Zf[1][q + NI * m] + cf.el[1][2] * Ef[m + NI * q], s1);
      }
      __stcs(P.u0 + g.off_e[1] + (ex + nx1 * (ey + (long long)ny * ez)) * NI + m, s0);
      __stcs(P.u1 + g.off_e[1] + (ex + 1 + nx1 * (ey + (long long)ny * (ez + 1))) * NI + m, s1);
      // z-edges: el20 sum_i w_i F_y(i, m) + el21 sum_j w_j F_x(j, m)
      s0 = 0.0; s1 = 0.0;
#pragma unroll
      for (int q = 0; q < NI; ++q) {
        s0 = fma(sA0[q], cf.el[2][0] * Yf[0][q + NI * m] + cf.el[2][1] * Wf[q + NI * m], s0);
        s1 = fma(sAP[q], cf.el[2][0] * Yf[1][q + NI * m] + cf.el[2][1] * Ef[q + NI * m], s1);
      }
      __stcs(P.u0 + g.off_e[2] + (ex + nx1 * (ey + ny1 * ez)) * NI + m, s0);
      __stcs(P.u1 + g.off_e[2] + (ex + 1 + nx1 * (ey + 1 + ny1 * ez)) * NI + m, s1);
    }
    // release the stage: every lane is done reading it; then the loads of item n + 2 go into it
    fence_proxy_async();
    __syncthreads();
    const int nxt = item + STAGES * gridDim.x;
    if (tid == 0 && nxt < nitems) issue_item<NI, A::SX, A::SR>(P, decode<NI>(g, nxt, nruns), stage, &mbar[b]);
  }
}

// ------------------------------------------------------------------------------------ pass A, line form
// Pass A with lane = (element, x-line (j, k)) instead of (element, parity class): no padded points
// (n_I^3 points per element instead of 8 ceil(n_I/2)^3), per-lane constants (D^{-1}(., j, k), the y / z
// coefficients and signs) in registers for the whole kernel, and three phases per item:
//  X: faces-in + D^{-1} along the lane's x-line (the y / z inputs of the line's points are the face
//     values (S +- N)(i, k), (B +- T)(i, j); the sign is the parity of the lane's j / k, P:302 sigma), the
//     x faces-out as the two parity sums Q_even / Q_odd of the line (W part -(Qe + Qo), E part -(Qe - Qo)),
//     uhat = D^{-1} (...) stored to shared memory;
//  Y: lane = (i, k): y faces-out = parity sums over j of c2_j uhat(i, j, k);
//  Z: lane = (i, j): z faces-out over k; and the edge line sums (U0 / U1 at the edges) as in k_v7_cond.
// Every output row of a group of elements is one contiguous skeleton range: coalesced stores.
template <int NI, int STAGES>
struct V8A {
  static constexpr int N2 = NI * NI, N3 = N2 * NI;
  // elements per item (x-run) and per thread group (G N2 <= 256 threads in the line phases)
  static constexpr int R = NI >= 6 ? 8 : (NI >= 4 ? 16 : 32);
  static constexpr int G = NI >= 6 ? 4 : (NI == 5 ? 8 : (NI == 4 ? 16 : (NI == 3 ? 16 : 32)));
  static constexpr int NT = ((G * N2 + 31) / 32) * 32;       // threads per CTA
  static constexpr int EWF = ((R * 2 * NI + 31) / 32) * 32;  // edge-phase slots per family (warp-rounded)
  static constexpr int MINB = STAGES == 2 ? 3 : (NT <= 128 ? 8 : (NT <= 160 ? 6 : 4));
  static constexpr int SX = ((R + 1) * N2 + 2 + 1) & ~1;
  static constexpr int SR = (R * N2 + 2 + 1) & ~1;
  static constexpr int STAGE = SX + 4 * SR;
  static constexpr int VS = N3 + (N3 % 2 == 0 ? 1 : 0);      // uhat per element (odd stride)
  static constexpr int SMEM = (STAGES * STAGE + SR + R * VS) * 8;
};

// Edge line sums of one element family (see k_v7_cond): F = 0 x-edges, 1 y-edges, 2 z-edges; hi = 0: the
// a0-weighted lines of the element's low faces (U0 at its low edge), hi = 1: the ap = sigma a0 weighted
// lines of its high faces (U1 at its high edge).  Line q-strides are compile-time per family.
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
__global__ void __launch_bounds__(V8A<NI, STAGES>::NT, V8A<NI, STAGES>::MINB) k_v7_lines(const __grid_constant__ V7Params P, int nitems,
                                                                  int nruns) {
  if (P.done != nullptr && *P.done != 0.0) return;
  using A = V8A<NI, STAGES>;
  constexpr int N2 = NI * NI, G = A::G, R = A::R;
  constexpr int EWF = A::EWF;
  const Geom& g = P.g;
  const V7Coef& cf = P.cf;
  const int nx = g.nx, ny = g.ny;
  const long long nx1 = nx + 1, ny1 = ny + 1;
  extern __shared__ __align__(16) double smem[];
  double* const zrow = smem + STAGES * A::STAGE;
  double* const sv = zrow + A::SR;
  __shared__ unsigned long long mbar[2];
  __shared__ Item sit[2];   // the decoded item of each stage (written by the issuing thread before its arrive)
  const int tid = threadIdx.x;
  for (int t = tid; t < A::SR; t += A::NT) zrow[t] = 0.0;
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < STAGES; ++s) {
      const int item = blockIdx.x + s * gridDim.x;
      if (item < nitems) {
        sit[s] = decode<NI, R>(g, item, nruns);
        issue_item<NI, A::SX, A::SR>(P, sit[s], smem + s * A::STAGE, &mbar[s]);
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
  for (int n = 0;; ++n) {
    const int item = blockIdx.x + n * gridDim.x;
    if (item >= nitems) break;
    const int b = STAGES == 1 ? 0 : (n & 1);
    double* const stage = smem + b * A::STAGE;
    mbar_wait(&mbar[b], (unsigned)((STAGES == 1 ? n : (n >> 1)) & 1));
    const int4 ih = *reinterpret_cast<const int4*>(&sit[b]);   // ex0, cnt, ey, ez
    const int par = sit[b].par, dirm = sit[b].dirm;
    const int ex0 = ih.x, cnt = ih.y, ey = ih.z, ez = ih.w;
    double* const X = stage + (par & 1);
    // the Dirichlet x-faces fx = 0, nx of a boundary run read as zero (block-uniform branch)
    if (ex0 == 0 || ex0 + cnt == nx) {
      if (tid < N2) {
        if (ex0 == 0) X[tid] = 0.0;
        if (ex0 + cnt == nx) X[cnt * N2 + tid] = 0.0;
      }
      __syncthreads();
    }
    const double* Yr[2];
    const double* Zr[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      Yr[s] = ((dirm >> (1 + s)) & 1) ? zrow : stage + A::SX + s * A::SR + ((par >> (1 + s)) & 1);
      Zr[s] = ((dirm >> (3 + s)) & 1) ? zrow : stage + A::SX + (2 + s) * A::SR + ((par >> (3 + s)) & 1);
    }
    // output bases of the item's first element (face / edge rows are contiguous along x)
    const long long d01 = P.u1 - P.u0;
    double* const ux = P.u0 + g.off_f[0] + (ex0 + nx1 * (ey + (long long)ny * ez)) * N2 + l;
    double* const uy = P.u0 + g.off_f[1] + (ex0 + (long long)nx * (ey + ny1 * ez)) * N2 + l;
    double* const uz = P.u0 + g.off_f[2] + (ex0 + (long long)nx * (ey + (long long)ny * ez)) * N2 + l;
    // ---- phase X
    if (lane_on) {
#pragma unroll
      for (int gr = 0; gr < R / G; ++gr) {
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
        if (el < cnt) {
          __stcs(ux + el * N2, -(qe + qo));              // face ex (the element's W face) in U0
          __stcs(ux + d01 + (el + 1) * N2, qo - qe);     // face ex + 1 (E) in U1
        }
      }
    }
    __syncthreads();
    // ---- phases Y, Z
    if (lane_on) {
#pragma unroll
      for (int gr = 0; gr < R / G; ++gr) {
        const int el = gr * G + eg;
        if (el < cnt) {
          const double* const v = sv + el * A::VS;
          double qe = 0.0, qo = 0.0;
#pragma unroll
          for (int j = 0; j < NI; ++j) {   // lane (i, k) = (la, lb)
            const double t = cf.c[1][j] * v[la + NI * (j + NI * lb)];
            if (j & 1) qo += t;
            else qe += t;
          }
          __stcs(uy + el * N2, -(qe + qo));                                // S face (ey) in U0
          __stcs(uy + d01 + (long long)nx * N2 + el * N2, qo - qe);        // N face (ey + 1) in U1
          qe = 0.0; qo = 0.0;
#pragma unroll
          for (int k = 0; k < NI; ++k) {   // lane (i, j) = (la, lb)
            const double t = cf.c[2][k] * v[l + N2 * k];
            if (k & 1) qo += t;
            else qe += t;
          }
          __stcs(uz + el * N2, -(qe + qo));                                   // B face (ez) in U0
          __stcs(uz + d01 + (long long)nx * ny * N2 + el * N2, qo - qe);      // T face (ez + 1) in U1
        }
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
        double s;
        long long dst;
        if (ef == 0) {
          s = edge_line<NI, 0>(cf, zb, zt, ys, yn, w, e, ehi, em);
          dst = g.off_e[0] + (ex + (long long)nx * (ey + ehi + ny1 * (ez + ehi))) * NI + em;
        } else if (ef == 1) {
          s = edge_line<NI, 1>(cf, zb, zt, ys, yn, w, e, ehi, em);
          dst = g.off_e[1] + (ex + ehi + nx1 * (ey + (long long)ny * (ez + ehi))) * NI + em;
        } else {
          s = edge_line<NI, 2>(cf, zb, zt, ys, yn, w, e, ehi, em);
          dst = g.off_e[2] + (ex + ehi + nx1 * (ey + ehi + ny1 * ez)) * NI + em;
        }
        __stcs((ehi ? P.u1 : P.u0) + dst, s);
      }
    }
    fence_proxy_async();
    __syncthreads();
    const int nxt = item + STAGES * gridDim.x;
    if (tid == 0 && nxt < nitems) {
      sit[b] = decode<NI, R>(g, nxt, nruns);
      issue_item<NI, A::SX, A::SR>(P, sit[b], stage, &mbar[b]);
    }
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

// One face entry: y = fd u + kf (u_lo + u_hi) + wA (a0_ea A0[eb] + ap_ea A1[eb]) + wB (a0_eb B0[ea] + ap_eb B1[ea])
//                     + U0 + U1   (the primary part of Eq. eq:east_east_primary_part_transformed summed over
// the face's two elements, + the two condensed parts from pass A)
template <int NI>
__device__ __forceinline__ double face_entry(const V7Params& P, const double* sfd, const double* sa0, const double* sap,
                                             long long i, int e, int ea, int eb, long long so, bool olo, bool ohi,
                                             long long ia0, long long ia1, bool oka0, bool oka1, long long ib0,
                                             long long ib1, bool okb0, bool okb1, double wA, double wB, double kf,
                                             double& u) {
  const double* __restrict__ x = P.x;
  u = __ldg(x + i);
  const double uo = ldv(x, i - so, olo) + ldv(x, i + so, ohi);
  const double ea_ = sa0[ea] * ldv(x, ia0 + eb, oka0) + sap[ea] * ldv(x, ia1 + eb, oka1);
  const double eb_ = sa0[eb] * ldv(x, ib0 + ea, okb0) + sap[eb] * ldv(x, ib1 + ea, okb1);
  return sfd[e] * u + kf * uo + wA * ea_ + wB * eb_ + __ldcs(P.u0 + i) + __ldcs(P.u1 + i);
}

template <int NI, bool DOT>
__global__ void __launch_bounds__(256, 4) k_v7_assemble(const __grid_constant__ V7Params P) {
  if (P.done != nullptr && *P.done != 0.0) return;
  constexpr int N2 = NI * NI;
  const Geom& g = P.g;
  const V7Coef& cf = P.cf;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long nx1 = nx + 1, ny1 = ny + 1;
  const double* __restrict__ x = P.x;
  double* __restrict__ y = P.y;
  const int cy = blockIdx.x % (ny + 1), cz = blockIdx.x / (ny + 1);
  // lane-indexed coefficients from shared memory (indexed kernel-parameter loads serialise per address)
  __shared__ double sfd[3][N2], sa0[8], sap[8], sself[3][8];
  for (int q = threadIdx.x; q < 3 * N2; q += blockDim.x) sfd[q / N2][q % N2] = cf.fd[q / N2][q % N2];
  if (threadIdx.x < 8) {
    sa0[threadIdx.x] = cf.a0[threadIdx.x];
    sap[threadIdx.x] = cf.ap[threadIdx.x];
    for (int e = 0; e < 3; ++e) sself[e][threadIdx.x] = cf.eself[e][threadIdx.x];
  }
  __syncthreads();
  double dot = 0.0;
  const bool zb0 = !zdir(g, cz), zb1 = !zdir(g, cz + 1);   // planes cz, cz + 1 free (as z-planes)
  // ---------------- x-faces (fx, ey = cy, ez = cz), fx = 0..nx; in-plane (ea, eb) = (j, k)
  if (cy < ny && cz < nz) {
    const long long base = g.off_f[0] + nx1 * (cy + (long long)ny * cz) * N2;
    const long long za = g.off_e[2] + nx1 * (cy + ny1 * cz) * NI;   // z-edges (fx, cy, cz); (fx, cy + 1, cz) at + nx1 NI
    const long long yb = g.off_e[1] + nx1 * (cy + (long long)ny * cz) * NI;   // y-edges (fx, cy, cz); cz + 1 at + nx1 ny NI
    const bool oka0 = in_f(cy, ny), oka1 = in_f(cy + 1, ny);
    const double wA = cf.ef[0][1], wB = cf.ef[0][2], kf = cf.kf[0];
    for (int t = threadIdx.x; t < (nx + 1) * N2; t += blockDim.x) {
      const int fx = t / N2, e = t - fx * N2, eb = e / NI, ea = e - eb * NI;
      double yv = 0.0;
      if (in_f(fx, nx)) {
        double u;
        const long long ia0 = za + (long long)fx * NI, ib0 = yb + (long long)fx * NI;
        yv = face_entry<NI>(P, sfd[0], sa0, sap, base + t, e, ea, eb, N2, fx - 1 > 0, fx + 1 < nx, ia0, ia0 + nx1 * NI,
                            oka0, oka1, ib0, ib0 + nx1 * ny * NI, zb0, zb1, wA, wB, kf, u);
        if (DOT) dot = fma(u, yv, dot);
      }
      __stcs(y + base + t, yv);
    }
  }
  // ---------------- y-faces (ex, fy = cy, ez = cz), ex = 0..nx-1; in-plane (ea, eb) = (i, k)
  if (cz < nz) {
    const long long base = g.off_f[1] + (long long)nx * (cy + ny1 * cz) * N2;
    const long long za = g.off_e[2] + nx1 * (cy + ny1 * cz) * NI;   // z-edges (ex, cy, cz), (ex + 1, ...) at + NI
    const long long xb = g.off_e[0] + (long long)nx * (cy + ny1 * cz) * NI;   // x-edges (ex, cy, cz); cz + 1 at + nx ny1 NI
    const bool fr = in_f(cy, ny);
    const double wA = cf.ef[1][0], wB = cf.ef[1][2], kf = cf.kf[1];
    for (int t = threadIdx.x; t < nx * N2; t += blockDim.x) {
      const int ex = t / N2, e = t - ex * N2, eb = e / NI, ea = e - eb * NI;
      double yv = 0.0;
      if (fr) {
        double u;
        const long long ia0 = za + (long long)ex * NI, ib0 = xb + (long long)ex * NI;
        yv = face_entry<NI>(P, sfd[1], sa0, sap, base + t, e, ea, eb, (long long)nx * N2, cy - 1 > 0, cy + 1 < ny, ia0,
                            ia0 + NI, in_f(ex, nx), in_f(ex + 1, nx), ib0, ib0 + (long long)nx * ny1 * NI, zb0, zb1, wA,
                            wB, kf, u);
        if (DOT) dot = fma(u, yv, dot);
      }
      __stcs(y + base + t, yv);
    }
  }
  // ---------------- z-faces (ex, ey = cy, fz = cz), ex = 0..nx-1; in-plane (ea, eb) = (i, j)
  if (cy < ny) {
    const long long base = g.off_f[2] + (long long)nx * (cy + (long long)ny * cz) * N2;
    const long long ya = g.off_e[1] + nx1 * (cy + (long long)ny * cz) * NI;   // y-edges (ex, cy, cz), (ex + 1, ...) at + NI
    const long long xb = g.off_e[0] + (long long)nx * (cy + ny1 * cz) * NI;   // x-edges (ex, cy, cz); cy + 1 at + nx NI
    const bool fr = zb0;
    const bool olo = cz - 1 >= 0 && !zdir(g, cz - 1), ohi = cz + 1 <= nz && !zdir(g, cz + 1);
    const bool okb0 = in_f(cy, ny), okb1 = in_f(cy + 1, ny);
    const double wA = cf.ef[2][0], wB = cf.ef[2][1], kf = cf.kf[2];
    for (int t = threadIdx.x; t < nx * N2; t += blockDim.x) {
      const int ex = t / N2, e = t - ex * N2, eb = e / NI, ea = e - eb * NI;
      double yv = 0.0;
      if (fr) {
        double u;
        const long long ia0 = ya + (long long)ex * NI, ib0 = xb + (long long)ex * NI;
        yv = face_entry<NI>(P, sfd[2], sa0, sap, base + t, e, ea, eb, (long long)nx * ny * N2, olo, ohi, ia0, ia0 + NI,
                            in_f(ex, nx), in_f(ex + 1, nx), ib0, ib0 + (long long)nx * NI, okb0, okb1, wA, wB, kf, u);
        if (DOT) dot = fma(u, yv, dot);
      }
      __stcs(y + base + t, yv);
    }
  }
  // ---------------- edges: the face-line sums (z-faces (ex, cy-1 / cy, cz) over j and y-faces (ex, cy, cz-1 / cz)
  // over k for an x-edge, cyclically for y / z) come from pass A in U0 + U1 at the edge's entries.
  // x-edges (ex, fy = cy, fz = cz), entry m
  {
    const long long base = g.off_e[0] + (long long)nx * (cy + ny1 * cz) * NI;
    const bool fr = in_f(cy, ny) && zb0;
    const bool ylo = cz - 1 >= 0 && !zdir(g, cz - 1), yhi = cz + 1 <= nz && !zdir(g, cz + 1);
    for (int t = threadIdx.x; t < nx * NI; t += blockDim.x) {
      const int ex = t / NI, m = t - ex * NI;
      const long long i0 = base + t;
      double yv = 0.0;
      if (fr) {
        const double u = __ldg(x + i0);
        const double vw = ldv(x, g.off_v + ex + nx1 * (cy + ny1 * cz), in_f(ex, nx));
        const double ve = ldv(x, g.off_v + ex + 1 + nx1 * (cy + ny1 * cz), in_f(ex + 1, nx));
        const double nb_y = ldv(x, i0 - (long long)nx * NI, cy - 1 > 0) + ldv(x, i0 + (long long)nx * NI, cy + 1 < ny);
        const long long pl = (long long)nx * ny1 * NI;
        const double nb_z = ldv(x, i0 - pl, ylo) + ldv(x, i0 + pl, yhi);
        yv = sself[0][m] * u + cf.ev[0] * (sa0[m] * vw + sap[m] * ve) + cf.el[0][1] * cf.K0p * nb_y +
             cf.el[0][2] * cf.K0p * nb_z + __ldcs(P.u0 + i0) + __ldcs(P.u1 + i0);
        if (DOT) dot = fma(u, yv, dot);
      }
      __stcs(y + i0, yv);
    }
  }
  // ---------------- y-edges (fx, ey = cy, fz = cz)
  if (cy < ny) {
    const long long base = g.off_e[1] + nx1 * (cy + (long long)ny * cz) * NI;
    const bool ylo = cz - 1 >= 0 && !zdir(g, cz - 1), yhi = cz + 1 <= nz && !zdir(g, cz + 1);
    for (int t = threadIdx.x; t < (nx + 1) * NI; t += blockDim.x) {
      const int fx = t / NI, m = t - fx * NI;
      const long long i0 = base + t;
      double yv = 0.0;
      if (in_f(fx, nx) && zb0) {
        const double u = __ldg(x + i0);
        const double vs = ldv(x, g.off_v + fx + nx1 * (cy + ny1 * cz), in_f(cy, ny));
        const double vn = ldv(x, g.off_v + fx + nx1 * (cy + 1 + ny1 * cz), in_f(cy + 1, ny));
        const double nb_x = ldv(x, i0 - NI, fx - 1 > 0) + ldv(x, i0 + NI, fx + 1 < nx);
        const long long pl = nx1 * ny * NI;
        const double nb_z = ldv(x, i0 - pl, ylo) + ldv(x, i0 + pl, yhi);
        yv = sself[1][m] * u + cf.ev[1] * (sa0[m] * vs + sap[m] * vn) + cf.el[1][0] * cf.K0p * nb_x +
             cf.el[1][2] * cf.K0p * nb_z + __ldcs(P.u0 + i0) + __ldcs(P.u1 + i0);
        if (DOT) dot = fma(u, yv, dot);
      }
      __stcs(y + i0, yv);
    }
  }
  // ---------------- z-edges (fx, fy = cy, ez = cz)
  if (cz < nz) {
    const long long base = g.off_e[2] + nx1 * (cy + ny1 * cz) * NI;
    const bool fry = in_f(cy, ny);
    for (int t = threadIdx.x; t < (nx + 1) * NI; t += blockDim.x) {
      const int fx = t / NI, m = t - fx * NI;
      const long long i0 = base + t;
      double yv = 0.0;
      if (in_f(fx, nx) && fry) {
        const double u = __ldg(x + i0);
        const double vb = ldv(x, g.off_v + fx + nx1 * (cy + ny1 * cz), zb0);
        const double vt = ldv(x, g.off_v + fx + nx1 * (cy + ny1 * (cz + 1)), zb1);
        const double nb_x = ldv(x, i0 - NI, fx - 1 > 0) + ldv(x, i0 + NI, fx + 1 < nx);
        const double nb_y = ldv(x, i0 - nx1 * NI, cy - 1 > 0) + ldv(x, i0 + nx1 * NI, cy + 1 < ny);
        yv = sself[2][m] * u + cf.ev[2] * (sa0[m] * vb + sap[m] * vt) + cf.el[2][0] * cf.K0p * nb_x +
             cf.el[2][1] * cf.K0p * nb_y + __ldcs(P.u0 + i0) + __ldcs(P.u1 + i0);
        if (DOT) dot = fma(u, yv, dot);
      }
      __stcs(y + i0, yv);
    }
  }
  // ---------------- vertices (fx, cy, cz): lines along the 6 incident edges
  {
    const bool fr = in_f(cy, ny) && zb0;
    const bool zlo_ok = cz - 1 >= 0 && !zdir(g, cz - 1), zhi_ok = cz + 1 <= nz && !zdir(g, cz + 1);
    for (int fx = threadIdx.x; fx <= nx; fx += blockDim.x) {
      const long long i0 = g.off_v + fx + nx1 * (cy + ny1 * cz);
      double yv = 0.0;
      if (fr && in_f(fx, nx)) {
        const double u = __ldg(x + i0);
        const long long xw = g.off_e[0] + (fx - 1 + (long long)nx * (cy + ny1 * cz)) * NI, xe = xw + NI;
        const long long ys = g.off_e[1] + (fx + nx1 * (cy - 1 + (long long)ny * cz)) * NI, yn = ys + nx1 * NI;
        const long long zb = g.off_e[2] + (fx + nx1 * (cy + ny1 * (cz - 1))) * NI, zt = zb + nx1 * ny1 * NI;
        double lx = 0.0, ly = 0.0, lz = 0.0;
#pragma unroll
        for (int q = 0; q < NI; ++q) {
          lx = fma(cf.ap[q], __ldg(x + xw + q), fma(cf.a0[q], __ldg(x + xe + q), lx));
          ly = fma(cf.ap[q], __ldg(x + ys + q), fma(cf.a0[q], __ldg(x + yn + q), ly));
          lz = fma(cf.ap[q], __ldg(x + zb + q), fma(cf.a0[q], __ldg(x + zt + q), lz));
        }
        const double nbx = ldv(x, i0 - 1, fx - 1 > 0) + ldv(x, i0 + 1, fx + 1 < nx);
        const double nby = ldv(x, i0 - nx1, cy - 1 > 0) + ldv(x, i0 + nx1, cy + 1 < ny);
        const long long pl = nx1 * ny1;
        const double nbz = ldv(x, i0 - pl, zlo_ok) + ldv(x, i0 + pl, zhi_ok);
        yv = cf.vself * u + cf.vl[0] * fma(cf.K0p, nbx, lx) + cf.vl[1] * fma(cf.K0p, nby, ly) + cf.vl[2] * fma(cf.K0p, nbz, lz);
        if (DOT) dot = fma(u, yv, dot);
      }
      __stcs(y + i0, yv);
    }
  }
  if (DOT) {
    // block partial of x . y in a fixed order (warp shuffles, then warps in order)
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += red[w];
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

bool v7_supported(int ni) { return ni >= 2 && ni <= 7; }

void v7_make_coef(int ni, const double* d, const double* a0, const double* ap, const double* lam, double K00,
                  double K0p, double w0, std::vector<unsigned char>& out) {
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
  for (int k = 0; k < ni; ++k)
    for (int j = 0; j < ni; ++j)
      for (int i = 0; i < ni; ++i) c.dinv[i + ni * (j + ni * k)] = 1.0 / (d[0] + d[1] * lam[i] + d[2] * lam[j] + d[3] * lam[k]);
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

// Number of pass-B blocks (the p . q partials the PCG sums): one per cell row.
long long v7_dot_parts(const Geom& g) { return (long long)(g.ny + 1) * (g.nz + 1); }

template <int NI>
static int launch_v7_t(V7Params& P, cudaStream_t st, int* nl) {
  const Geom& g = P.g;
  int dev = 0;
  cudaGetDevice(&dev);
  static const char* sg = getenv("SC_V7_STAGES");
  static const char* sa = getenv("SC_V7_A");
  const int two = sg && sg[0] == '2';
  const int lines = !(sa && sa[0] == 'c');
  // per device: dynamic shared memory opt-in and resident CTAs per SM of the chosen pass-A kernel
  static int attr_done[64][2][2] = {{{0}}}, per_sm[64][2][2] = {{{0}}}, nsm_c[64] = {0};
  const void* fn;
  int smem, nthr, run;
  if (lines) {
    fn = two ? (const void*)v7::k_v7_lines<NI, 2> : (const void*)v7::k_v7_lines<NI, 1>;
    smem = two ? v7::V8A<NI, 2>::SMEM : v7::V8A<NI, 1>::SMEM;
    nthr = v7::V8A<NI, 1>::NT;
    run = v7::V8A<NI, 1>::R;
  } else {
    fn = two ? (const void*)v7::k_v7_cond<NI, 2> : (const void*)v7::k_v7_cond<NI, 1>;
    smem = two ? v7::V7A<NI, 2>::SMEM : v7::V7A<NI, 1>::SMEM;
    nthr = 128;
    run = v7::RUN;
  }
  if (dev < 64 && !attr_done[dev][lines][two]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev][lines][two], fn, nthr, smem);
    cudaDeviceGetAttribute(&nsm_c[dev], cudaDevAttrMultiProcessorCount, dev);
    attr_done[dev][lines][two] = 1;
  }
  const int nruns = (g.nx + run - 1) / run;
  const int nitems = nruns * g.ny * g.nz;
  const int slots = (dev < 64 ? max(per_sm[dev][lines][two], 1) * nsm_c[dev] : 148);
  const int grid = nitems < slots ? nitems : slots;
  if (grid > 0) {
    if (lines) {
      if (two) v7::k_v7_lines<NI, 2><<<grid, nthr, smem, st>>>(P, nitems, nruns);
      else v7::k_v7_lines<NI, 1><<<grid, nthr, smem, st>>>(P, nitems, nruns);
    } else {
      if (two) v7::k_v7_cond<NI, 2><<<grid, nthr, smem, st>>>(P, nitems, nruns);
      else v7::k_v7_cond<NI, 1><<<grid, nthr, smem, st>>>(P, nitems, nruns);
    }
  }
  (*nl)++;
  const unsigned rows = (unsigned)((g.ny + 1) * (g.nz + 1));
  if (P.dotp) v7::k_v7_assemble<NI, true><<<rows, 256, 0, st>>>(P);
  else v7::k_v7_assemble<NI, false><<<rows, 256, 0, st>>>(P);
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
    default: return (int)cudaErrorInvalidValue;
  }
  if (ev) cudaEventRecord(ev[1], st);
  return e;
}

}  // namespace sc
