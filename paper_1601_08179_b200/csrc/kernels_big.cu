// Condensed operator v4 for n_I >= 8 (p >= 9), uniform geometry.
//
// One CTA (3-8 warps, BL::NW) per element.  The elements are processed in the 8 parity colours
// (ex, ey, ez mod 2), one launch per colour: two elements of one colour share no face, edge or
// vertex, so the assembly R^ (a8) is a plain read-modify-write of y (zeroed first) --
// deterministic and atomic-free -- and a3 is a plain gather of the element's shell.
//
// Condensed part (Table 2 of PAPER.md P:425-440, faces-in / D^{-1} / faces-out, in the sigma-split
// form ap = sigma a0):
//   u(i,j,k) = c1_i Px^{s_i}(j,k) + c2_j Py^{s_j}(i,k) + c3_k Pz^{s_k}(i,j),   Px^s = W + (-1)^s E, ...
//   v = u D^{-1};  Qx^s(j,k) = sum_{i: s_i = s} c1_i v,  likewise Qy (over j), Qz (over k)
//   W -= Qx^0 + Qx^1, E -= Qx^0 - Qx^1, ...                     (c_d = d_d a0, 7 FP64 ops / point)
// Thread mapping: lane -> j (SW = 16 or 32 lanes per j-group), (warp, half) -> a residue class of
// i (NG = 8 H classes), fully unrolled loop over k.  The k-sums (Qz) complete in registers, the
// i-sums (Qx) in registers over the thread's i values and then across the warps that share the
// parity of i (fixed-order tree through shared memory), the j-sums (Qy) through a per-warp
// shared-memory transpose.  D^{-1} is recomputed per point (reciprocal + 2 Newton steps).
// Primary part (Eq. 26 generalised): faces in the closed form of kernels_col.cu, edges
// and vertices from the arrowhead rows of Ktilde with a0-weighted line sums of faces / edges.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>
#include <vector>
#include "sc_device.cuh"

namespace sc {


struct BigParams {
  Geom g;
  const double* x;
  double* y;
  const double* done;
  BigCoef cf;
};

// Warps per CTA for 8 <= n_I <= 23 (two j-groups of 16 lanes per warp for n_I <= 16, so NG = 2 NW
// residue classes of i).  Measured per n_I at cfg3 sizes (tools/gpu_v4_nw.sh, ms per apply for
// 4 warps -> the table's choice): n_I = 9: 1.99 -> 1.86 (3 warps), 11: 1.74 -> 1.61 (6),
// 12: 1.69 -> 1.51 (3), 13: 1.30 -> 1.25 (7); n_I = 10, 14: 4 warps stay best.
constexpr int nw_small(int ni) { return ni == 9 ? 3 : ni == 11 ? 6 : ni == 12 ? 3 : ni == 13 ? 7 : 4; }

template <int NI>
struct BL {
  static constexpr int N2 = NI * NI;
  static constexpr int SW = NI <= 16 ? 16 : 32;   // lanes per j-group
  static constexpr int H = 32 / SW;                // j-groups per warp
  // warps per CTA: 4 up to n_I = 23 (two or more CTAs share an SM, so one CTA's gather / tree /
  // output phases overlap another's condensed part; measured p=12 -3.6 %, p=16 -4.6 %,
  // p=24 -15 % against 8 warps); 8 from n_I = 24 (one CTA per SM: 213 KB at n_I = 31)
  static constexpr int NW = (NI >= 8 && NI <= 23) ? nw_small(NI) : 8, NT = 32 * NW;
  static constexpr int MINB = NW < 8 ? 2 : 1;
  static constexpr int NG = NW * H;                // residue classes of i
  static constexpr int NIT = (NI + NG - 1) / NG;   // i values per thread
  static constexpr int SH = 6 * N2 + 12 * NI + 8;  // shell: faces w e s n b t | 12 edges | 8 vertices
  static constexpr int O_SH = 0;
  static constexpr int O_P = SH;                   // Px^0 Px^1 Py^0 Py^1 Pz^0 Pz^1
  static constexpr int O_Q = O_P + 6 * N2;         // Qx^0 Qx^1 Qy^0 Qy^1 Qz^0 Qz^1
  static constexpr int O_LS = O_Q + 6 * N2;        // face line sums [6][2][NI][2] (R+, R-)
  static constexpr int O_ES = O_LS + 24 * NI;      // edge line sums [12][2]
  // row stride of the Qy transpose buffers: SW + 2, so that the reduction's lanes (k, s) read
  // rows k at column offset s from 16 distinct bank pairs per half-warp (SW + 1: 2-way conflicts)
  static constexpr int YS = SW + 2;
  static constexpr int O_Y = O_ES + 24;            // [8 H][NI][YS]; reused by the Qx tree
  static constexpr int TOTAL = O_Y + NW * H * NI * YS;
  static_assert((NW / 2) * H * NI * SW <= NW * H * NI * YS, "Qx tree slots");
};

__device__ __forceinline__ void cp_async8b(double* smem, const double* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ double sgn(int m) { return (m & 1) ? -1.0 : 1.0; }
__device__ __forceinline__ double eo_row_b(const double* r, int hi) { return hi ? r[0] - r[1] : r[0] + r[1]; }

// UNI: uniform geometry (the d-dependent coefficients are kernel parameters, constant-bank
// operands); otherwise each CTA derives them from its element's d_e (metric) into shared
// memory (graded / anisotropic non-uniform grids).
template <int NI, bool UNI, int CH>
__global__ void __launch_bounds__(BL<NI>::NT, BL<NI>::MINB) k_apply_big(const __grid_constant__ BigParams P, int colour) {
  using B = BL<NI>;
  constexpr int N2 = B::N2, SW = B::SW, H = B::H, NG = B::NG, YS = B::YS, NT = B::NT, NW = B::NW;
  if (P.done != nullptr && *P.done != 0.0) return;
  extern __shared__ double sm[];
  __shared__ long long sBase[26];
  __shared__ int sDir[26];
  // lane-divergent coefficient lookups go through shared memory (the constant bank serialises
  // them): L[3][32], e[3][32], a0[32], lam[32]
  __shared__ double sT[256];
  const Geom& g = P.g;
  const BigCoef& cf = P.cf;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int cx = colour & 1, cy = (colour >> 1) & 1, cz = colour >> 2;
  const int ncx = (g.nx - cx + 1) >> 1, ncy = (g.ny - cy + 1) >> 1;
  const int bid = blockIdx.x;
  const int ex = cx + 2 * (bid % ncx), ey = cy + 2 * ((bid / ncx) % ncy), ez = cz + 2 * (bid / (ncx * ncy));
  // element geometry: d_e (uniform: the parameter block's)
  double dd[4];
  if constexpr (UNI) {
#pragma unroll
    for (int q = 0; q < 4; ++q) dd[q] = cf.d[q];
  } else {
    metric(g, ex, ey, ez, dd);
  }
  __shared__ double sCg[3 * 32], sDlg[3 * 32];   // non-uniform: c[d][m], dl[d][m] of this element
  for (int t = tid; t < 256; t += NT) {
    if constexpr (UNI) {
      sT[t] = t < 96 ? (&cf.L[0][0])[t] : t < 192 ? (&cf.e[0][0])[t - 96] : t < 224 ? cf.a0[t - 192] : cf.lam[t - 224];
    } else {
      const int q = (t >> 5) % 3, m = t & 31;
      sT[t] = t < 96 ? dd[1 + q] * cf.w0 * cf.lam[m] : t < 192 ? dd[1 + q] * cf.w0 * cf.a0[m]
                                                      : t < 224 ? cf.a0[t - 192] : cf.lam[t - 224];
      if (t < 96) {
        sCg[t] = dd[1 + q] * cf.a0[m];
        sDlg[t] = dd[1 + q] * cf.lam[m];
      }
    }
  }
  auto Cc = [&](int q, int m) -> double { if constexpr (UNI) return cf.c[q][m]; else return sCg[q * 32 + m]; };
  auto Dl = [&](int q, int m) -> double { if constexpr (UNI) return cf.dl[q][m]; else return sDlg[q * 32 + m]; };
  const double F0[3] = {dd[0] * cf.w0 + dd[1] * cf.K00, dd[0] * cf.w0 + dd[2] * cf.K00, dd[0] * cf.w0 + dd[3] * cf.K00};
  const double k0p[3] = {dd[1] * cf.K0p, dd[2] * cf.K0p, dd[3] * cf.K0p};
  const double* const sLt = sT;
  const double* const sEt = sT + 96;
  const double* const sA0t = sT + 192;
  const double* const sLamt = sT + 224;
  __shared__ double sDl1[32];   // d2 Lam_j (lane-divergent)
  if (tid < 32) sDl1[tid] = dd[2] * cf.lam[tid];
  if (tid < 26) {
    bool dr;
    sBase[tid] = entity_base(g, ex, ey, ez, tid, &dr);
    sDir[tid] = dr;
  }
  __syncthreads();
  double* const sh = sm + B::O_SH;
  // ---- a3: the element's shell (Dirichlet entities as 0): faces as 6 contiguous blocks,
  // 8-byte cp.async (all loads of a thread in flight at once)
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const double* src = P.x + sBase[f];
    const bool dr = sDir[f];
#pragma unroll
    for (int r = 0; r < (N2 + NT - 1) / NT; ++r) {
      const int q = tid + r * NT;
      if (q < N2) {
#if defined(SC_EXP) && SC_EXP == 43
        sh[f * N2 + q] = (double)q;   // ablation (timing only): no shell gather of the faces
#else
        if (dr) sh[f * N2 + q] = 0.0;
        else cp_async8b(sh + f * N2 + q, src + q);
#endif
      }
    }
  }
  for (int t = tid; t < 12 * NI + 8; t += NT) {
    int ent, loc;
    if (t < 12 * NI) { const int e = t / NI; ent = 6 + e; loc = t - e * NI; }
    else { ent = 18 + (t - 12 * NI); loc = 0; }
    if (sDir[ent]) sh[6 * N2 + t] = 0.0;
    else cp_async8b(sh + 6 * N2 + t, P.x + sBase[ent] + loc);
  }
  // n_I > 16 (one CTA per SM): the old values of y at this element's outputs (read-modify-write
  // at the end) are loaded now, so their latency overlaps the whole element (no other CTA of
  // this colour touches them).  n_I <= 16 keeps the registers for occupancy (3 CTAs per SM) and
  // loads them in the output phase.
  constexpr bool EARLY = NI > 16;
  constexpr int RF = (N2 + NT - 1) / NT, RE = (12 * NI + 8 + NT - 1) / NT;
  double yold[6][RF], yoldE[RE];
  auto load_yold = [&]() {
#pragma unroll
    for (int f = 0; f < 6; ++f)
#pragma unroll
      for (int r = 0; r < RF; ++r) {
        const int q = tid + r * NT;
#if defined(SC_EXP) && SC_EXP == 44
        yold[f][r] = 0.0;   // ablation (timing only): no read of y before the face stores
#else
        yold[f][r] = (q < N2 && !sDir[f]) ? P.y[sBase[f] + q] : 0.0;
#endif
      }
#pragma unroll
    for (int r = 0; r < RE; ++r) {
      const int t = tid + r * NT;
      yoldE[r] = 0.0;
      if (t < 12 * NI + 8) {
        const int ent = t < 12 * NI ? 6 + t / NI : 18 + (t - 12 * NI);
        if (!sDir[ent]) yoldE[r] = P.y[sBase[ent] + (t < 12 * NI ? t - (ent - 6) * NI : 0)];
      }
    }
  };
  if constexpr (EARLY) {
    load_yold();
  } else {
    // the old values are loaded in the output phase (registers kept for occupancy): prefetch
    // their lines into L2 now, one prefetch per 128 bytes of each face block, one per edge end
    auto pf = [&](long long a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(P.y + a)); };
#pragma unroll
    for (int f = 0; f < 6; ++f)
      if (!sDir[f])
        for (int q = 16 * tid; q < N2 + 15; q += 16 * NT) pf(sBase[f] + (q < N2 ? q : N2 - 1));
    if (tid < 24 && !sDir[6 + (tid >> 1)]) pf(sBase[6 + (tid >> 1)] + ((tid & 1) ? NI - 1 : 0));
    if (tid >= 32 && tid < 40 && !sDir[18 + tid - 32]) pf(sBase[18 + tid - 32]);
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  // ---- faces-in operands P^s = lo + (-1)^s hi, a0-weighted line sums (R+, R-) of faces / edges
  double* const sP = sm + B::O_P;
  double* const sQ = sm + B::O_Q;
  double* const sLS = sm + B::O_LS;
  double* const sES = sm + B::O_ES;
  for (int t = tid; t < 3 * N2; t += NT) {
    const int f = t / N2, q = t - f * N2;
    const double lo = sh[2 * f * N2 + q], hi = sh[(2 * f + 1) * N2 + q];
    sP[2 * f * N2 + q] = lo + hi;
    sP[(2 * f + 1) * N2 + q] = lo - hi;
  }
  for (int t = tid; t < 12 * NI + 12; t += NT) {
    const double* F;
    int st;
    if (t < 12 * NI) {   // (face f, d): d = 0 sums over the first coordinate a at b = c, d = 1 over b at a = c
      const int fd = t / NI, c = t - fd * NI, f = fd >> 1;
      F = (fd & 1) ? sh + f * N2 + c : sh + f * N2 + NI * c;
      st = (fd & 1) ? NI : 1;
    } else {
      F = sh + 6 * N2 + (t - 12 * NI) * NI;
      st = 1;
    }
    double rp = 0.0, rm = 0.0;
#pragma unroll
    for (int a = 0; a < NI; ++a) {
      if (a & 1) rm = fma(cf.a0[a], F[a * st], rm);
      else rp = fma(cf.a0[a], F[a * st], rp);
    }
    double* o = t < 12 * NI ? sLS + 2 * t : sES + 2 * (t - 12 * NI);
    o[0] = rp;
    o[1] = rm;
  }
  __syncthreads();

  // ---- a4-a6: condensed part
  {
    const int j = lane % SW, h = lane / SW, ig = warp * H + h;
    const bool jok = j < NI;
    const int jc = jok ? j : 0;
    const double c2j = jok ? Cc(1, jc) : 0.0;
    const double* Pxs = sP + (ig & 1) * N2;            // Px^{s_i}; s_i = ig & 1 (NG even)
    const double* Pyj = sP + (2 + (j & 1)) * N2;       // Py^{s_j}
    const double* Pz0 = sP + 4 * N2;
    const double* Pz1 = sP + 5 * N2;
    double* const Yb = sm + B::O_Y + (warp * H + h) * NI * YS;
    double qx[NI];
#pragma unroll
    for (int k = 0; k < NI; ++k) qx[k] = 0.0;
#pragma unroll 1
    for (int it = 0; it < B::NIT; ++it) {
      const int i = ig + it * NG;
      const bool iok = i < NI;
      const unsigned am = __ballot_sync(0xffffffffu, iok);
      if (iok) {
        const double c1i = Cc(0, i);
        const double pz0 = Pz0[i + NI * jc], pz1 = Pz1[i + NI * jc];
        const double* Pyi = Pyj + i;
        // D^{-1} = 1 / (d0 + d1 Lam_i + d2 Lam_j + d3 Lam_k) recomputed per point (MUFU
        // approximation + 2 Newton steps, within 1 ulp of the table value: SURVEY c12): with
        // 1-3 CTAs per SM an L2 table load per point stalls the loop (measured 6-12 % slower)
        const double dij = dd[0] + Dl(0, i) + sDl1[jc];
        double qz0 = 0.0, qz1 = 0.0;
        if constexpr (CH > 0) {
          // The k line in chunks of CH points, software-pipelined by hand: the operand loads of
          // chunk c + 1 are issued before the transpose stores of chunk c (all in one dynamic shared
          // array, so the compiler may not move a load above an earlier store: written point by
          // point, the line ran as one serial load -> arithmetic -> store chain).
          const double* const px = Pxs + jc;
          double* const yb = Yb + j;
          double ax[NI], ay[NI], vv[NI];
  #pragma unroll
          for (int k = 0; k < CH && k < NI; ++k) { ax[k] = px[NI * k]; ay[k] = Pyi[NI * k]; }
  #pragma unroll
          for (int c0 = 0; c0 < NI; c0 += CH) {
  #pragma unroll
            for (int k = c0; k < c0 + CH && k < NI; ++k) {
              const double u = fma(c1i, ax[k], fma(c2j, ay[k], Cc(2, k) * ((k & 1) ? pz1 : pz0)));
              const double D = dij + Dl(2, k);
              double r;
              asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(D));
              double e = fma(-D, r, 1.0);
              r = fma(r, e, r);
              e = fma(-D, r, 1.0);
              const double dinv = fma(r, e, r);
              const double v = u * dinv;
              vv[k] = v;
              qx[k] = fma(c1i, v, qx[k]);
              if (k & 1) qz1 = fma(Cc(2, k), v, qz1);
              else qz0 = fma(Cc(2, k), v, qz0);
            }
  #pragma unroll
            for (int k = c0 + CH; k < c0 + 2 * CH && k < NI; ++k) { ax[k] = px[NI * k]; ay[k] = Pyi[NI * k]; }
  #pragma unroll
            for (int k = c0; k < c0 + CH && k < NI; ++k) yb[k * YS] = c2j * vv[k];
          }
        } else {
          // point by point (CH = 0): fewer registers; chosen where the pipelined form would cost
          // a CTA per SM (launch_big_t)
#pragma unroll
          for (int k = 0; k < NI; ++k) {
            const double u = fma(c1i, Pxs[jc + NI * k], fma(c2j, Pyi[NI * k], Cc(2, k) * ((k & 1) ? pz1 : pz0)));
            const double D = dij + Dl(2, k);
            double r;
            asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(D));
            double e = fma(-D, r, 1.0);
            r = fma(r, e, r);
            e = fma(-D, r, 1.0);
            const double dinv = fma(r, e, r);
            const double v = u * dinv;
            qx[k] = fma(c1i, v, qx[k]);
            Yb[k * YS + j] = c2j * v;
            if (k & 1) qz1 = fma(Cc(2, k), v, qz1);
            else qz0 = fma(Cc(2, k), v, qz0);
          }
        }
        if (jok) {
          sQ[4 * N2 + i + NI * j] = qz0;
          sQ[5 * N2 + i + NI * j] = qz1;
        }
        __syncwarp(am);
        // Qy^s(i, k) = sum over j of parity s: one (k, s) pair per lane and pass
        for (int pr = j; pr < 2 * NI; pr += SW) {
          const int k = pr >> 1, s = pr & 1;
          const double* yr = Yb + k * YS + s;
          double a0s = 0.0, a1s = 0.0;
#pragma unroll
          for (int jj = 0; jj < NI; jj += 4) {
            if (jj + s < NI) a0s += yr[jj];
            if (jj + 2 + s < NI) a1s += yr[jj + 2];
          }
          sQ[(2 + s) * N2 + i + NI * k] = a0s + a1s;
        }
        __syncwarp(am);
      }
    }
    // Qx: fixed-order tree over the warps holding the same parity of i (H == 1: warp parity;
    // H == 2: the half), through the (now free) transpose buffers
    constexpr int STMIN = H == 1 ? 2 : 1;
    double* const slots = sm + B::O_Y;
    if constexpr (H == 2) {
      // any NW: the upper ceil half of the remaining warps hands its sums to the lower half
#pragma unroll
      for (int n = NW; n > 1; n = (n + 1) >> 1) {
        const int half = (n + 1) >> 1;
        __syncthreads();
        if (warp >= half && warp < n) {
          double* sl = slots + ((warp - half) * H + h) * NI * SW + j;
#pragma unroll
          for (int k = 0; k < NI; ++k) sl[k * SW] = qx[k];
        }
        __syncthreads();
        if (warp < n - half) {
          const double* sl = slots + (warp * H + h) * NI * SW + j;
#pragma unroll
          for (int k = 0; k < NI; ++k) qx[k] += sl[k * SW];
        }
      }
    } else {
#pragma unroll 1
      for (int st = NW / 2; st >= STMIN; st >>= 1) {
        __syncthreads();
        if (warp >= st && warp < 2 * st) {
          double* sl = slots + ((warp - st) * H + h) * NI * SW + j;
#pragma unroll
          for (int k = 0; k < NI; ++k) sl[k * SW] = qx[k];
        }
        __syncthreads();
        if (warp < st) {
          const double* sl = slots + (warp * H + h) * NI * SW + j;
#pragma unroll
          for (int k = 0; k < NI; ++k) qx[k] += sl[k * SW];
        }
      }
    }
    if (warp < STMIN && jok) {
      double* Qx = sQ + (H == 1 ? warp : h) * N2 + j;
#pragma unroll
      for (int k = 0; k < NI; ++k) Qx[NI * k] = qx[k];
    }
  }
  __syncthreads();

  // ---- a6 + a7 + a8: outputs (primary - condensed part on faces, primary on edges / vertices),
  // read-modify-write into y (each face / edge / vertex of this element is written by this CTA only
  // within the colour's launch)
  const double* const Ed = sh + 6 * N2;
  const double* const Vv = Ed + 12 * NI;
  const double K00 = cf.K00, K0p = cf.K0p, w0 = cf.w0, w02 = w0 * w0;
  if constexpr (!EARLY) load_yold();
  // faces: f = 2 d + hi; coordinates (a, b) of directions (la, lb); bounding edges (local id - 6)
  // ea0 / ea1 at index b (coefficient e[la][a], sign of a), eb0 / eb1 at index a (e[lb][b], sign of b)
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    constexpr int EA0[6] = {8, 9, 8, 10, 4, 6}, EA1[6] = {10, 11, 9, 11, 5, 7};
    constexpr int EB0[6] = {4, 5, 0, 1, 0, 2}, EB1[6] = {6, 7, 2, 3, 1, 3};
    const int d = f >> 1, hi = f & 1, la = d == 0 ? 1 : 0, lb = d == 2 ? 1 : 2;
    if (sDir[f]) continue;
    double* const yf = P.y + sBase[f];
    constexpr int R = RF;
    double val[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = min(tid + r * NT, N2 - 1), b = q / NI, a = q - b * NI;
      const double fd = F0[d] + sLt[la * 32 + a] + sLt[lb * 32 + b];
      const double self = sh[f * N2 + q], opp = sh[(f ^ 1) * N2 + q];
      const double ta = sEt[la * 32 + a] * fma(sgn(a), Ed[EA1[f] * NI + b], Ed[EA0[f] * NI + b]);
      const double tb = sEt[lb * 32 + b] * fma(sgn(b), Ed[EB1[f] * NI + a], Ed[EB0[f] * NI + a]);
      const double Q = fma(hi ? -1.0 : 1.0, sQ[(2 * d + 1) * N2 + q], sQ[2 * d * N2 + q]);
      val[r] = fma(fd, self, fma(k0p[d], opp, ta + tb)) - Q;
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int q = tid + r * NT;
      if (q < N2) yf[q] = yold[f][r] + val[r];
    }
  }
  // edges (one thread per edge node) and vertices
#pragma unroll
  for (int rr = 0; rr < RE; ++rr) {
    const int t = tid + rr * NT;
    if (t >= 12 * NI + 8) continue;
    const int ent = t < 12 * NI ? 6 + t / NI : 18 + (t - 12 * NI);
    if (sDir[ent]) continue;
    double* const dst = P.y + sBase[ent] + (t < 12 * NI ? t - (ent - 6) * NI : 0);
    const double old = yoldE[rr];
    double val;
    if (t < 12 * NI) {
      const int e = ent - 6, c = t - e * NI, grp = e >> 2, b0 = e & 1, b1 = (e >> 1) & 1;
      const double uu = Ed[e * NI + c];
      // along the edge (interior row of Ktilde): the two end vertices; boundary directions o1 (bit
      // b0) and o2 (bit b1): the parallel edges and the face line sums of Ktilde rows 0 / p
      int v0, v1, p10, p11, l1, p20, p21, l2;
      if (grp == 0) {          // x-edge (jb, kb) = (b0, b1)
        v0 = 2 * b0 + 4 * b1; v1 = v0 + 1;
        p10 = 2 * b1; p11 = 2 * b1 + 1; l1 = ((4 + b1) * 2 + 1) * NI + c;     // o1 = y: z-face b1, sum over j
        p20 = b0; p21 = b0 + 2; l2 = ((2 + b0) * 2 + 1) * NI + c;             // o2 = z: y-face b0, sum over k
      } else if (grp == 1) {   // y-edge (ib, kb) = (b0, b1)
        v0 = b0 + 4 * b1; v1 = v0 + 2;
        p10 = 4 + 2 * b1; p11 = 5 + 2 * b1; l1 = ((4 + b1) * 2 + 0) * NI + c;  // o1 = x: z-face b1, sum over i
        p20 = 4 + b0; p21 = 6 + b0; l2 = (b0 * 2 + 1) * NI + c;                // o2 = z: x-face b0, sum over k
      } else {                 // z-edge (ib, jb) = (b0, b1)
        v0 = b0 + 2 * b1; v1 = v0 + 4;
        p10 = 8 + 2 * b1; p11 = 9 + 2 * b1; l1 = ((2 + b1) * 2 + 0) * NI + c;  // o1 = x: y-face b1, sum over i
        p20 = 8 + b0; p21 = 10 + b0; l2 = (b0 * 2 + 0) * NI + c;               // o2 = y: x-face b0, sum over j
      }
      const double tal = sA0t[c] * fma(sgn(c), Vv[v1], Vv[v0]) + sLamt[c] * uu;
      const double u10 = Ed[p10 * NI + c], u11 = Ed[p11 * NI + c], u20 = Ed[p20 * NI + c], u21 = Ed[p21 * NI + c];
      const double t1 = (b0 ? fma(K0p, u10, K00 * u11) : fma(K00, u10, K0p * u11)) + eo_row_b(sLS + 2 * l1, b0);
      const double t2 = (b1 ? fma(K0p, u20, K00 * u21) : fma(K00, u20, K0p * u21)) + eo_row_b(sLS + 2 * l2, b1);
      const int o1 = grp == 0 ? 1 : 0, o2 = grp == 2 ? 1 : 2;
      auto dsel = [&](int q) { return q == 0 ? dd[1] : (q == 1 ? dd[2] : dd[3]); };   // no local-memory indexing
      val = w02 * (dd[0] * uu + dsel(grp) * tal) + w0 * (dsel(o1) * t1 + dsel(o2) * t2);
    } else {
      const int v = t - 12 * NI, ib = v & 1, jb = (v >> 1) & 1, kb = v >> 2;
      const double uu = Vv[v];
      // partner vertices along x / y / z: (lo, hi) of the pair containing v.  (Written with
      // arithmetic offsets: an earlier bitwise form, Vv[v | 4] / Vv[v & ~4], gave wrong vertex
      // values in some builds -- not root-caused; the parity tests pin this.)
      const int xl = v - ib, yl = v - 2 * jb, zl = v - 4 * kb;
      const double x0v = Vv[xl], x1v = Vv[xl + 1], y0v = Vv[yl], y1v = Vv[yl + 2], z0v = Vv[zl], z1v = Vv[zl + 4];
      const double tx = (ib ? fma(K0p, x0v, K00 * x1v) : fma(K00, x0v, K0p * x1v)) + eo_row_b(sES + 2 * (jb + 2 * kb), ib);
      const double ty = (jb ? fma(K0p, y0v, K00 * y1v) : fma(K00, y0v, K0p * y1v)) + eo_row_b(sES + 2 * (4 + ib + 2 * kb), jb);
      const double tz = (kb ? fma(K0p, z0v, K00 * z1v) : fma(K00, z0v, K0p * z1v)) + eo_row_b(sES + 2 * (8 + ib + 2 * jb), kb);
      val = w02 * (w0 * dd[0] * uu + dd[1] * tx + dd[2] * ty + dd[3] * tz);
    }
    *dst = old + val;
  }
}

// Two builds of every kernel: the k line point by point (CH = 0) or software-pipelined in
// chunks of 2 (CH = 2, more registers).  The pipelined one is used unless its register count
// costs resident CTAs per SM (measured: p = 9 2.61 -> 2.42 ms, p = 16 1.08 -> 1.02, p = 20
// 1.38 -> 1.17, p = 24 1.11 -> 0.94, p = 32 0.91 -> 0.86; p = 12 keeps CH = 0: 4 instead of 5
// CTAs per SM would make it 9 % slower).
template <int NI, bool UNI, int CH>
static int occupancy_big(size_t smem) {
  cudaFuncSetAttribute(k_apply_big<NI, UNI, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_apply_big<NI, UNI, CH>, BL<NI>::NT, smem) != cudaSuccess)
    return 0;
  return nb;
}

template <int NI, bool UNI>
static int launch_big_t(const BigParams& P, cudaStream_t st, int* nl) {
  using B = BL<NI>;
  static_assert(sizeof(double) * B::TOTAL <= 225 * 1024, "shared memory budget");
  const size_t smem = sizeof(double) * B::TOTAL;
  static int auto_pipe_d[kMaxDev];   // per device: 0 = not queried, else 1 + choice
  // (the occupancy queries also set both builds' shared-memory limit on this device)
  const int dv = dev_slot();
  if (!auto_pipe_d[dv]) auto_pipe_d[dv] = 1 + (occupancy_big<NI, UNI, 2>(smem) >= occupancy_big<NI, UNI, 0>(smem) ? 1 : 0);
  const int auto_pipe = auto_pipe_d[dv] - 1;
  const char* force = getenv("SC_V4_PIPE");   // tests: 0 / 1 force a build (same arithmetic, same order)
  const int pipelined = (force && (force[0] == '0' || force[0] == '1')) ? force[0] - '0' : auto_pipe;
  for (int c = 0; c < 8; ++c) {
    const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
    const long long n = (long long)((P.g.nx - cx + 1) >> 1) * ((P.g.ny - cy + 1) >> 1) * ((P.g.nz - cz + 1) >> 1);
    if (n <= 0) continue;
    if (pipelined) k_apply_big<NI, UNI, 2><<<(unsigned)n, B::NT, smem, st>>>(P, c);
    else k_apply_big<NI, UNI, 0><<<(unsigned)n, B::NT, smem, st>>>(P, c);
    (*nl)++;
  }
  return cudaGetLastError();
}

bool big_supported(int ni) { return ni >= 8 && ni <= 31; }

int launch_apply_big(const Geom& g, const double* x, double* y, const double* done, const void* coef, void* stream,
                     int* nl, void* events) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  cudaError_t err = cudaMemsetAsync(y, 0, sizeof(double) * g.n_total, st);
  if (err != cudaSuccess) return err;
  if (ev) cudaEventRecord(ev[0], st);
  BigParams P;
  P.g = g; P.x = x; P.y = y; P.done = done;
  memcpy(&P.cf, coef, sizeof(BigCoef));
  int rc = cudaErrorInvalidValue;
  switch (g.ni) {
#define BCASE(N) case N: rc = g.uniform ? launch_big_t<N, true>(P, st, nl) : launch_big_t<N, false>(P, st, nl); break;
    BCASE(8) BCASE(9) BCASE(10) BCASE(11) BCASE(12) BCASE(13) BCASE(14) BCASE(15) BCASE(16) BCASE(17)
    BCASE(18) BCASE(19) BCASE(20) BCASE(21) BCASE(22) BCASE(23) BCASE(24) BCASE(25) BCASE(26) BCASE(27)
    BCASE(28) BCASE(29) BCASE(30) BCASE(31)
#undef BCASE
    default: break;
  }
  if (ev) cudaEventRecord(ev[1], st);
  return rc;
}

// Host-side coefficient block of the v4 operator (uniform geometry d).
void big_make_coef(int ni, const double* d, const double* a0, const double* lam, double K00, double K0p, double w0,
                   std::vector<unsigned char>& coef) {
  BigCoef cf;
  memset(&cf, 0, sizeof(cf));
  for (int q = 0; q < 3; ++q)
    for (int m = 0; m < ni; ++m) {
      cf.c[q][m] = d[1 + q] * a0[m];
      cf.e[q][m] = d[1 + q] * w0 * a0[m];
      cf.L[q][m] = d[1 + q] * w0 * lam[m];
      cf.dl[q][m] = d[1 + q] * lam[m];
    }
  for (int m = 0; m < ni; ++m) { cf.a0[m] = a0[m]; cf.lam[m] = lam[m]; }
  for (int q = 0; q < 3; ++q) {
    cf.F0[q] = d[0] * w0 + d[1 + q] * K00;
    cf.k0p[q] = d[1 + q] * K0p;
  }
  for (int q = 0; q < 4; ++q) cf.d[q] = d[q];
  cf.K00 = K00; cf.K0p = K0p; cf.w0 = w0;
  coef.resize(sizeof(BigCoef));
  memcpy(coef.data(), &cf, sizeof(BigCoef));
}

}  // namespace sc
