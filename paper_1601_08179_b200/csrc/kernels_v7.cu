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

// 8-byte global -> shared copy, zero fill when !ok (src-size 0)
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}

// ------------------------------------------------------------------------------------ pass A
template <int NI>
__global__ void __launch_bounds__(128, 4) k_v7_cond(const __grid_constant__ V7Params P) {
  if (P.done != nullptr && *P.done != 0.0) return;
  constexpr int N2 = NI * NI, M = (NI + 1) / 2;
  constexpr int PJ = NI + 1, PK = NI + 1;   // padded D^{-1} table strides (k: see the bank note below)
  const Geom& g = P.g;
  const V7Coef& cf = P.cf;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const int run = blockIdx.x, ey = blockIdx.y, ez = blockIdx.z;
  const int ex0 = run * RUN;
  const int cnt = min(RUN, nx - ex0);
  __shared__ double sX[(RUN + 1) * N2];
  __shared__ double sY[2][RUN * N2];
  __shared__ double sZ[2][RUN * N2];
  // D^{-1} at i + PJ j + PKK k with the 8 class bases on distinct bank pairs (cf. kernels_v6.cu di_pk)
  constexpr int PKK = di_pk(PJ, PK);
  __shared__ double sD[PKK * PK + 2];
  __shared__ double sC[3][8];
  const int tid = threadIdx.x;
  for (int t = tid; t < PKK * PK + 2; t += 128) {
    const int k = t / PKK, r = t - k * PKK, j = r / PJ, i = r - j * PJ;
    sD[t] = (i < NI && j < NI && k < NI) ? cf.dinv[i + NI * (j + NI * k)] : 0.0;
  }
  if (tid < 24) sC[tid / 8][tid % 8] = (tid % 8) < NI ? cf.c[tid / 8][tid % 8] : 0.0;
  // faces of the run (Dirichlet faces and faces beyond the slab read as 0)
  {   // asynchronous 8-byte copies (cp.async, zero-filled where masked): all of a thread's loads in flight
    const long long xb = g.off_f[0] + ((long long)ex0 + (long long)(nx + 1) * (ey + (long long)ny * ez)) * N2;
    for (int t = tid; t < (RUN + 1) * N2; t += 128) {
      const int fx = ex0 + t / N2;
      const bool ok = t < (cnt + 1) * N2 && fx > 0 && fx < nx;
      cp_async8(sX + t, P.x + (ok ? xb + t : 0), ok);
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int fy = ey + s;
      const bool fok = fy > 0 && fy < ny;
      const long long yb = g.off_f[1] + ((long long)ex0 + (long long)nx * (fy + (long long)(ny + 1) * ez)) * N2;
      const int fz = ez + s;
      const bool zok = !zdir(g, fz);
      const long long zb = g.off_f[2] + ((long long)ex0 + (long long)nx * (ey + (long long)ny * fz)) * N2;
      for (int t = tid; t < RUN * N2; t += 128) {
        const bool in = t < cnt * N2;
        cp_async8(sY[s] + t, P.x + ((in && fok) ? yb + t : 0), in && fok);
        cp_async8(sZ[s] + t, P.x + ((in && zok) ? zb + t : 0), in && zok);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  const int el = warp * 4 + (lane >> 3);          // element of the run
  const int cls = lane & 7, si = cls >> 2, sj = (cls >> 1) & 1, sk = cls & 1;
  const int CI = (NI - si + 1) >> 1, CJ = (NI - sj + 1) >> 1, CK = (NI - sk + 1) >> 1;
  const double gi = si ? -1.0 : 1.0, gj = sj ? -1.0 : 1.0, gk = sk ? -1.0 : 1.0;
  const bool act = el < cnt;
  const double* W = sX + el * N2 + sj + NI * sk;      // x-face entries (j, k)
  const double* E = W + N2;
  const double* S = sY[0] + el * N2 + si + NI * sk;   // y-face entries (i, k)
  const double* Nn = sY[1] + el * N2 + si + NI * sk;
  const double* B = sZ[0] + el * N2 + si + NI * sj;   // z-face entries (i, j)
  const double* T = sZ[1] + el * N2 + si + NI * sj;
  const double* Dc = sD + si + PJ * sj + PKK * sk;
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
  const long long ex = ex0 + el;
  // output rows (entries of the element's faces in U0 / U1), written straight from the lanes (staging
  // them in shared memory for row-wise stores measured slower: 11.0 -> 12.0 ms at cfg5)
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
#pragma unroll
    for (int jj = 0; jj < M; ++jj) {
      const double c2 = sC[1][sj + 2 * jj];
      const int ox = 2 * jj + 2 * NI * kk;
      const double xin = (jj < CJ && kk < CK) ? fma(gi, E[ox], W[ox]) : 0.0;
      double qx = 0.0;
#pragma unroll
      for (int ii = 0; ii < M; ++ii) {
        const double u = fma(c1[ii], xin, fma(c2, yin[ii], c3 * zin[ii][jj]));
        const double v = u * Dc[2 * ii + 2 * PJ * jj + 2 * PKK * kk];
        qx = fma(c1[ii], v, qx);
        qy[ii] = fma(c2, v, qy[ii]);
        qz[ii][jj] = fma(c3, v, qz[ii][jj]);
      }
      // x pair (s_i = 0 / 1: lane ^ 4): W part -(Q0 + Q1) (s_i = 0 lane), E part -(Q0 - Q1) (s_i = 1 lane)
      const double qp = __shfl_xor_sync(0xffffffffu, qx, 4);
      if (act && jj < CJ && kk < CK) {
        if (si == 0) uxw[sj + 2 * jj + NI * (sk + 2 * kk)] = -(qx + qp);
        else uxe[sj + 2 * jj + NI * (sk + 2 * kk)] = qx - qp;
      }
    }
#pragma unroll
    for (int ii = 0; ii < M; ++ii) {   // y pair (lane ^ 2): S -(Q0 + Q1), N -(Q0 - Q1)
      const double qp = __shfl_xor_sync(0xffffffffu, qy[ii], 2);
      if (act && ii < CI && kk < CK) {
        if (sj == 0) uys[si + 2 * ii + NI * (sk + 2 * kk)] = -(qy[ii] + qp);
        else uyn[si + 2 * ii + NI * (sk + 2 * kk)] = qy[ii] - qp;
      }
    }
  }
#pragma unroll
  for (int ii = 0; ii < M; ++ii)   // z pair (lane ^ 1): B -(Q0 + Q1), T -(Q0 - Q1)
#pragma unroll
    for (int jj = 0; jj < M; ++jj) {
      const double qp = __shfl_xor_sync(0xffffffffu, qz[ii][jj], 1);
      if (act && ii < CI && jj < CJ) {
        if (sk == 0) uzb[si + 2 * ii + NI * (sj + 2 * jj)] = -(qz[ii][jj] + qp);
        else uzt[si + 2 * ii + NI * (sj + 2 * jj)] = qz[ii][jj] - qp;
      }
    }
}

// ------------------------------------------------------------------------------------ pass B
// One thread per skeleton entry of class `cls` (0..2 x / y / z faces, 3..5 x / y / z edges, 6
// vertices); blockIdx.y = entity row (the slow indices), threadIdx / blockIdx.x run over the row's
// contiguous entries.
// Free (non-Dirichlet, inside the slab) lattice test for an entity given by its three grid indices
// and which of them are "face" (f) indices.
__device__ __forceinline__ bool in_f(int v, int n) { return v > 0 && v < n; }
__device__ __forceinline__ bool in_e(int v, int n) { return v >= 0 && v < n; }

template <int NI>
__device__ __forceinline__ double ldv(const double* __restrict__ x, long long i, bool ok) {
  const double v = __ldg(x + (ok ? i : 0));   // always a valid address: the load is not predicated
  return ok ? v : 0.0;
}

template <int NI, bool DOT>
__global__ void __launch_bounds__(256) k_v7_assemble(const __grid_constant__ V7Params P, int cls) {
  if (P.done != nullptr && *P.done != 0.0) return;
  constexpr int N2 = NI * NI;
  const Geom& g = P.g;
  const V7Coef& cf = P.cf;
  const int nx = g.nx, ny = g.ny, nz = g.nz;
  const long long nx1 = nx + 1, ny1 = ny + 1;
  const double* __restrict__ x = P.x;
  const int row = blockIdx.y;   // y-ish index + (count) * z-ish index
  double dot = 0.0;
  // lane-indexed coefficients from shared memory (indexed kernel-parameter loads serialise per address)
  __shared__ double sfd[49], sa0[8], sap[8], sself[8];
  {
    const int f = cls <= 2 ? cls : 0, e = cls >= 3 && cls <= 5 ? cls - 3 : 0;
    for (int q = threadIdx.x; q < N2; q += blockDim.x) sfd[q] = cf.fd[f][q];
    if (threadIdx.x < 8) {
      sa0[threadIdx.x] = cf.a0[threadIdx.x];
      sap[threadIdx.x] = cf.ap[threadIdx.x];
      sself[threadIdx.x] = cf.eself[e][threadIdx.x];
    }
    __syncthreads();
  }
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  // all rows are (x-run of entities) x (per-entity entries); decode (a = x index, e = entry)
  if (cls <= 2) {
    // ---------------- faces: one thread per (face, first in-plane entry ea), loop over the second (eb).
    // y(ea, eb) = fd u + K0p-term (opposite faces) + wA (a0_ea A0[eb] + ap_ea A1[eb]) + wB (a0_eb B0[ea] + ap_eb B1[ea])
    //             + U0 + U1;  A = the edges along the second in-plane direction, B = along the first.
    const int a = t / NI, ea = t - a * NI;
    const int rowlen = cls == 0 ? nx + 1 : nx;
    if (a < rowlen) {
      long long fid, so, ia0, ia1, ib0, ib1;
      bool fr, olo, ohi, oka0, oka1, okb0, okb1;
      double wA, wB, kf;
      if (cls == 0) {            // x-face (fx, ey, ez): A = z-edges (fx, ey / ey+1, ez), B = y-edges (fx, ey, ez / ez+1)
        const int ey_ = row % ny, ez_ = row / ny, fx = a;
        fid = fx + nx1 * (ey_ + (long long)ny * ez_);
        fr = in_f(fx, nx);
        so = N2; olo = fx - 1 > 0; ohi = fx + 1 < nx;
        ia0 = g.off_e[2] + (fx + nx1 * (ey_ + ny1 * ez_)) * NI; ia1 = ia0 + nx1 * NI;
        oka0 = in_f(ey_, ny); oka1 = in_f(ey_ + 1, ny);
        ib0 = g.off_e[1] + (fx + nx1 * (ey_ + (long long)ny * ez_)) * NI + ea; ib1 = ib0 + nx1 * ny * NI;
        okb0 = !zdir(g, ez_); okb1 = !zdir(g, ez_ + 1);
        wA = cf.ef[0][1]; wB = cf.ef[0][2]; kf = cf.kf[0];
      } else if (cls == 1) {     // y-face (ex, fy, ez): A = z-edges (ex / ex+1, fy, ez), B = x-edges (ex, fy, ez / ez+1)
        const int fy = row % (ny + 1), ez_ = row / (ny + 1), ex_ = a;
        fid = ex_ + (long long)nx * (fy + ny1 * ez_);
        fr = in_f(fy, ny);
        so = (long long)nx * N2; olo = fy - 1 > 0; ohi = fy + 1 < ny;
        ia0 = g.off_e[2] + (ex_ + nx1 * (fy + ny1 * ez_)) * NI; ia1 = ia0 + NI;
        oka0 = in_f(ex_, nx); oka1 = in_f(ex_ + 1, nx);
        ib0 = g.off_e[0] + (ex_ + (long long)nx * (fy + ny1 * ez_)) * NI + ea; ib1 = ib0 + (long long)nx * ny1 * NI;
        okb0 = !zdir(g, ez_); okb1 = !zdir(g, ez_ + 1);
        wA = cf.ef[1][0]; wB = cf.ef[1][2]; kf = cf.kf[1];
      } else {                   // z-face (ex, ey, fz): A = y-edges (ex / ex+1, ey, fz), B = x-edges (ex, ey / ey+1, fz)
        const int ey_ = row % ny, fz = row / ny, ex_ = a;
        fid = ex_ + (long long)nx * (ey_ + (long long)ny * fz);
        fr = !zdir(g, fz);
        so = (long long)nx * ny * N2; olo = fz - 1 >= 0 && !zdir(g, fz - 1); ohi = fz + 1 <= nz && !zdir(g, fz + 1);
        ia0 = g.off_e[1] + (ex_ + nx1 * (ey_ + (long long)ny * fz)) * NI; ia1 = ia0 + NI;
        oka0 = in_f(ex_, nx); oka1 = in_f(ex_ + 1, nx);
        ib0 = g.off_e[0] + (ex_ + (long long)nx * (ey_ + ny1 * fz)) * NI + ea; ib1 = ib0 + (long long)nx * NI;
        okb0 = in_f(ey_, ny); okb1 = in_f(ey_ + 1, ny);
        wA = cf.ef[2][0]; wB = cf.ef[2][1]; kf = cf.kf[2];
      }
      const long long i0 = g.off_f[cls] + fid * N2 + ea;
      if (fr) {
        const double b0 = ldv<NI>(x, ib0, okb0), b1 = ldv<NI>(x, ib1, okb1);
        const double a0e = sa0[ea], ape = sap[ea];
#pragma unroll
        for (int eb = 0; eb < NI; ++eb) {
          const long long i = i0 + NI * eb;
          const double u = __ldg(x + i);
          const double uo = ldv<NI>(x, i - so, olo) + ldv<NI>(x, i + so, ohi);
          const double ea_ = a0e * ldv<NI>(x, ia0 + eb, oka0) + ape * ldv<NI>(x, ia1 + eb, oka1);
          const double eb_ = sa0[eb] * b0 + sap[eb] * b1;
          const double yv = sfd[ea + NI * eb] * u + kf * uo + wA * ea_ + wB * eb_ + P.u0[i] + P.u1[i];
          if (DOT) dot = fma(u, yv, dot);
          P.y[i] = yv;
        }
      } else {
#pragma unroll
        for (int eb = 0; eb < NI; ++eb) P.y[i0 + NI * eb] = 0.0;
      }
    }
  } else if (cls <= 5) {
    // ---------------- edges (entry m along the edge)
    const int a = t / NI, m = t - a * NI;
    const int dir = cls - 3;
    const int rowlen = dir == 0 ? nx : nx + 1;
    if (a < rowlen) {
      long long i0;
      bool fr;
      double yv = 0.0;
      if (dir == 0) {   // x-edge (ex, fy, fz): lines in z-faces (ex, fy-1 / fy, fz) over j, y-faces (ex, fy, fz-1 / fz) over k
        const int fy = row % (ny + 1), fz = row / (ny + 1), ex_ = a;
        i0 = g.off_e[0] + (ex_ + (long long)nx * (fy + ny1 * fz)) * NI + m;
        fr = in_f(fy, ny) && !zdir(g, fz);
        if (fr) {
          const double u = __ldg(x + i0);
          const double vw = ldv<NI>(x, g.off_v + ex_ + nx1 * (fy + ny1 * fz), in_f(ex_, nx));
          const double ve = ldv<NI>(x, g.off_v + ex_ + 1 + nx1 * (fy + ny1 * fz), in_f(ex_ + 1, nx));
          const long long zlo = g.off_f[2] + (ex_ + (long long)nx * (fy - 1 + (long long)ny * fz)) * N2 + m;   // entries (i = m, j)
          const long long zhi = zlo + (long long)nx * N2;
          const long long ylo = g.off_f[1] + (ex_ + (long long)nx * (fy + ny1 * (fz - 1))) * N2 + m;         // entries (i = m, k)
          const long long yhi = ylo + (long long)nx * ny1 * N2;
          const bool zf_ok = !zdir(g, fz);
          double lz = 0.0, ly = 0.0;
#pragma unroll
          for (int q = 0; q < NI; ++q) {
            lz = fma(cf.ap[q], zf_ok ? __ldg(x + zlo + NI * q) : 0.0, fma(cf.a0[q], zf_ok ? __ldg(x + zhi + NI * q) : 0.0, lz));
            ly = fma(cf.ap[q], __ldg(x + ylo + NI * q), fma(cf.a0[q], __ldg(x + yhi + NI * q), ly));
          }
          const double nb_y = ldv<NI>(x, i0 - (long long)nx * NI, fy - 1 > 0) + ldv<NI>(x, i0 + (long long)nx * NI, fy + 1 < ny);
          const long long pl = (long long)nx * ny1 * NI;
          const double nb_z = ldv<NI>(x, i0 - pl, fz - 1 >= 0 && !zdir(g, fz - 1)) + ldv<NI>(x, i0 + pl, fz + 1 <= nz && !zdir(g, fz + 1));
          yv = sself[m] * u + cf.ev[0] * (sa0[m] * vw + sap[m] * ve) + cf.el[0][1] * fma(cf.K0p, nb_y, lz) +
               cf.el[0][2] * fma(cf.K0p, nb_z, ly);
          if (DOT) dot = u * yv;
        }
      } else if (dir == 1) {   // y-edge (fx, ey, fz): lines in z-faces (fx-1 / fx, ey, fz) over i, x-faces (fx, ey, fz-1 / fz) over k
        const int ey_ = row % ny, fz = row / ny, fx = a;
        i0 = g.off_e[1] + (fx + nx1 * (ey_ + (long long)ny * fz)) * NI + m;
        fr = in_f(fx, nx) && !zdir(g, fz);
        if (fr) {
          const double u = __ldg(x + i0);
          const double vs = ldv<NI>(x, g.off_v + fx + nx1 * (ey_ + ny1 * fz), in_f(ey_, ny));
          const double vn = ldv<NI>(x, g.off_v + fx + nx1 * (ey_ + 1 + ny1 * fz), in_f(ey_ + 1, ny));
          const long long zlo = g.off_f[2] + (fx - 1 + (long long)nx * (ey_ + (long long)ny * fz)) * N2 + NI * m;  // entries (i, j = m)
          const long long zhi = zlo + N2;
          const long long xlo = g.off_f[0] + (fx + nx1 * (ey_ + (long long)ny * (fz - 1))) * N2 + m;        // entries (j = m, k)
          const long long xhi = xlo + nx1 * ny * N2;
          double lz = 0.0, lx = 0.0;
#pragma unroll
          for (int q = 0; q < NI; ++q) {
            lz = fma(cf.ap[q], __ldg(x + zlo + q), fma(cf.a0[q], __ldg(x + zhi + q), lz));
            lx = fma(cf.ap[q], __ldg(x + xlo + NI * q), fma(cf.a0[q], __ldg(x + xhi + NI * q), lx));
          }
          const double nb_x = ldv<NI>(x, i0 - NI, fx - 1 > 0) + ldv<NI>(x, i0 + NI, fx + 1 < nx);
          const long long pl = nx1 * ny * NI;
          const double nb_z = ldv<NI>(x, i0 - pl, fz - 1 >= 0 && !zdir(g, fz - 1)) + ldv<NI>(x, i0 + pl, fz + 1 <= nz && !zdir(g, fz + 1));
          yv = sself[m] * u + cf.ev[1] * (sa0[m] * vs + sap[m] * vn) + cf.el[1][0] * fma(cf.K0p, nb_x, lz) +
               cf.el[1][2] * fma(cf.K0p, nb_z, lx);
          if (DOT) dot = u * yv;
        }
      } else {   // z-edge (fx, fy, ez): lines in y-faces (fx-1 / fx, fy, ez) over i, x-faces (fx, fy-1 / fy, ez) over j
        const int fy = row % (ny + 1), ez_ = row / (ny + 1), fx = a;
        i0 = g.off_e[2] + (fx + nx1 * (fy + ny1 * ez_)) * NI + m;
        fr = in_f(fx, nx) && in_f(fy, ny);
        if (fr) {
          const double u = __ldg(x + i0);
          const double vb = ldv<NI>(x, g.off_v + fx + nx1 * (fy + ny1 * ez_), !zdir(g, ez_));
          const double vt = ldv<NI>(x, g.off_v + fx + nx1 * (fy + ny1 * (ez_ + 1)), !zdir(g, ez_ + 1));
          const long long ylo = g.off_f[1] + (fx - 1 + (long long)nx * (fy + ny1 * ez_)) * N2 + NI * m;   // entries (i, k = m)
          const long long yhi = ylo + N2;
          const long long xlo = g.off_f[0] + (fx + nx1 * (fy - 1 + (long long)ny * ez_)) * N2 + NI * m;   // entries (j, k = m)
          const long long xhi = xlo + nx1 * N2;
          double ly = 0.0, lx = 0.0;
#pragma unroll
          for (int q = 0; q < NI; ++q) {
            ly = fma(cf.ap[q], __ldg(x + ylo + q), fma(cf.a0[q], __ldg(x + yhi + q), ly));
            lx = fma(cf.ap[q], __ldg(x + xlo + q), fma(cf.a0[q], __ldg(x + xhi + q), lx));
          }
          const double nb_x = ldv<NI>(x, i0 - NI, fx - 1 > 0) + ldv<NI>(x, i0 + NI, fx + 1 < nx);
          const double nb_y = ldv<NI>(x, i0 - nx1 * NI, fy - 1 > 0) + ldv<NI>(x, i0 + nx1 * NI, fy + 1 < ny);
          yv = sself[m] * u + cf.ev[2] * (sa0[m] * vb + sap[m] * vt) + cf.el[2][0] * fma(cf.K0p, nb_x, ly) +
               cf.el[2][1] * fma(cf.K0p, nb_y, lx);
          if (DOT) dot = u * yv;
        }
      }
      P.y[i0] = yv;
    }
  } else {
    // ---------------- vertices (fx, fy, fz): lines along the 6 incident edges
    const int fx = t, fy = row % (ny + 1), fz = row / (ny + 1);
    if (fx <= nx) {
      const long long i0 = g.off_v + fx + nx1 * (fy + ny1 * fz);
      const bool fr = in_f(fx, nx) && in_f(fy, ny) && !zdir(g, fz);
      double yv = 0.0;
      if (fr) {
        const double u = __ldg(x + i0);
        const long long xw = g.off_e[0] + (fx - 1 + (long long)nx * (fy + ny1 * fz)) * NI, xe = xw + NI;
        const long long ys = g.off_e[1] + (fx + nx1 * (fy - 1 + (long long)ny * fz)) * NI, yn = ys + nx1 * NI;
        const long long zb = g.off_e[2] + (fx + nx1 * (fy + ny1 * (fz - 1))) * NI, zt = zb + nx1 * ny1 * NI;
        double lx = 0.0, ly = 0.0, lz = 0.0;
#pragma unroll
        for (int q = 0; q < NI; ++q) {
          lx = fma(cf.ap[q], __ldg(x + xw + q), fma(cf.a0[q], __ldg(x + xe + q), lx));
          ly = fma(cf.ap[q], __ldg(x + ys + q), fma(cf.a0[q], __ldg(x + yn + q), ly));
          lz = fma(cf.ap[q], __ldg(x + zb + q), fma(cf.a0[q], __ldg(x + zt + q), lz));
        }
        const double nbx = ldv<NI>(x, i0 - 1, fx - 1 > 0) + ldv<NI>(x, i0 + 1, fx + 1 < nx);
        const double nby = ldv<NI>(x, i0 - nx1, fy - 1 > 0) + ldv<NI>(x, i0 + nx1, fy + 1 < ny);
        const long long pl = nx1 * ny1;
        const double nbz = ldv<NI>(x, i0 - pl, fz - 1 >= 0 && !zdir(g, fz - 1)) + ldv<NI>(x, i0 + pl, fz + 1 <= nz && !zdir(g, fz + 1));
        yv = cf.vself * u + cf.vl[0] * fma(cf.K0p, nbx, lx) + cf.vl[1] * fma(cf.K0p, nby, ly) + cf.vl[2] * fma(cf.K0p, nbz, lz);
        if (DOT) dot = u * yv;
      }
      P.y[i0] = yv;
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
      P.dotp[(long long)blockIdx.z * gridDim.y * gridDim.x + (long long)blockIdx.y * gridDim.x + blockIdx.x] = s;
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

// Number of pass-B blocks (the p . q partials the PCG sums).
static void v7_grid(const Geom& g, int cls, dim3& grid) {
  const int ni = g.ni, nx = g.nx, ny = g.ny, nz = g.nz;
  long long len, rows;
  switch (cls) {
    case 0: len = (long long)(nx + 1) * ni; rows = (long long)ny * nz; break;     // faces: thread per (face, entry row)
    case 1: len = (long long)nx * ni; rows = (long long)(ny + 1) * nz; break;
    case 2: len = (long long)nx * ni; rows = (long long)ny * (nz + 1); break;
    case 3: len = (long long)nx * ni; rows = (long long)(ny + 1) * (nz + 1); break;
    case 4: len = (long long)(nx + 1) * ni; rows = (long long)ny * (nz + 1); break;
    case 5: len = (long long)(nx + 1) * ni; rows = (long long)(ny + 1) * nz; break;
    default: len = nx + 1; rows = (long long)(ny + 1) * (nz + 1); break;
  }
  grid = dim3((unsigned)((len + 255) / 256), (unsigned)rows, 1);
}

long long v7_dot_parts(const Geom& g) {
  long long tot = 0;
  for (int c = 0; c < 7; ++c) {
    dim3 gr;
    v7_grid(g, c, gr);
    tot += (long long)gr.x * gr.y;
  }
  return tot;
}

template <int NI>
static int launch_v7_t(V7Params& P, cudaStream_t st, int* nl) {
  const Geom& g = P.g;
  dim3 ga((unsigned)((g.nx + v7::RUN - 1) / v7::RUN), (unsigned)g.ny, (unsigned)g.nz);
  v7::k_v7_cond<NI><<<ga, 128, 0, st>>>(P);
  (*nl)++;
  double* dotp = P.dotp;
  for (int c = 0; c < 7; ++c) {
    dim3 gb;
    v7_grid(g, c, gb);
    if (dotp) {
      v7::k_v7_assemble<NI, true><<<gb, 256, 0, st>>>(P, c);
      P.dotp += (long long)gb.x * gb.y;
    } else {
      v7::k_v7_assemble<NI, false><<<gb, 256, 0, st>>>(P, c);
    }
    (*nl)++;
  }
  P.dotp = dotp;
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
