// Operator variants of the paper's operator comparison (§7 "Efficiency of operators",
// P:493-504, Table 3 `tab:operator_complexities`), applied in the NODAL GLL basis:
//
//   y = Rhat Hhat Rhat^T x,   Hhat_e = H_BB - H_BI H_II^{-1} H_IB   (Eq. 17)
//
// TPC: Alg. 3 (`alg:face_to_eigenspace`) with the tensor-product
// suboperators of Table 1 (`tab:suboperators`) for the condensed part and the nodal
// primary part H_BB (Eqs. eq:east_east_primary_part / eq:east_west_primary_part):
//   faces in : T_f = (S M_II) (x) (S M_II) u_f                       (2 n_I^3 per face)
//              u^(a,b,c) = d1 [a0_a T_w(b,c) + ap_a T_e(b,c)] + d2 [..] + d3 [..]   (n_I^3 per face)
//   diagonal : v^ = D^{-1} u^   (Eq. eq:hii_diagonal)          (n_I^3)
//   faces out: Q_w(b,c) = sum_a a0_a v^(a,b,c), ...                   (n_I^3 per face)
//              v_w = -d1 (S M_II)^T (x) (S M_II)^T Q_w                (2 n_I^3 per face)
//   -> 37 n_I^3 multiplications, primary part 12 n_I^3 + O(n_I^2) (Table 3).
// With S_II M_II S_II^T = I (Eq. eq:generalized_eigenvalues; DESIGN reading R5) the
// suboperators of Table 1 read H_EFw = d1 (S M) (x) (S M) (x) (S K_I0) and H_FwE = its transpose;
// S K_I0 = a0 and S K_Ip = ap are the transformed basis' arrowhead columns.
//
// MMC (Alg. 2 `alg:face_to_face`): the element matrix Hhat_e (every shell node, primary
// and condensed part) is precomputed -- O(n_I^5) per distinct geometry (Table 3), by applying the
// element TPC operator to the unit vectors -- and applied to all elements' shells with one DGEMM
// ("a single call to DGEMM"; cuBLAS here), preceded by a gather kernel (R^T) and followed by
// an entity-centric assembly kernel (R, fixed summation order, no atomics).
#include <cuda_runtime.h>
#include "sc_device.cuh"

namespace sc {

// ---------------------------------------------------------------- element TPC (one CTA)
struct TpcShared {
  double *U, *T, *O, *W, *SM, *K, *w, *a0, *ap, *lam;
  int kc, wlen;
};

__host__ __device__ inline int tpc_kc(int ni) {
  int n2 = ni * ni;
  int kc = 2048 / n2;
  if (kc < 1) kc = 1;
  if (kc > ni) kc = ni;
  return kc;
}

__host__ __device__ inline size_t tpc_smem_doubles(int p) {
  const int ni = p - 1, n2 = ni * ni, nsh = 6 * n2 + 12 * ni + 8;
  int kc = tpc_kc(ni);
  int wlen = kc * n2 > 6 * n2 ? kc * n2 : 6 * n2;
  return (size_t)nsh + 6 * n2 + 6 * n2 + wlen + n2 + (p + 1) * (p + 1) + (p + 1) + 3 * ni;
}

__device__ inline TpcShared tpc_carve(double* sm, int p) {
  const int ni = p - 1, n2 = ni * ni, nsh = 6 * n2 + 12 * ni + 8;
  TpcShared s;
  s.kc = tpc_kc(ni);
  s.wlen = s.kc * n2 > 6 * n2 ? s.kc * n2 : 6 * n2;
  s.U = sm;
  s.T = s.U + nsh;
  s.O = s.T + 6 * n2;
  s.W = s.O + 6 * n2;
  s.SM = s.W + s.wlen;
  s.K = s.SM + n2;
  s.w = s.K + (p + 1) * (p + 1);
  s.a0 = s.w + (p + 1);
  s.ap = s.a0 + ni;
  s.lam = s.ap + ni;
  return s;
}

// Copy the 1-D tables (device `vt`, layout VT_* in sc_internal.h) into shared memory.
__device__ inline void tpc_load_tables(const TpcShared& s, const double* __restrict__ vt, int p) {
  const int ni = p - 1, n2 = ni * ni, np1 = p + 1;
  for (int t = threadIdx.x; t < n2; t += blockDim.x) s.SM[t] = vt[VT_SM + t];
  for (int t = threadIdx.x; t < np1 * np1; t += blockDim.x) s.K[t] = vt[VT_K + t];
  for (int t = threadIdx.x; t < np1; t += blockDim.x) s.w[t] = vt[VT_W + t];
  for (int t = threadIdx.x; t < ni; t += blockDim.x) {
    s.a0[t] = vt[VT_A0 + t];
    s.ap[t] = vt[VT_AP + t];
    s.lam[t] = vt[VT_LAM + t];
  }
}

// out_f(b,c) = scale_f * sum_{r,q} A'(b,r) A'(c,q) in_f(r,q) for the 6 faces (face arrays
// [r + n_I q]); A'(b,r) = A[b][r] (forward, Table 1 right column) or A[r][b] (transposed, left).
__device__ inline void face_transform6(const double* in, double* tmp, double* out, const double* A, int ni,
                                       bool trans, const double* scale6) {
  const int n2 = ni * ni;
  for (int t = threadIdx.x; t < 6 * n2; t += blockDim.x) {
    int f = t / n2, r = t - f * n2, b = r % ni, q = r / ni;
    const double* F = in + f * n2 + ni * q;
    double acc = 0.0;
    for (int m = 0; m < ni; ++m) acc += (trans ? A[m * ni + b] : A[b * ni + m]) * F[m];
    tmp[f * n2 + b + ni * q] = acc;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 6 * n2; t += blockDim.x) {
    int f = t / n2, r = t - f * n2, b = r % ni, c = r / ni;
    const double* Tm = tmp + f * n2 + b;
    double acc = 0.0;
    for (int m = 0; m < ni; ++m) acc += (trans ? A[m * ni + c] : A[c * ni + m]) * Tm[ni * m];
    out[f * n2 + b + ni * c] = scale6 ? scale6[f] * acc : acc;
  }
  __syncthreads();
}

// Nodal primary part H_BB u_B at shell node (i,j,k): the restriction of
// H_e = d0 M(x)M(x)M + d1 M(x)M(x)K + d2 M(x)K(x)M + d3 K(x)M(x)M to shell rows and
// columns.  A 1-D line through the node lies in the shell entirely when one of its two fixed
// coordinates is 0 or p; otherwise only its end points q = 0, p are shell nodes.
__device__ inline double primary_nodal(const double* U, const double* K, const double* w, int p, int ni,
                                       const double d[4], int i, int j, int k) {
  const int np1 = p + 1;
  const int c[3] = {i, j, k};
  const bool b[3] = {i == 0 || i == p, j == 0 || j == p, k == 0 || k == p};
  double y = d[0] * w[i] * w[j] * w[k] * U[shell_index(p, ni, i, j, k)];
  for (int dir = 0; dir < 3; ++dir) {
    const int o1 = (dir + 1) % 3, o2 = (dir + 2) % 3;
    const double* Kr = K + c[dir] * np1;
    int cc[3] = {i, j, k};
    double t = 0.0;
    if (b[o1] || b[o2]) {
      for (int q = 0; q <= p; ++q) {
        cc[dir] = q;
        t += Kr[q] * U[shell_index(p, ni, cc[0], cc[1], cc[2])];
      }
    } else {
      cc[dir] = 0;
      t = Kr[0] * U[shell_index(p, ni, cc[0], cc[1], cc[2])];
      cc[dir] = p;
      t += Kr[p] * U[shell_index(p, ni, cc[0], cc[1], cc[2])];
    }
    y += d[1 + dir] * w[c[o1]] * w[c[o2]] * t;
  }
  return y;
}

// Condensed part of one element (Alg. 3 with Table 1): s.U holds the nodal shell input; on return
// s.T[0 .. 6 n2) holds the condensed face outputs -H_FI H_II^{-1} H_IF u_F (faces w,e,s,n,b,t).
// dinv: uniform D^{-1} table (a fastest) or null (recomputed from d and Lambda).
__device__ inline void tpc_condensed(const TpcShared& s, int ni, const double d[4], const double* __restrict__ dinv) {
  const int n2 = ni * ni;
  const double* W_ = s.T;
  const double* E_ = s.T + n2;
  const double* S_ = s.T + 2 * n2;
  const double* N_ = s.T + 3 * n2;
  const double* B_ = s.T + 4 * n2;
  const double* T_ = s.T + 5 * n2;
  // faces in: T_f = (S M) (x) (S M) u_f
  face_transform6(s.U, s.W, s.T, s.SM, ni, false, nullptr);
  for (int t = threadIdx.x; t < 2 * n2; t += blockDim.x) s.O[4 * n2 + t] = 0.0;
  __syncthreads();
  for (int c0 = 0; c0 < ni; c0 += s.kc) {
    const int kc = min(s.kc, ni - c0);
    for (int t = threadIdx.x; t < kc * n2; t += blockDim.x) {
      const int a = t % ni, b = (t / ni) % ni, c = c0 + t / n2;
      const double u = d[1] * (s.a0[a] * W_[b + ni * c] + s.ap[a] * E_[b + ni * c]) +
                       d[2] * (s.a0[b] * S_[a + ni * c] + s.ap[b] * N_[a + ni * c]) +
                       d[3] * (s.a0[c] * B_[a + ni * b] + s.ap[c] * T_[a + ni * b]);
      const double di = dinv ? dinv[a + ni * (b + ni * c)]
                             : 1.0 / (d[0] + d[1] * s.lam[a] + d[2] * s.lam[b] + d[3] * s.lam[c]);
      s.W[t] = u * di;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * kc * ni + n2; t += blockDim.x) {
      if (t < kc * ni) {                   // x-lines: Q_w, Q_e = sum_a (a0_a, ap_a) v^(a,b,c)
        const int b = t % ni, cc = t / ni;
        double qa = 0.0, qp = 0.0;
        for (int a = 0; a < ni; ++a) {
          const double v = s.W[a + ni * b + n2 * cc];
          qa += s.a0[a] * v; qp += s.ap[a] * v;
        }
        s.O[b + ni * (c0 + cc)] = qa;
        s.O[n2 + b + ni * (c0 + cc)] = qp;
      } else if (t < 2 * kc * ni) {        // y-lines: Q_s, Q_n = sum_b
        const int tt = t - kc * ni, a = tt % ni, cc = tt / ni;
        double qa = 0.0, qp = 0.0;
        for (int b = 0; b < ni; ++b) {
          const double v = s.W[a + ni * b + n2 * cc];
          qa += s.a0[b] * v; qp += s.ap[b] * v;
        }
        s.O[2 * n2 + a + ni * (c0 + cc)] = qa;
        s.O[3 * n2 + a + ni * (c0 + cc)] = qp;
      } else {                             // z-lines: Q_b, Q_t = sum_c (accumulated over chunks)
        const int ab = t - 2 * kc * ni;
        double qa = 0.0, qp = 0.0;
        for (int cc = 0; cc < kc; ++cc) {
          const double v = s.W[ab + n2 * cc];
          qa += s.a0[c0 + cc] * v; qp += s.ap[c0 + cc] * v;
        }
        s.O[4 * n2 + ab] += qa;
        s.O[5 * n2 + ab] += qp;
      }
    }
    __syncthreads();
  }
  // faces out: v_f = -d_dir (S M)^T (x) (S M)^T Q_f  (into s.T)
  const double scale[6] = {-d[1], -d[1], -d[2], -d[2], -d[3], -d[3]};
  face_transform6(s.O, s.W, s.T, s.SM, ni, true, scale);
}

// ---------------------------------------------------------------- TPC kernel
__global__ void k_apply_tpc(Geom g, const double* __restrict__ vt, const double* __restrict__ x,
                            double* __restrict__ y) {
  const int p = g.p, ni = g.ni, n2 = ni * ni, nsh = 6 * n2 + 12 * ni + 8;
  extern __shared__ double sm[];
  TpcShared s = tpc_carve(sm, p);
  __shared__ long long sBase[26];
  __shared__ int sDir[26];
  const long long e = blockIdx.x;
  const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
  double d[4];
  metric(g, ex, ey, ez, d);
  if (threadIdx.x < 26) {
    bool dr;
    sBase[threadIdx.x] = entity_base(g, ex, ey, ez, threadIdx.x, &dr);
    sDir[threadIdx.x] = dr;
  }
  tpc_load_tables(s, vt, p);
  __syncthreads();
  for (int t = threadIdx.x; t < nsh; t += blockDim.x) {
    int i, j, k, ent, loc;
    shell_node(p, ni, t, &i, &j, &k, &ent, &loc);
    s.U[t] = sDir[ent] ? 0.0 : x[sBase[ent] + loc];
  }
  __syncthreads();
  tpc_condensed(s, ni, d, g.uniform ? g.dinv : nullptr);
  for (int t = threadIdx.x; t < nsh; t += blockDim.x) {
    int i, j, k, ent, loc;
    shell_node(p, ni, t, &i, &j, &k, &ent, &loc);
    if (sDir[ent]) continue;
    double val = primary_nodal(s.U, s.K, s.w, p, ni, d, i, j, k);
    if (t < 6 * n2) val += s.T[t];
    atomicAdd(&y[sBase[ent] + loc], val);
  }
}

// ---------------------------------------------------------------- MMC
// Column `c` of the element matrix Hhat_e (shell numbering of shell_node) of geometry `gi`
// (uniform: element (0,0,0); otherwise element gi): the element operator applied to e_c.
__global__ void k_mmc_columns(Geom g, const double* __restrict__ vt, double* __restrict__ H, int nB, long long g0) {
  const int p = g.p, ni = g.ni, n2 = ni * ni;
  extern __shared__ double sm[];
  TpcShared s = tpc_carve(sm, p);
  const int c = blockIdx.x;
  const long long gi = g0 + blockIdx.y;
  const int ex = (int)(gi % g.nx), ey = (int)((gi / g.nx) % g.ny), ez = (int)(gi / ((long long)g.nx * g.ny));
  double d[4];
  metric(g, ex, ey, ez, d);
  tpc_load_tables(s, vt, p);
  for (int t = threadIdx.x; t < nB; t += blockDim.x) s.U[t] = (t == c) ? 1.0 : 0.0;
  __syncthreads();
  tpc_condensed(s, ni, d, g.uniform ? g.dinv : nullptr);
  double* col = H + (size_t)gi * nB * nB + (size_t)c * nB;
  for (int t = threadIdx.x; t < nB; t += blockDim.x) {
    int i, j, k, ent, loc;
    shell_node(p, ni, t, &i, &j, &k, &ent, &loc);
    double val = primary_nodal(s.U, s.K, s.w, p, ni, d, i, j, k);
    if (t < 6 * n2) val += s.T[t];
    col[t] = val;
  }
}

// R^T: X[e][s] = x at shell node s of element e (0 on Dirichlet entities).
__global__ void k_mmc_gather(Geom g, const double* __restrict__ x, double* __restrict__ X, int nB, long long ne) {
  __shared__ long long sBase[26];
  __shared__ int sDir[26];
  const int p = g.p, ni = g.ni;
  for (long long e = blockIdx.x; e < ne; e += gridDim.x) {
    const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
    __syncthreads();
    if (threadIdx.x < 26) {
      bool dr;
      sBase[threadIdx.x] = entity_base(g, ex, ey, ez, threadIdx.x, &dr);
      sDir[threadIdx.x] = dr;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nB; t += blockDim.x) {
      int i, j, k, ent, loc;
      shell_node(p, ni, t, &i, &j, &k, &ent, &loc);
      X[e * nB + t] = sDir[ent] ? 0.0 : x[sBase[ent] + loc];
    }
  }
}

// R: y[q] = sum over the elements sharing skeleton node q (fixed order: ez, ey, ex ascending) of
// Y[e][s_e(q)]; Dirichlet and padding entries are written as 0.
__global__ void k_mmc_assemble(Geom g, const double* __restrict__ Y, double* __restrict__ y, int nB) {
  const int p = g.p, ni = g.ni;
  const int nel[3] = {g.nx, g.ny, g.nz};
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.n_total;
       q += (long long)gridDim.x * blockDim.x) {
    int G[3];
    bool dr;
    if (!decode_entry(g, q, &G[0], &G[1], &G[2], &dr) || dr) { y[q] = 0.0; continue; }
    int lo[3], hi[3];
    for (int dd = 0; dd < 3; ++dd) {
      if (G[dd] % p == 0) {
        lo[dd] = G[dd] / p - 1; hi[dd] = G[dd] / p;
        if (lo[dd] < 0) lo[dd] = 0;
        if (hi[dd] > nel[dd] - 1) hi[dd] = nel[dd] - 1;
      } else {
        lo[dd] = hi[dd] = G[dd] / p;
      }
    }
    double acc = 0.0;
    for (int ez = lo[2]; ez <= hi[2]; ++ez)
      for (int ey = lo[1]; ey <= hi[1]; ++ey)
        for (int ex = lo[0]; ex <= hi[0]; ++ex) {
          const long long e = ex + (long long)g.nx * (ey + (long long)g.ny * ez);
          const int s = shell_index(p, ni, G[0] - p * ex, G[1] - p * ey, G[2] - p * ez);
          acc += Y[e * nB + s];
        }
    y[q] = acc;
  }
}

// ---------------------------------------------------------------- solvers UC / DC / BC
// DC: element contributions to diag(Rhat Hhat Rhat^T) in the nodal basis.  Primary part: the
// diagonal of H_e = d0 M(x)M(x)M + d1 M(x)M(x)K + ... at the shell node; condensed part (face nodes
// only): with H_EFw = d1 (S M)(x)(S M)(x)a0 (Table 1), diag(H_FwI H_II^{-1} H_IFw)(j,k) =
// d1^2 sum_{b,c} (S M)_{b j}^2 (S M)_{c k}^2 G_w(b,c),  G_w(b,c) = sum_a a0_a^2 D^{-1}(a,b,c).
__global__ void k_var_diag(Geom g, const double* __restrict__ vt, double* __restrict__ diag) {
  const int p = g.p, ni = g.ni, n2 = ni * ni, nsh = 6 * n2 + 12 * ni + 8, np1 = p + 1;
  extern __shared__ double sm[];
  double* G = sm;                // 6 n2: G_f(b,c) per face f
  double* SM2 = G + 6 * n2;      // (S M)^2 entrywise
  double* K = SM2 + n2;          // (p+1)^2
  double* w = K + np1 * np1;
  double* a0 = w + np1;
  double* ap = a0 + ni;
  double* lam = ap + ni;
  const long long e = blockIdx.x;
  const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
  double d[4];
  metric(g, ex, ey, ez, d);
  for (int t = threadIdx.x; t < n2; t += blockDim.x) SM2[t] = vt[VT_SM + t] * vt[VT_SM + t];
  for (int t = threadIdx.x; t < np1 * np1; t += blockDim.x) K[t] = vt[VT_K + t];
  for (int t = threadIdx.x; t < np1; t += blockDim.x) w[t] = vt[VT_W + t];
  for (int t = threadIdx.x; t < ni; t += blockDim.x) {
    a0[t] = vt[VT_A0 + t]; ap[t] = vt[VT_AP + t]; lam[t] = vt[VT_LAM + t];
  }
  __syncthreads();
  // G_f(r,s): sum over the face-normal eigen-index m of a_m^2 / D, (r,s) the in-face eigen-indices
  for (int t = threadIdx.x; t < 6 * n2; t += blockDim.x) {
    const int f = t / n2, rr = t % n2, r = rr % ni, q = rr / ni, dir = f >> 1;
    const double* a = (f & 1) ? ap : a0;
    double acc = 0.0;
    for (int m = 0; m < ni; ++m) {
      const int ii = dir == 0 ? m : r, jj = dir == 0 ? r : (dir == 1 ? m : q), kk = dir == 2 ? m : q;
      acc += a[m] * a[m] / (d[0] + d[1] * lam[ii] + d[2] * lam[jj] + d[3] * lam[kk]);
    }
    G[t] = acc;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nsh; t += blockDim.x) {
    int i, j, k, ent, loc;
    shell_node(p, ni, t, &i, &j, &k, &ent, &loc);
    bool dr;
    const long long base = entity_base(g, ex, ey, ez, ent, &dr);
    if (dr) continue;
    double val = d[0] * w[i] * w[j] * w[k] + d[1] * K[i * np1 + i] * w[j] * w[k] + d[2] * w[i] * K[j * np1 + j] * w[k] +
                 d[3] * w[i] * w[j] * K[k * np1 + k];
    if (ent < 6) {
      const int dir = ent >> 1, u = loc % ni, v = loc / ni;   // face coords (u, v) in-plane order
      const double* Gf = G + ent * n2;
      double acc = 0.0;
      for (int c = 0; c < ni; ++c)
        for (int b = 0; b < ni; ++b) acc += SM2[b * ni + u] * SM2[c * ni + v] * Gf[b + ni * c];
      val -= d[1 + dir] * d[1 + dir] * acc;
    }
    atomicAdd(&diag[base + loc], val);
  }
}

// BC: z = Shat^T Ptilde Shat r entity by entity (the exact inverse of every assembled face / edge /
// vertex self-block: in the transformed basis these blocks are diagonal, Ptilde = the BT
// diagonal, DESIGN reading R12), i.e. 4 n_I^3 per face (Table 4 "BC: 24 n_I^3").
// UC / DC: z = m .* r with m = free mask / 1/diag.
__global__ void k_var_prec(Geom g, int mode, const double* __restrict__ m, const double* __restrict__ r,
                           double* __restrict__ z) {
  const int ni = g.ni, n2 = ni * ni;
  if (mode != 2) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.n_total;
         i += (long long)gridDim.x * blockDim.x)
      z[i] = m[i] * r[i];
    return;
  }
  extern __shared__ double sm[];
  double* S = sm;            // S_II row-major
  double* t0 = S + n2;       // n2
  double* t1 = t0 + n2;      // n2
  for (int t = threadIdx.x; t < n2; t += blockDim.x) S[t] = g.tab[TAB_MAT + MAT_S * SC_NIMAX * SC_NIMAX + t];
  const long long nf = g.n_f[0] + g.n_f[1] + g.n_f[2], ned = g.n_e[0] + g.n_e[1] + g.n_e[2];
  for (long long ent = blockIdx.x; ent < nf + ned + 1; ent += gridDim.x) {
    __syncthreads();
    if (ent < nf) {
      const int c = ent < g.n_f[0] ? 0 : (ent < g.n_f[0] + g.n_f[1] ? 1 : 2);
      const long long id = ent - (c == 0 ? 0 : (c == 1 ? g.n_f[0] : g.n_f[0] + g.n_f[1]));
      const long long base = g.off_f[c] + id * n2;
      for (int t = threadIdx.x; t < n2; t += blockDim.x) {      // t0 = (I (x) S) r : along the first coord
        const int a = t % ni, q = t / ni;
        double acc = 0.0;
        for (int u = 0; u < ni; ++u) acc += S[a * ni + u] * r[base + u + ni * q];
        t0[t] = acc;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < n2; t += blockDim.x) {      // t1 = Ptilde (S (x) I) t0
        const int a = t % ni, b = t / ni;
        double acc = 0.0;
        for (int v = 0; v < ni; ++v) acc += S[b * ni + v] * t0[a + ni * v];
        t1[t] = m[base + t] * acc;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < n2; t += blockDim.x) {      // t0 = (S^T (x) I) t1
        const int a = t % ni, v = t / ni;
        double acc = 0.0;
        for (int b = 0; b < ni; ++b) acc += S[b * ni + v] * t1[a + ni * b];
        t0[t] = acc;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < n2; t += blockDim.x) {      // z = (I (x) S^T) t0
        const int u = t % ni, v = t / ni;
        double acc = 0.0;
        for (int a = 0; a < ni; ++a) acc += S[a * ni + u] * t0[a + ni * v];
        z[base + t] = acc;
      }
    } else if (ent < nf + ned) {   // a whole edge class row-range per block: warp per edge
      const long long e0 = ent - nf;
      const int c = e0 < g.n_e[0] ? 0 : (e0 < g.n_e[0] + g.n_e[1] ? 1 : 2);
      const long long id = e0 - (c == 0 ? 0 : (c == 1 ? g.n_e[0] : g.n_e[0] + g.n_e[1]));
      const long long base = g.off_e[c] + id * ni;
      for (int t = threadIdx.x; t < ni; t += blockDim.x) {
        double acc = 0.0;
        for (int u = 0; u < ni; ++u) acc += S[t * ni + u] * r[base + u];
        t0[t] = m[base + t] * acc;
      }
      __syncthreads();
      for (int t = threadIdx.x; t < ni; t += blockDim.x) {
        double acc = 0.0;
        for (int a = 0; a < ni; ++a) acc += S[a * ni + t] * t0[a];
        z[base + t] = acc;
      }
    } else {                       // vertices (and the padding entries) in one grid-stride pass
      for (long long i = threadIdx.x; i < g.n_total - g.off_v; i += blockDim.x)
        z[g.off_v + i] = m[g.off_v + i] * r[g.off_v + i];
    }
  }
}

// m = 1 where mask != 0 (free entries), else 0 (UC's preconditioner).
__global__ void k_unit_mask(const double* __restrict__ mask, double* __restrict__ m, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    m[i] = mask[i] != 0.0 ? 1.0 : 0.0;
}

// r = b on free entries (mask != 0), x = 0.
__global__ void k_var_init(const double* __restrict__ b, const double* __restrict__ mask, double* __restrict__ r,
                           double* __restrict__ x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    r[i] = mask[i] != 0.0 ? b[i] : 0.0;
    x[i] = 0.0;
  }
}

// r -= alpha q
__global__ void k_var_update(double* __restrict__ r, const double* __restrict__ q, long long n,
                             const double* __restrict__ scal) {
  if (scal[SCAL_DONE] != 0.0) return;
  const double alpha = scal[SCAL_ALPHA];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    r[i] -= alpha * q[i];
}

// x += alpha p (if this iteration's alpha step ran) ; p = z + beta p (unless converged) ; first = 1: p = z.
__global__ void k_var_direction(double* __restrict__ x, double* __restrict__ p, const double* __restrict__ z,
                                long long n, const double* __restrict__ scal, int first) {
  if (first) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
      p[i] = z[i];
    return;
  }
  if (scal[SCAL_RAN] == 0.0 || scal[SCAL_BREAK] != 0.0) return;
  const double alpha = scal[SCAL_ALPHA], beta = scal[SCAL_BETA];
  const bool dir = scal[SCAL_DONE] == 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double pi = p[i];
    x[i] += alpha * pi;
    if (dir) p[i] = z[i] + beta * pi;
  }
}

// ---------------------------------------------------------------- launchers
// Dynamic shared-memory opt-in for the element kernels (the largest need, p = 32, is ~204 KB).
static cudaError_t set_smem_attr(const void* fn, size_t bytes, size_t* done) {
  const int dv = dev_slot();
  if (done[dv] >= bytes) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[dv] = bytes;
  return e;
}

int launch_apply_tpc(const Geom& g, const double* vt, const double* x, double* y, void* stream, int* nl,
                     void* events) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  cudaError_t err = cudaMemsetAsync(y, 0, sizeof(double) * g.n_total, st);
  if (err != cudaSuccess) return err;
  const long long ne = (long long)g.nx * g.ny * g.nz;
  if (ev) cudaEventRecord(ev[0], st);
  if (ne > 0) {
    static size_t attr[kMaxDev];
    const size_t smem = sizeof(double) * tpc_smem_doubles(g.p);
    if ((err = set_smem_attr((const void*)k_apply_tpc, smem, attr)) != cudaSuccess) return err;
    k_apply_tpc<<<(unsigned)ne, 256, smem, st>>>(g, vt, x, y);
    (*nl)++;
  }
  if (ev) cudaEventRecord(ev[1], st);
  return cudaGetLastError();
}

int launch_mmc_columns(const Geom& g, const double* vt, double* H, int nB, long long ngeom, void* stream, int* nl) {
  static size_t attr[kMaxDev];
  const size_t smem = sizeof(double) * tpc_smem_doubles(g.p);
  cudaError_t err = set_smem_attr((const void*)k_mmc_columns, smem, attr);
  if (err != cudaSuccess) return err;
  for (long long g0 = 0; g0 < ngeom; g0 += 65535) {   // grid.y limit
    const long long cnt = ngeom - g0 < 65535 ? ngeom - g0 : 65535;
    k_mmc_columns<<<dim3((unsigned)nB, (unsigned)cnt), 256, smem, (cudaStream_t)stream>>>(g, vt, H, nB, g0);
    (*nl)++;
  }
  return cudaGetLastError();
}

int launch_mmc_gather(const Geom& g, const double* x, double* X, int nB, void* stream, int* nl) {
  const long long ne = (long long)g.nx * g.ny * g.nz;
  const unsigned grid = (unsigned)(ne < 148LL * 16 ? ne : 148LL * 16);
  if (ne > 0) {
    k_mmc_gather<<<grid, 256, 0, (cudaStream_t)stream>>>(g, x, X, nB, ne);
    (*nl)++;
  }
  return cudaGetLastError();
}

int launch_mmc_assemble(const Geom& g, const double* Y, double* y, int nB, void* stream, int* nl) {
  k_mmc_assemble<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(g, Y, y, nB);
  (*nl)++;
  return cudaGetLastError();
}

int launch_var_diag(const Geom& g, const double* vt, double* diag, void* stream, int* nl) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t err = cudaMemsetAsync(diag, 0, sizeof(double) * g.n_total, st);
  if (err != cudaSuccess) return err;
  const long long ne = (long long)g.nx * g.ny * g.nz;
  const int ni = g.ni, n2 = ni * ni, np1 = g.p + 1;
  const size_t smem = sizeof(double) * (7 * n2 + np1 * np1 + np1 + 3 * ni);
  static size_t attr[kMaxDev];
  if ((err = set_smem_attr((const void*)k_var_diag, smem, attr)) != cudaSuccess) return err;
  if (ne > 0) {
    k_var_diag<<<(unsigned)ne, 256, smem, st>>>(g, vt, diag);
    (*nl)++;
  }
  return cudaGetLastError();
}

int launch_var_prec(const Geom& g, int mode, const double* m, const double* r, double* z, void* stream, int* nl) {
  const size_t smem = mode == 2 ? sizeof(double) * 3 * g.ni * g.ni : 0;
  k_var_prec<<<mode == 2 ? 148 * 8 : SC_RED_BLOCKS, mode == 2 ? 128 : 256, smem, (cudaStream_t)stream>>>(g, mode, m, r, z);
  (*nl)++;
  return cudaGetLastError();
}

int launch_unit_mask(const double* mask, double* m, long long n, void* stream, int* nl) {
  k_unit_mask<<<SC_RED_BLOCKS, 256, 0, (cudaStream_t)stream>>>(mask, m, n);
  (*nl)++;
  return cudaGetLastError();
}

int launch_var_init(const double* b, const double* mask, double* r, double* x, long long n, void* stream, int* nl) {
  k_var_init<<<SC_RED_BLOCKS, 256, 0, (cudaStream_t)stream>>>(b, mask, r, x, n);
  (*nl)++;
  return cudaGetLastError();
}

int launch_var_update(double* r, const double* q, long long n, const double* scal, void* stream, int* nl) {
  k_var_update<<<SC_RED_BLOCKS, 256, 0, (cudaStream_t)stream>>>(r, q, n, scal);
  (*nl)++;
  return cudaGetLastError();
}

int launch_var_direction(double* x, double* p, const double* z, long long n, const double* scal, int first,
                         void* stream, int* nl) {
  k_var_direction<<<SC_RED_BLOCKS, 256, 0, (cudaStream_t)stream>>>(x, p, z, n, scal, first);
  (*nl)++;
  return cudaGetLastError();
}

}  // namespace sc
