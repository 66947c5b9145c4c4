// Condensed operator (TPT, Table 2 of PAPER.md P:425-440) and the BT preconditioner
// diagonal, v1: one CTA per element, shell staged in shared memory, assembly by fp64
// atomics into a zeroed output (faces: 2 contributors -> order-independent result).
//
// Per element (transformed basis, all loads from the skeleton vector):
//   a4 faces-in : u(i,j,k) = d1[a0_i W(j,k) + ap_i E(j,k)] + d2[a0_j S(i,k) + ap_j N(i,k)]
//                            + d3[a0_k B(i,j) + ap_k T(i,j)]                     (6 n_I^3 mult)
//   a5 diagonal : v = u * D^{-1},  D = d0 + d1 Lam_i + d2 Lam_j + d3 Lam_k         (n_I^3 mult)
//   a6 faces-out: W -= d1 sum_i a0_i v, E -= d1 sum_i ap_i v, ... (6 n_I^3 mult) -> 13 n_I^3
//   a7 primary  : Htilde_BB u_B with Mtilde = diag(w0,1..1,w0) and the arrowhead Ktilde
//                 (Eq. eq:east_east_primary_part_transformed)
//   a8 gather   : atomicAdd into the assembled skeleton vector (Dirichlet entities skipped).
#include <cuda_runtime.h>
#include "sc_device.cuh"

namespace sc {

static __device__ __forceinline__ double shU(const double* sU, int p, int ni, int i, int j, int k) {
  return sU[shell_index(p, ni, i, j, k)];
}

// Primary part (Htilde_BB u_B) at shell node (i,j,k), Eq. eq:east_east_primary_part_transformed
// generalised: y = d0 m_i m_j m_k u + sum_dir d_dir (prod of m over the other dirs) * (Ktilde u)_dir,
// where the 1-D sum runs over shell nodes only.
static __device__ double primary_at(const double* sU, int p, int ni, const double* d, const double* lam,
                                    const double* a0, const double* ap, double K00, double K0p, double w0,
                                    int i, int j, int k) {
  int c[3] = {i, j, k};
  bool b[3] = {i == 0 || i == p, j == 0 || j == p, k == 0 || k == p};
  double m[3] = {b[0] ? w0 : 1.0, b[1] ? w0 : 1.0, b[2] ? w0 : 1.0};
  double y = d[0] * m[0] * m[1] * m[2] * shU(sU, p, ni, i, j, k);
  for (int dir = 0; dir < 3; ++dir) {
    int o1 = (dir + 1) % 3, o2 = (dir + 2) % 3;
    int cc[3] = {c[0], c[1], c[2]};
    double t;
    if (!b[dir]) {
      int mm = c[dir] - 1;
      cc[dir] = 0; double u0 = shU(sU, p, ni, cc[0], cc[1], cc[2]);
      cc[dir] = p; double up = shU(sU, p, ni, cc[0], cc[1], cc[2]);
      t = a0[mm] * u0 + lam[mm] * shU(sU, p, ni, i, j, k) + ap[mm] * up;
    } else {
      bool first = (c[dir] == 0);
      cc[dir] = 0; double u0 = shU(sU, p, ni, cc[0], cc[1], cc[2]);
      cc[dir] = p; double up = shU(sU, p, ni, cc[0], cc[1], cc[2]);
      t = first ? (K00 * u0 + K0p * up) : (K0p * u0 + K00 * up);
      if (b[o1] || b[o2]) {  // the whole 1-D line lies in the shell: dense Ktilde row 0 / p
        const double* row = first ? a0 : ap;
        for (int q = 1; q < p; ++q) {
          cc[dir] = q;
          t += row[q - 1] * shU(sU, p, ni, cc[0], cc[1], cc[2]);
        }
      }
    }
    y += d[1 + dir] * m[o1] * m[o2] * t;
  }
  return y;
}

__global__ void k_apply_v1(Geom g, const double* __restrict__ x, double* __restrict__ y,
                           const double* __restrict__ done) {
  if (done != nullptr && *done != 0.0) return;
  const int p = g.p, ni = g.ni, n2 = ni * ni, nsh = 6 * n2 + 12 * ni + 8;
  const int kc_max = max(1, min(ni, 4096 / n2));
  extern __shared__ double sm[];
  double* sU = sm;               // shell input, nsh
  double* sO = sU + nsh;         // condensed face outputs, 6 n2
  double* sLam = sO + 6 * n2;
  double* sA0 = sLam + ni;
  double* sAp = sA0 + ni;
  double* sV = sAp + ni;         // kc_max * n2
  __shared__ long long sBase[26];
  __shared__ int sDir[26];
  const int e = blockIdx.x;
  const int ex = e % g.nx, ey = (e / g.nx) % g.ny, ez = e / (g.nx * g.ny);
  double d[4];
  metric(g, ex, ey, ez, d);
  const double K00 = g.tab[TAB_SCAL + 0], K0p = g.tab[TAB_SCAL + 1], w0 = g.tab[TAB_SCAL + 2];
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid < 26) {
    bool dr;
    sBase[tid] = entity_base(g, ex, ey, ez, tid, &dr);
    sDir[tid] = dr && !g.nodir;
  }
  for (int t = tid; t < ni; t += nt) {
    sLam[t] = g.tab[TAB_LAM + t];
    sA0[t] = g.tab[TAB_A0 + t];
    sAp[t] = g.tab[TAB_AP + t];
  }
  __syncthreads();
  for (int s = tid; s < nsh; s += nt) {
    int i, j, k, ent, loc;
    shell_node(p, ni, s, &i, &j, &k, &ent, &loc);
    sU[s] = sDir[ent] ? 0.0 : x[sBase[ent] + loc];
  }
  for (int t = tid; t < 2 * n2; t += nt) sO[4 * n2 + t] = 0.0;   // b/t accumulate over k-chunks
  __syncthreads();
  const double* W = sU;
  const double* E = sU + n2;
  const double* S = sU + 2 * n2;
  const double* N = sU + 3 * n2;
  const double* B = sU + 4 * n2;
  const double* T = sU + 5 * n2;
  for (int k0 = 0; k0 < ni; k0 += kc_max) {
    const int kc = min(kc_max, ni - k0);
    for (int t = tid; t < kc * n2; t += nt) {
      int i = t % ni, j = (t / ni) % ni, kk = t / n2, k = k0 + kk;
      double u = d[1] * (sA0[i] * W[j + ni * k] + sAp[i] * E[j + ni * k]) +
                 d[2] * (sA0[j] * S[i + ni * k] + sAp[j] * N[i + ni * k]) +
                 d[3] * (sA0[k] * B[i + ni * j] + sAp[k] * T[i + ni * j]);
      double dinv = g.dinv ? g.dinv[i + ni * (j + ni * k)]
                           : 1.0 / (d[0] + d[1] * sLam[i] + d[2] * sLam[j] + d[3] * sLam[k]);
      sV[t] = u * dinv;
    }
    __syncthreads();
    for (int t = tid; t < 2 * kc * ni + n2; t += nt) {
      if (t < kc * ni) {                   // x-lines: sum over i
        int j = t % ni, kk = t / ni;
        double qa = 0.0, qp = 0.0;
        for (int i = 0; i < ni; ++i) {
          double v = sV[i + ni * j + n2 * kk];
          qa += sA0[i] * v; qp += sAp[i] * v;
        }
        sO[0 * n2 + j + ni * (k0 + kk)] = -d[1] * qa;
        sO[1 * n2 + j + ni * (k0 + kk)] = -d[1] * qp;
      } else if (t < 2 * kc * ni) {        // y-lines: sum over j
        int tt = t - kc * ni, i = tt % ni, kk = tt / ni;
        double qa = 0.0, qp = 0.0;
        for (int j = 0; j < ni; ++j) {
          double v = sV[i + ni * j + n2 * kk];
          qa += sA0[j] * v; qp += sAp[j] * v;
        }
        sO[2 * n2 + i + ni * (k0 + kk)] = -d[2] * qa;
        sO[3 * n2 + i + ni * (k0 + kk)] = -d[2] * qp;
      } else {                             // z-lines: partial sum over this chunk's k
        int tt = t - 2 * kc * ni;          // = i + ni j
        double qa = 0.0, qp = 0.0;
        for (int kk = 0; kk < kc; ++kk) {
          double v = sV[tt + n2 * kk];
          qa += sA0[k0 + kk] * v; qp += sAp[k0 + kk] * v;
        }
        sO[4 * n2 + tt] -= d[3] * qa;
        sO[5 * n2 + tt] -= d[3] * qp;
      }
    }
    __syncthreads();
  }
  for (int s = tid; s < nsh; s += nt) {
    int i, j, k, ent, loc;
    shell_node(p, ni, s, &i, &j, &k, &ent, &loc);
    if (sDir[ent]) continue;
    double val = primary_at(sU, p, ni, d, sLam, sA0, sAp, K00, K0p, w0, i, j, k);
    if (s < 6 * n2) val += sO[s];
    atomicAdd(&y[sBase[ent] + loc], val);
  }
}

// Element contributions to diag(Rhat Htilde Rhat^T):
//   primary  d0 m_i m_j m_k + d1 kap_i m_j m_k + d2 m_i kap_j m_k + d3 m_i m_j kap_k,
//            kap = (K00, Lam_1..Lam_nI, K00), m = (w0, 1, .., 1, w0)
//   condensed (face nodes only): - d_dir^2 sum_q a_q^2 D^{-1}(..q..), a = a0 (low face) / ap (high face).
__global__ void k_diag(Geom g, double* __restrict__ diag) {
  const int p = g.p, ni = g.ni, n2 = ni * ni, nsh = 6 * n2 + 12 * ni + 8;
  const int e = blockIdx.x;
  const int ex = e % g.nx, ey = (e / g.nx) % g.ny, ez = e / (g.nx * g.ny);
  double d[4];
  metric(g, ex, ey, ez, d);
  const double K00 = g.tab[TAB_SCAL + 0], w0 = g.tab[TAB_SCAL + 2];
  const double* lam = g.tab + TAB_LAM;
  const double* a0 = g.tab + TAB_A0;
  const double* ap = g.tab + TAB_AP;
  for (int s = threadIdx.x; s < nsh; s += blockDim.x) {
    int i, j, k, ent, loc;
    shell_node(p, ni, s, &i, &j, &k, &ent, &loc);
    bool dr;
    long long base = entity_base(g, ex, ey, ez, ent, &dr);
    if (dr) continue;
    int c[3] = {i, j, k};
    double m[3], kap[3];
    for (int q = 0; q < 3; ++q) {
      bool bb = (c[q] == 0 || c[q] == p);
      m[q] = bb ? w0 : 1.0;
      kap[q] = bb ? K00 : lam[c[q] - 1];
    }
    double val = d[0] * m[0] * m[1] * m[2] + d[1] * kap[0] * m[1] * m[2] + d[2] * m[0] * kap[1] * m[2] +
                 d[3] * m[0] * m[1] * kap[2];
    if (ent < 6) {
      int dir = ent >> 1;
      const double* a = (ent & 1) ? ap : a0;
      double acc = 0.0;
      for (int q = 1; q < p; ++q) {
        int cc[3] = {i, j, k};
        cc[dir] = q;
        double D = d[0] + d[1] * lam[cc[0] - 1] + d[2] * lam[cc[1] - 1] + d[3] * lam[cc[2] - 1];
        acc += a[q - 1] * a[q - 1] / D;
      }
      val -= d[1 + dir] * d[1 + dir] * acc;
    }
    atomicAdd(&diag[base + loc], val);
  }
}

__global__ void k_invert_diag(Geom g, double* __restrict__ diag) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < g.n_total;
       q += (long long)gridDim.x * blockDim.x) {
    int gx, gy, gz;
    bool dr;
    bool ok = decode_entry(g, q, &gx, &gy, &gz, &dr);
    diag[q] = (ok && !dr) ? 1.0 / diag[q] : 0.0;
  }
}

static size_t apply_smem_bytes(int ni) {
  int n2 = ni * ni, nsh = 6 * n2 + 12 * ni + 8, kc = ni < 1 ? 1 : (4096 / n2 < 1 ? 1 : (4096 / n2 > ni ? ni : 4096 / n2));
  return sizeof(double) * (size_t)(nsh + 6 * n2 + 3 * ni + kc * n2);
}

int launch_apply(const Geom& g, const double* x, double* y, const double* done, void* stream, int* nl, void* events) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t* ev = (cudaEvent_t*)events;
  cudaError_t err = cudaMemsetAsync(y, 0, sizeof(double) * g.n_total, st);
  if (err != cudaSuccess) return err;
  if (ev) cudaEventRecord(ev[0], st);
  long long ne = (long long)g.nx * g.ny * g.nz;
  if (ne == 0) return cudaSuccess;
  size_t smem = apply_smem_bytes(g.ni);
  static bool attr_set[kMaxDev];   // per device
  const int dv = dev_slot();
  if (!attr_set[dv]) {
    cudaFuncSetAttribute(k_apply_v1, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set[dv] = true;
  }
  k_apply_v1<<<(unsigned)ne, 256, smem, st>>>(g, x, y, done);
  (*nl)++;
  if (ev) cudaEventRecord(ev[1], st);
  return cudaGetLastError();
}

int launch_diag(const Geom& g, double* diag, void* stream, int* nl) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t err = cudaMemsetAsync(diag, 0, sizeof(double) * g.n_total, st);
  if (err != cudaSuccess) return err;
  long long ne = (long long)g.nx * g.ny * g.nz;
  k_diag<<<(unsigned)ne, 256, 0, st>>>(g, diag);
  (*nl)++;
  return cudaGetLastError();
}

int launch_invert_diag(const Geom& g, double* diag, void* stream, int* nl) {
  k_invert_diag<<<1184, 256, 0, (cudaStream_t)stream>>>(g, diag);
  (*nl)++;
  return cudaGetLastError();
}

}  // namespace sc
