// L0: host 1-D transformed basis in long double (readings R2, R6).
//
// PAPER.md P:156-158  GLL Lagrange basis, lumped (diagonal) mass M = diag(w).
// PAPER.md P:119-123  K_ij = int phi_i' phi_j' (exact by GLL quadrature: degree 2p-2 <= 2p-1).
// PAPER.md P:302      S_II M_II S_II^T = I,  S_II K_II S_II^T = Lambda.
// PAPER.md P:381-395  Mtilde = diag(M00, I, Mpp); Ktilde arrowhead with
//                     Ktilde_I0 = S_II K_I0 (a0), Ktilde_Ip = S_II K_Ip (ap), Ktilde_II = Lambda.
//
// Construction (independent of any test-side construction): Newton on L_p' for the GLL nodes, the
// closed-form GLL differentiation matrix, K = D^T W D, reflection symmetrisation, a cyclic
// Jacobi eigen-solver on W^{-1/2} K_II W^{-1/2}, parity projection of every eigenvector
// (the centro-symmetric pencil has even/odd eigenvectors), ascending Lambda,
// sign rule a0_m > 0, and ap := sigma * a0 after checking |ap - sigma a0|.
#include "sc_internal.h"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

namespace sc {

typedef long double ld;

static void legendre(int p, ld x, ld* L, ld* dL) {
  // L_p(x) and L_p'(x) by the three-term recurrence.
  ld l0 = 1.0L, l1 = x, d0 = 0.0L, d1 = 1.0L;
  if (p == 0) { *L = 1.0L; *dL = 0.0L; return; }
  for (int n = 1; n < p; ++n) {
    ld l2 = ((2 * n + 1) * x * l1 - n * l0) / (n + 1);
    ld d2 = d0 + (2 * n + 1) * l1;   // L'_{n+1} = L'_{n-1} + (2n+1) L_n
    l0 = l1; l1 = l2; d0 = d1; d1 = d2;
  }
  *L = l1; *dL = d1;
}

static void jacobi_eigen(int n, std::vector<ld>& A, std::vector<ld>& V) {
  // Cyclic Jacobi for a symmetric n x n matrix A (row-major); on exit diag(A) holds the
  // eigenvalues and the columns of V the orthonormal eigenvectors.
  V.assign(n * n, 0.0L);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0L;
  for (int sweep = 0; sweep < 100; ++sweep) {
    ld off = 0.0L, diag = 0.0L;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) (i == j ? diag : off) += A[i * n + j] * A[i * n + j];
    if (off <= 1e-38L * diag) break;
    for (int pidx = 0; pidx < n - 1; ++pidx)
      for (int q = pidx + 1; q < n; ++q) {
        ld apq = A[pidx * n + q];
        if (fabsl(apq) < 1e-300L) continue;
        ld app = A[pidx * n + pidx], aqq = A[q * n + q];
        ld theta = (aqq - app) / (2.0L * apq);
        ld t = (theta >= 0 ? 1.0L : -1.0L) / (fabsl(theta) + sqrtl(theta * theta + 1.0L));
        ld c = 1.0L / sqrtl(t * t + 1.0L), s = t * c;
        for (int k = 0; k < n; ++k) {  // A <- J^T A J
          ld akp = A[k * n + pidx], akq = A[k * n + q];
          A[k * n + pidx] = c * akp - s * akq;
          A[k * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          ld apk = A[pidx * n + k], aqk = A[q * n + k];
          A[pidx * n + k] = c * apk - s * aqk;
          A[q * n + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          ld vkp = V[k * n + pidx], vkq = V[k * n + q];
          V[k * n + pidx] = c * vkp - s * vkq;
          V[k * n + q] = s * vkp + c * vkq;
        }
      }
  }
}

bool build_basis_1d(int p, Basis1D& B, std::string& err) {
  if (p < 2 || p > SC_PMAX) { err = "p out of range [2, 32]"; return false; }
  const int n = p + 1, ni = p - 1;
  std::vector<ld> x(n), w(n);
  // GLL nodes: -1, roots of L_p', +1.  Initial guesses: Chebyshev-Gauss-Lobatto points.
  x[0] = -1.0L; x[p] = 1.0L;
  for (int i = 1; i < p; ++i) {
    ld xi = -cosl(3.14159265358979323846264338327950288L * i / p);
    for (int it = 0; it < 100; ++it) {
      ld L, dL;
      legendre(p, xi, &L, &dL);
      // L'' from Legendre's equation (1-x^2) L'' - 2x L' + p(p+1) L = 0
      ld d2L = (2.0L * xi * dL - (ld)p * (p + 1) * L) / (1.0L - xi * xi);
      ld dx = dL / d2L;
      xi -= dx;
      if (fabsl(dx) < 1e-19L) break;
    }
    x[i] = xi;
  }
  for (int i = 0; i < n / 2; ++i) {   // exact antisymmetry
    ld s = 0.5L * (x[p - i] - x[i]);
    x[i] = -s; x[p - i] = s;
  }
  if (p % 2 == 0) x[p / 2] = 0.0L;
  std::vector<ld> Lx(n);
  for (int i = 0; i < n; ++i) {
    ld L, dL;
    legendre(p, x[i], &L, &dL);
    Lx[i] = L;
    w[i] = 2.0L / ((ld)p * (p + 1) * L * L);
  }
  for (int i = 0; i < n / 2; ++i) { ld s = 0.5L * (w[i] + w[p - i]); w[i] = w[p - i] = s; }
  // GLL differentiation matrix D[q][j] = phi_j'(x_q).
  std::vector<ld> D(n * n, 0.0L);
  for (int q = 0; q < n; ++q)
    for (int j = 0; j < n; ++j)
      if (q != j) D[q * n + j] = Lx[q] / (Lx[j] * (x[q] - x[j]));
  D[0] = -(ld)p * (p + 1) / 4.0L;
  D[p * n + p] = (ld)p * (p + 1) / 4.0L;
  // K = D^T W D, symmetrised and reflection-symmetrised (K_ij = K_{p-i,p-j}).
  std::vector<ld> K(n * n, 0.0L);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      ld s = 0.0L;
      for (int q = 0; q < n; ++q) s += D[q * n + i] * w[q] * D[q * n + j];
      K[i * n + j] = s;
    }
  std::vector<ld> Ks(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      Ks[i * n + j] = 0.25L * (K[i * n + j] + K[j * n + i] + K[(p - i) * n + (p - j)] + K[(p - j) * n + (p - i)]);
  K.swap(Ks);
  // Generalized eigenproblem (K_II, M_II) via A = W^{-1/2} K_II W^{-1/2}.
  std::vector<ld> A(ni * ni), V;
  for (int a = 0; a < ni; ++a)
    for (int b = 0; b < ni; ++b)
      A[a * ni + b] = K[(a + 1) * n + (b + 1)] / sqrtl(w[a + 1] * w[b + 1]);
  jacobi_eigen(ni, A, V);
  std::vector<int> order(ni);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return A[a * ni + a] < A[b * ni + b]; });
  std::vector<ld> S(ni * ni), lam(ni), a0(ni), ap(ni);
  B.parity_err = 0.0;
  for (int m = 0; m < ni; ++m) {
    int c = order[m];
    lam[m] = A[c * ni + c];
    std::vector<ld> s(ni);
    for (int i = 0; i < ni; ++i) s[i] = V[i * ni + c] / sqrtl(w[i + 1]);   // row m of S_II
    // parity projection: s <- (s + sigma J s)/2, then M-normalise
    ld par = 0.0L;
    for (int i = 0; i < ni; ++i) par += s[i] * s[ni - 1 - i] * w[i + 1];
    ld sg = par >= 0 ? 1.0L : -1.0L;
    std::vector<ld> t(ni);
    for (int i = 0; i < ni; ++i) t[i] = 0.5L * (s[i] + sg * s[ni - 1 - i]);
    ld nrm = 0.0L;
    for (int i = 0; i < ni; ++i) nrm += t[i] * t[i] * w[i + 1];
    nrm = sqrtl(nrm);
    ld va0 = 0.0L, vap = 0.0L;
    for (int i = 0; i < ni; ++i) {
      t[i] /= nrm;
      va0 += t[i] * K[(i + 1) * n + 0];
      vap += t[i] * K[(i + 1) * n + p];
    }
    ld sgn = va0 >= 0 ? 1.0L : -1.0L;      // sign rule a0_m > 0
    for (int i = 0; i < ni; ++i) S[m * ni + i] = sgn * t[i];
    a0[m] = sgn * va0;
    ap[m] = sgn * vap;
    B.sigma[m] = (ap[m] * a0[m] >= 0) ? 1 : -1;
    double e = (double)fabsl(ap[m] - B.sigma[m] * a0[m]) / (double)fabsl(a0[m]);
    B.parity_err = std::max(B.parity_err, e);
    if (a0[m] <= 0) { err = "a0_m vanishes: eigenvector orthogonal to K_I0"; return false; }
  }
  B.p = p; B.ni = ni;
  for (int i = 0; i < n; ++i) { B.x[i] = (double)x[i]; B.w[i] = (double)w[i]; }
  for (int m = 0; m < ni; ++m) {
    B.lam[m] = (double)lam[m];
    B.a0[m] = (double)a0[m];
    B.ap[m] = (double)(B.sigma[m] * a0[m]);
    for (int i = 0; i < ni; ++i) B.S[m * ni + i] = (double)S[m * ni + i];
  }
  B.K00 = (double)K[0];
  B.K0p = (double)K[p];
  B.w0 = (double)w[0];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) B.K[i * n + j] = (double)K[i * n + j];
  // sanity: eigen-residuals in long double
  ld res = 0.0L;
  for (int m = 0; m < ni; ++m)
    for (int q = 0; q < ni; ++q) {
      ld smk = 0.0L, smm = 0.0L;
      for (int i = 0; i < ni; ++i)
        for (int j = 0; j < ni; ++j) {
          smk += S[m * ni + i] * K[(i + 1) * n + (j + 1)] * S[q * ni + j];
          if (i == j) smm += S[m * ni + i] * w[i + 1] * S[q * ni + j];
        }
      res = std::max(res, fabsl(smk - (m == q ? lam[m] : 0.0L)) / lam[ni - 1]);
      res = std::max(res, fabsl(smm - (m == q ? 1.0L : 0.0L)));
    }
  B.eig_err = (double)res;
  if (B.eig_err > 1e-12) { err = "eigen-solver residual too large"; return false; }
  return true;
}

}  // namespace sc
