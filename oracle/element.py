"""Element Helmholtz matrix and its static condensation (ORACLE, test infrastructure only).

* d_e  : Eq. eq:metriccoeffelement
         d_e = (h1 h2 h3 / 8) (lambda, 4/h1^2, 4/h2^2, 4/h3^2).
* H_e  : Eq. eq:helmholtz_operator
         H_e = d0 M(x)M(x)M + d1 M(x)M(x)K + d2 M(x)K(x)M + d3 K(x)M(x)M,
         rightmost Kronecker factor acting on direction 1 (x, fastest local
         index i); local node (i,j,k) has index i + n j + n^2 k, n = p+1.
* B / I: P:173 -- interior = all three local indices in 1..p-1.
* Hhat : Eq. eq:condensation_system
         Hhat = H_BB - H_BI H_II^{-1} H_IB,
         applied as written (H_II^{-1} by a direct factorisation).
"""
import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import basis


def metric_coefficients(h, lam):
    """d_e of Eq. eq:metriccoeffelement for element widths h = (h1, h2, h3)."""
    h1, h2, h3 = (float(v) for v in h)
    if lam < 0 or not np.isfinite(lam):
        raise ValueError("lambda must be finite and >= 0 (P:101)")
    if min(h1, h2, h3) <= 0:
        raise ValueError("element widths must be > 0")
    s = h1 * h2 * h3 / 8.0
    return np.array([s * lam, s * 4.0 / h1 ** 2, s * 4.0 / h2 ** 2, s * 4.0 / h3 ** 2])


def local_index(p, i, j, k):
    n = p + 1
    return i + n * j + n * n * k


def boundary_interior_split(p):
    """Local lattice indices of boundary (B) and interior (I) nodes, ascending."""
    n = p + 1
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    on_b = (i == 0) | (i == p) | (j == 0) | (j == p) | (k == 0) | (k == p)
    idx = (i + n * j + n * n * k).ravel()
    on_b = on_b.ravel()
    return idx[on_b], idx[~on_b]


def element_matrix(p, d, sparse=True):
    """H_e of Eq. eq:helmholtz_operator as a (p+1)^3 square matrix (sparse CSR or dense)."""
    _, w, K = basis.mass_stiffness(p)
    M = sp.diags(w)
    Ks = sp.csr_matrix(K)
    kr = lambda a, b, c: sp.kron(a, sp.kron(b, c, format="csr"), format="csr")
    H = d[0] * kr(M, M, M) + d[1] * kr(M, M, Ks) + d[2] * kr(M, Ks, M) + d[3] * kr(Ks, M, M)
    H = H.tocsr()
    return H if sparse else H.toarray()


class CondensedElement:
    """Static condensation of one element geometry.

    apply(XB): columns of XB are element boundary vectors (ordered as
    ``self.bidx``); returns Hhat XB = H_BB XB - H_BI H_II^{-1} H_IB XB.
    """

    def __init__(self, p, d):
        self.p = p
        self.d = np.asarray(d, dtype=np.float64)
        self.bidx, self.iidx = boundary_interior_split(p)
        H = element_matrix(p, self.d, sparse=True)
        self.H = H
        self.H_BB = H[self.bidx][:, self.bidx].tocsr()
        self.H_BI = H[self.bidx][:, self.iidx].tocsr()
        self.H_IB = H[self.iidx][:, self.bidx].tocsr()
        H_II = H[self.iidx][:, self.iidx]
        nI = len(self.iidx)
        # dense Cholesky (multi-threaded LAPACK) up to p = 32 (n_I^3 = 29791, 7.1 GB): measured
        # 17 s at p = 24 and 73 s at p = 32 on 8 cores, against 103 s for the sparse LU at p = 24
        if nI <= 30000:
            self._chol = scipy.linalg.cho_factor(H_II.toarray())
            self._solve = lambda R: scipy.linalg.cho_solve(self._chol, R)
        else:
            lu = spla.splu(H_II.tocsc())
            self._solve = lambda R: lu.solve(np.asarray(R))
        self._dense = None

    def solve_II(self, R):
        """H_II^{-1} R (R: n_I x m)."""
        return self._solve(R)

    def apply(self, XB):
        XB = np.asarray(XB, dtype=np.float64)
        if self._dense is not None:
            return self._dense @ XB
        T = self.H_IB @ XB
        return self.H_BB @ XB - self.H_BI @ self.solve_II(T)

    def explicit(self):
        """Dense Hhat (n_B x n_B); cached, used MMC-style as one DGEMM."""
        if self._dense is None:
            HIB = self.H_IB.toarray()
            self._dense = self.H_BB.toarray() - self.H_BI @ self.solve_II(HIB)
        return self._dense

    def condense_rhs(self, FB, FI):
        """Fhat = F_B - H_BI H_II^{-1} F_I (Eq. eq:condensation_system)."""
        return FB - self.H_BI @ self.solve_II(FI)

    def recover(self, FI, UB):
        """u_I = H_II^{-1} (F_I - H_IB u_B) (Eq. eq:condensation_inner)."""
        return self.solve_II(FI - self.H_IB @ UB)
