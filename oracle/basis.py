"""1-D GLL nodal basis (ORACLE, test infrastructure only).

PAPER.md P:156-158: "Lagrange polynomials to the Gauss-Lobatto-Legendre (GLL)
quadrature points constitute the one-dimensional nodal basis functions ... The
mass matrix is approximated via GLL quadrature, generating a diagonal matrix".
P:119-123: M_ij = int phi_i phi_j, K_ij = int phi_i' phi_j'.
"""
import numpy as np
from numpy.polynomial import legendre as L
import scipy.linalg


def gll(p):
    """GLL nodes (ascending, x_0=-1, x_p=+1) and weights for degree p >= 1.

    Nodes: +-1 and the roots of L_p'(x); weights w_i = 2 / (p (p+1) L_p(x_i)^2).
    The interior roots (companion-matrix eigenvalues) are polished by Newton
    steps on L_p' and symmetrised (x_i = -x_{p-i}).
    """
    if p < 1:
        raise ValueError("p must be >= 1")
    cp = np.zeros(p + 1)
    cp[p] = 1.0                      # Legendre series coefficients of L_p
    dcp = L.legder(cp)               # L_p'
    ddcp = L.legder(dcp)             # L_p''
    if p >= 2:
        r = np.sort(np.real(L.legroots(dcp)))
        for _ in range(3):
            r = r - L.legval(r, dcp) / L.legval(r, ddcp)
        r = 0.5 * (r - r[::-1])      # exact antisymmetry
        x = np.concatenate([[-1.0], r, [1.0]])
    else:
        x = np.array([-1.0, 1.0])
    w = 2.0 / (p * (p + 1) * L.legval(x, cp) ** 2)
    w = 0.5 * (w + w[::-1])
    return x, w


def lagrange_derivative_matrix(x):
    """Dm[q, j] = phi_j'(x_q) for the Lagrange basis on nodes x.

    Definition: phi_j(x) = prod_{m != j} (x - x_m) / (x_j - x_m).  With the
    barycentric weights b_j = 1 / prod_{m != j} (x_j - x_m):
      phi_j'(x_q) = (b_j / b_q) / (x_q - x_j)           (q != j)
      phi_q'(x_q) = sum_{m != q} 1 / (x_q - x_m).
    """
    n = len(x)
    diff = x[:, None] - x[None, :]
    np.fill_diagonal(diff, 1.0)
    b = 1.0 / np.prod(diff, axis=1)
    Dm = (b[None, :] / b[:, None]) / diff
    np.fill_diagonal(Dm, 0.0)
    inv = 1.0 / diff
    np.fill_diagonal(inv, 0.0)
    Dm[np.arange(n), np.arange(n)] = inv.sum(axis=1)
    return Dm


def mass_stiffness(p):
    """GLL-lumped 1-D mass (vector of weights) and exact stiffness K = Dm^T diag(w) Dm.

    GLL quadrature with p+1 points is exact to degree 2p-1 >= 2p-2, the degree
    of phi_i' phi_j', so K is the exact integral.
    """
    x, w = gll(p)
    Dm = lagrange_derivative_matrix(x)
    K = Dm.T @ (w[:, None] * Dm)
    K = 0.5 * (K + K.T)
    return x, w, K


def interior_eigen(p):
    """Generalized eigenproblem of (K_II, M_II), Eq. eq:generalized_eigenvalues.

    Returns (Lam ascending, S_II) with S_II M_II S_II^T = I and
    S_II K_II S_II^T = diag(Lam); rows of S_II are the M-orthonormal
    eigenvectors.  Sign convention: (S_II K_I0)_m > 0.
    Used by the oracle ONLY to express vectors in the transformed basis.
    """
    x, w, K = mass_stiffness(p)
    I = slice(1, p)
    lam, V = scipy.linalg.eigh(K[I, I], np.diag(w[I]))
    S = V.T.copy()
    a0 = S @ K[I, 0]
    S *= np.sign(a0)[:, None]
    return lam, S
