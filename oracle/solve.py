"""Alg. 1 pipeline, block-Jacobi preconditioner, transformed-basis helpers
(ORACLE, test infrastructure only).

* condensed_rhs : Alg. 1 Fhat_e = F_B - H_BI H_II^{-1} F_I, gathered by R;
                  F_e = (h1 h2 h3 / 8) (w(x)w(x)w) * f(x_e)  (GLL-lumped mass).
* recover       : Alg. 1 u_I = H_II^{-1} (F_I - H_IB u_B).
* dirichlet_rhs : the condensed RHS with inhomogeneous Dirichlet data (E3): b_F - A_FD g_D.
* full_system   : the uncondensed SEM system R H_L R^T u = R F, dense, tiny grids.
* BlockJacobi   : the paper's block preconditioner: exact inverse of the
                  assembled self-block of every face, edge and vertex.  In the transformed
                  system it is the diagonal preconditioner of solver BT, and the two
                  produce identical PCG iterates (SURVEY c14 / finding 4).
* transform     : the basis change S = diag(1, S_II, 1) of P:361-369 applied along every
                  axis of the lattice.  Restricted to the skeleton it is the block-diagonal
                  Shat (faces S_II(x)S_II, edges S_II, vertices 1); dual vectors (residuals,
                  operator outputs, right-hand sides) map as Shat v, primal vectors
                  (solutions, operator inputs) as Shat^{-T} v  (Htilde = T H T^T).
"""
import numpy as np

from . import basis, element, mesh


def element_load(grid, f_lattice):
    """F_e[l, e] = (h1 h2 h3/8) w_i w_j w_k f(x_{e,ijk})."""
    p = grid.p
    _, w = basis.gll(p)
    w3 = np.einsum("k,j,i->kji", w, w, w).ravel()
    G = mesh.element_global_indices(grid)
    jac = np.prod(mesh.element_widths(grid), axis=1) / 8.0
    return (np.asarray(f_lattice).ravel()[G] * w3[None, :] * jac[:, None]).T


def condensed_rhs(op, f_lattice):
    """b = R (F_B - H_BI H_II^{-1} F_I), Dirichlet entries 0 (lattice vector)."""
    grid = op.grid
    Fe = element_load(grid, f_lattice)
    b = np.zeros(grid.n_lattice)
    for elems, ce in op.groups:
        FB = Fe[op.bidx][:, elems]
        FI = Fe[op.iidx][:, elems]
        Fh = ce.condense_rhs(FB, FI)
        np.add.at(b, op.GB[elems].ravel(), Fh.T.ravel())
    b[~op.free] = 0.0
    return b


def dirichlet_rhs(op, f_lattice, g_lattice):
    """Condensed right-hand side with inhomogeneous Dirichlet data g (the paper's E3):
    the skeleton unknowns split into free (F) and Dirichlet (D) nodes, u_D = g_D, and the condensed
    system R Hhat R^T u = R Fhat (Alg. 1) restricted to F reads
        A_FF u_F = (R Fhat)_F - A_FD g_D,
    computed element by element: Fhat_e - Hhat_e g_e, g_e = the element's boundary values of g on D
    (0 on F), gathered by R, Dirichlet entries 0."""
    grid = op.grid
    Fe = element_load(grid, f_lattice)
    dmask = mesh.dirichlet_mask(grid)
    gD = np.where(dmask, np.asarray(g_lattice, dtype=np.float64).ravel(), 0.0)
    b = np.zeros(grid.n_lattice)
    for elems, ce in op.groups:
        FB = Fe[op.bidx][:, elems]
        FI = Fe[op.iidx][:, elems]
        Fh = ce.condense_rhs(FB, FI) - ce.apply(gD[op.GB[elems]].T)
        np.add.at(b, op.GB[elems].ravel(), Fh.T.ravel())
    b[~op.free] = 0.0
    return b


def recover(op, f_lattice, u_skel, dirichlet=None):
    """Full lattice solution: skeleton from u_skel (free nodes) and, if given, the Dirichlet data
    `dirichlet` (lattice vector, used on the domain-boundary nodes); interiors by Eq.
    eq:condensation_inner."""
    grid = op.grid
    Fe = element_load(grid, f_lattice)
    u = np.where(op.free, np.asarray(u_skel).ravel(), 0.0)
    if dirichlet is not None:
        dmask = mesh.dirichlet_mask(grid)
        u = np.where(dmask, np.asarray(dirichlet, dtype=np.float64).ravel(), u)
    for elems, ce in op.groups:
        UB = u[op.GB[elems]].T
        FI = Fe[op.iidx][:, elems]
        UI = ce.recover(FI, UB)
        u[op.GI[elems].ravel()] = UI.T.ravel()
    return u


def full_system(grid, f_lattice):
    """Dense R H_L R^T and R F restricted to the free (non-Dirichlet) lattice nodes."""
    G = mesh.element_global_indices(grid)
    N = grid.n_lattice
    A = np.zeros((N, N))
    widths = mesh.element_widths(grid)
    for e in range(grid.n_elements):
        H = element.element_matrix(grid.p, element.metric_coefficients(widths[e], grid.lam), sparse=False)
        A[np.ix_(G[e], G[e])] += H
    F = mesh.gather(grid, element_load(grid, f_lattice), G)
    free = ~mesh.dirichlet_mask(grid)
    return A[np.ix_(free, free)], F[free], free


def entity_keys(grid, g):
    """Skeleton entity key (on-plane flags, gx//p, gy//p, gz//p) of lattice nodes g."""
    nx1, ny1, _ = mesh.lattice_dims(grid)
    p = grid.p
    gx, gy, gz = g % nx1, (g // nx1) % ny1, g // (nx1 * ny1)
    fl = (gx % p == 0).astype(np.int64) + 2 * (gy % p == 0) + 4 * (gz % p == 0)
    return [(int(a), int(b), int(c), int(d)) for a, b, c, d in zip(fl, gx // p, gy // p, gz // p)]


def assembled_diagonal(op):
    """diag(Rhat Hhat Rhat^T) on the lattice, 0 off the free skeleton: solver DC's diagonal
    preconditioner ("DC adds diagonal preconditioning"), summed element by element from the
    dense element Schur complements (P:107-109 assembly)."""
    d = np.zeros(op.grid.n_lattice)
    for elems, ce in op.groups:
        hd = np.diag(ce.explicit())
        for e in elems:
            np.add.at(d, op.GB[e], hd)
    return np.where(op.free, d, 0.0)


class BlockJacobi:
    """Inverse of the assembled face / edge / vertex self-blocks."""

    def __init__(self, op):
        self.op = op
        grid = op.grid
        blocks = {}
        members = {}
        for elems, ce in op.groups:
            Hh = ce.explicit()
            for e in elems:
                gB = op.GB[e]
                keys = entity_keys(grid, gB)
                byk = {}
                for loc, k in enumerate(keys):
                    byk.setdefault(k, []).append(loc)
                for k, locs in byk.items():
                    locs = np.array(locs)
                    order = np.argsort(gB[locs])
                    locs = locs[order]
                    if k not in blocks:
                        blocks[k] = np.zeros((len(locs), len(locs)))
                        members[k] = gB[locs]
                    blocks[k] += Hh[np.ix_(locs, locs)]
        self.items = []
        free = op.free
        for k, B in blocks.items():
            idx = members[k]
            if not free[idx[0]]:
                continue
            self.items.append((idx, np.linalg.inv(B)))

    def diagonal_blocks(self):
        return self.items

    def apply(self, r):
        r = np.asarray(r).ravel()
        z = np.zeros_like(r)
        for idx, Binv in self.items:
            z[idx] = Binv @ r[idx]
        return z


def _transform_axis(v, A, axis, p):
    """Apply the n_I x n_I matrix A to the element-interior segment of every
    element interval along ``axis`` of the lattice array v (planes untouched)."""
    v = np.moveaxis(v, axis, -1)
    n1 = v.shape[-1]
    ne = (n1 - 1) // p
    out = v.copy()
    for e in range(ne):
        seg = v[..., e * p + 1:(e + 1) * p]
        out[..., e * p + 1:(e + 1) * p] = seg @ A.T
    return np.moveaxis(out, -1, axis)


def transform(grid, vlat, kind):
    """kind: 'dual' (Shat v), 'primal' (Shat^{-T} v), 'dual_inv' (Shat^{-1} v),
    'primal_inv' (Shat^T v).  S^{-1} = M_II S^T from S M_II S^T = I."""
    p = grid.p
    _, S = basis.interior_eigen(p)
    _, w = basis.gll(p)
    MII = np.diag(w[1:p])
    A = {"dual": S, "primal": S @ MII, "dual_inv": MII @ S.T, "primal_inv": S.T}[kind]
    nx1, ny1, nz1 = mesh.lattice_dims(grid)
    v = np.asarray(vlat, dtype=np.float64).reshape(nz1, ny1, nx1)
    for axis in (2, 1, 0):
        v = _transform_axis(v, A, axis, p)
    return v.ravel()


def transformed_norm(grid, skel_mask):
    """norm(r) = || Shat r ||_2 over skeleton nodes (stopping rule in the transformed system, c6)."""
    def norm(r):
        t = transform(grid, np.where(skel_mask, r, 0.0), "dual")
        t = t[skel_mask]
        return float(np.sqrt(np.dot(t, t)))
    return norm
