"""Assembled condensed operator y = R Hhat R^T x (ORACLE, test infrastructure only).

PAPER.md P:236 (Alg. 1): the condensed system R Hhat R^T u = Fhat.  The
element operator is the dense Schur complement of element.py; elements are
grouped by geometry (one Schur matrix per distinct (h1,h2,h3)) and each group
is applied as one matrix-matrix product over all its elements' boundary
vectors -- the MMC idea of P:501-513 ("a single call to DGEMM").
Homogeneous Dirichlet: input Dirichlet entries are ignored and
output Dirichlet entries are 0.  Vectors live on the GLL lattice (flat, x
fastest); element-interior lattice entries are ignored on input, 0 on output.
"""
import numpy as np

from . import element, mesh


class AssembledCondensedOperator:
    def __init__(self, grid, explicit_max_p=12):
        self.grid = grid
        self.p = grid.p
        self.G = mesh.element_global_indices(grid)
        self.bidx, self.iidx = element.boundary_interior_split(grid.p)
        self.GB = self.G[:, self.bidx]
        self.GI = self.G[:, self.iidx]
        widths = mesh.element_widths(grid)
        keys, inv = np.unique(widths, axis=0, return_inverse=True)
        self.groups = []
        for gi, h in enumerate(keys):
            elems = np.nonzero(inv.ravel() == gi)[0]
            ce = element.CondensedElement(grid.p, element.metric_coefficients(h, grid.lam))
            if grid.p <= explicit_max_p:
                ce.explicit()
            self.groups.append((elems, ce))
        self.free = mesh.free_skeleton_mask(grid)
        self.skel = mesh.skeleton_mask(grid)

    def apply(self, x):
        x = np.where(self.free, np.asarray(x, dtype=np.float64).ravel(), 0.0)
        y = np.zeros(self.grid.n_lattice)
        for elems, ce in self.groups:
            XB = x[self.GB[elems]].T               # n_B x m  (R^T, restricted to B)
            YB = ce.apply(XB)                      # Hhat X
            np.add.at(y, self.GB[elems].ravel(), YB.T.ravel())   # R
        y[~self.free] = 0.0
        return y

    def elements_touching(self, g):
        """Element indices (e = ex + nx(ey + ny ez)) whose closure contains lattice node g."""
        nx, ny, nz = self.grid.ne
        nx1, ny1, _ = mesh.lattice_dims(self.grid)
        p = self.p
        gx, gy, gz = g % nx1, (g // nx1) % ny1, g // (nx1 * ny1)
        def cand(c, n):
            s = {c // p}
            if c % p == 0:
                s.add(c // p - 1)
            return [v for v in s if 0 <= v < n]
        return [ex + nx * (ey + ny * ez) for ez in cand(gz, nz) for ey in cand(gy, ny) for ex in cand(gx, nx)]

    def apply_at(self, x, targets):
        """y[targets] of self.apply(x), computed from the touching elements only.

        For checks at sizes where a full oracle application is too slow: the
        result depends only on the <= 8 elements around each target node.
        """
        x = np.asarray(x, dtype=np.float64).ravel()
        out = np.zeros(len(targets))
        for t, g in enumerate(targets):
            if not self.free[g]:
                continue
            acc = 0.0
            for e in self.elements_touching(g):
                for elems, ce in self.groups:
                    if e in set(elems.tolist()):
                        xb = np.where(self.free[self.GB[e]], x[self.GB[e]], 0.0)
                        yb = ce.apply(xb[:, None])[:, 0]
                        loc = np.nonzero(self.GB[e] == g)[0][0]
                        acc += yb[loc]
                        break
            out[t] = acc
        return out
