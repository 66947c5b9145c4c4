"""Cartesian lattice numbering, gather R and scatter R^T (ORACLE, test infrastructure only).

PAPER.md P:105-110: "R gathers the contributions from the elements, and its
transpose R^T scatters the global degrees of freedom to those local to the
elements".  Global GLL lattice node (gx, gy, gz) = (ex p + i, ey p + j,
ez p + k), flat index g = gx + nx1 (gy + ny1 gz), x fastest; element index
e = ex + nx (ey + ny ez).  Nodes shared by neighbouring elements coincide
automatically (C0 continuity).
"""
import numpy as np

from . import basis


def lattice_dims(grid):
    nx, ny, nz = grid.ne
    p = grid.p
    return nx * p + 1, ny * p + 1, nz * p + 1


def element_global_indices(grid):
    """G[e, l]: global lattice index of local node l = i + n j + n^2 k of element e."""
    p = grid.p
    n = p + 1
    nx, ny, nz = grid.ne
    nx1, ny1, _ = lattice_dims(grid)
    ez, ey, ex = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ex, ey, ez = ex.ravel(), ey.ravel(), ez.ravel()
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    gx = ex[:, None] * p + i[None, :]
    gy = ey[:, None] * p + j[None, :]
    gz = ez[:, None] * p + k[None, :]
    return (gx + nx1 * (gy + ny1 * gz)).astype(np.int64)


def lattice_ijk(grid):
    nx1, ny1, nz1 = lattice_dims(grid)
    gz, gy, gx = np.meshgrid(np.arange(nz1), np.arange(ny1), np.arange(nx1), indexing="ij")
    return gx.ravel(), gy.ravel(), gz.ravel()


def skeleton_mask(grid):
    """True at lattice nodes on some element boundary (the condensed unknowns)."""
    gx, gy, gz = lattice_ijk(grid)
    p = grid.p
    return (gx % p == 0) | (gy % p == 0) | (gz % p == 0)


def dirichlet_mask(grid):
    """True at lattice nodes on the domain boundary (homogeneous Dirichlet).

    grid.extra["dirichlet_z"] = (lo, hi) can declare the z = 0 / z = top planes as interior
    cuts (a slab of a larger domain), which are then not Dirichlet."""
    gx, gy, gz = lattice_ijk(grid)
    nx1, ny1, nz1 = lattice_dims(grid)
    zlo, zhi = grid.extra.get("dirichlet_z", (True, True))
    return (gx == 0) | (gx == nx1 - 1) | (gy == 0) | (gy == ny1 - 1) | ((gz == 0) & zlo) | ((gz == nz1 - 1) & zhi)


def free_skeleton_mask(grid):
    return skeleton_mask(grid) & ~dirichlet_mask(grid)


def scatter(grid, xlat, G=None):
    """R^T: lattice vector -> element-local matrix X[l, e]."""
    if G is None:
        G = element_global_indices(grid)
    return np.asarray(xlat).ravel()[G].T


def gather(grid, Xloc, G=None):
    """R: element-local matrix X[l, e] -> lattice vector (sum of contributions)."""
    if G is None:
        G = element_global_indices(grid)
    out = np.zeros(grid.n_lattice)
    np.add.at(out, G.ravel(), np.asarray(Xloc).T.ravel())
    return out


def lattice_coordinates(grid):
    """Physical coordinates (x, y, z) of every lattice node (flat, x fastest)."""
    xi, _ = basis.gll(grid.p)
    p = grid.p
    coords = []
    for d, h in enumerate((grid.hx, grid.hy, grid.hz)):
        e0 = grid.edges(d)
        c = np.empty(len(h) * p + 1)
        for e in range(len(h)):
            c[e * p:(e + 1) * p + 1] = e0[e] + 0.5 * (1.0 + xi) * h[e]
        coords.append(c)
    Z, Y, X = np.meshgrid(coords[2], coords[1], coords[0], indexing="ij")
    return X.ravel(), Y.ravel(), Z.ravel()


def element_widths(grid):
    """Per-element (h1, h2, h3), shape (n_e, 3), element index e = ex + nx (ey + ny ez)."""
    nx, ny, nz = grid.ne
    ez, ey, ex = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return np.stack([grid.hx[ex.ravel()], grid.hy[ey.ravel()], grid.hz[ez.ravel()]], axis=1)
