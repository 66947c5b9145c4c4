"""Counter-based splitmix64 generator.

z = seed * 0x9E3779B97F4A7C15 + g   (mod 2^64)
z ^= z >> 30; z *= 0xBF58476D1CE4E5B9
z ^= z >> 27; z *= 0x94D049BB133111EB
z ^= z >> 31
v = 2 * ((z >> 11) * 2^-53) - 1           in [-1, 1)

g is the global GLL-lattice index g = ix + nx1 * (iy + ny1 * iz) with
nx1 = n_x p + 1, ny1 = n_y p + 1.  The same value is produced by the CUDA
generator (``sc_fill_random``), independent of slab decomposition.
"""
import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed, g):
    """Vectorised splitmix64 finaliser of (seed, counter g); returns uint64."""
    g = np.asarray(g, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) * _GOLDEN + g
        z = z ^ (z >> np.uint64(30))
        z = z * _M1
        z = z ^ (z >> np.uint64(27))
        z = z * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(seed, g):
    """uniform[-1, 1) doubles keyed by (seed, g)."""
    z = splitmix64(seed, g)
    return 2.0 * ((z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)) - 1.0


def lattice_shape(ne, p):
    """(nz1, ny1, nx1) shape of the GLL lattice of a Cartesian grid, x fastest."""
    nx, ny, nz = ne
    return (nz * p + 1, ny * p + 1, nx * p + 1)


def lattice_random(seed, ne, p, skeleton_only=True, zero_dirichlet=True):
    """Seeded uniform[-1,1] nodal vector on the GLL lattice (shape (nz1, ny1, nx1)).

    skeleton_only: zero the element-interior lattice nodes (not on any element
    boundary); zero_dirichlet: zero the nodes on the domain boundary.
    """
    nz1, ny1, nx1 = lattice_shape(ne, p)
    g = np.arange(nx1 * ny1 * nz1, dtype=np.uint64)
    v = uniform_pm1(seed, g).reshape(nz1, ny1, nx1)
    iz, iy, ix = np.meshgrid(np.arange(nz1), np.arange(ny1), np.arange(nx1), indexing="ij")
    if skeleton_only:
        skel = (ix % p == 0) | (iy % p == 0) | (iz % p == 0)
        v = np.where(skel, v, 0.0)
    if zero_dirichlet:
        bnd = (ix == 0) | (ix == nx1 - 1) | (iy == 0) | (iy == ny1 - 1) | (iz == 0) | (iz == nz1 - 1)
        v = np.where(bnd, 0.0, v)
    return v
