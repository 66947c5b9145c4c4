"""Workload grids of BASELINE.json; plain data, no method arithmetic.

A Grid is a Cartesian mesh of cuboidal elements ("only the case
of cuboidal elements") with per-direction element widths h_x[nx], h_y[ny],
h_z[nz], polynomial degree p and Helmholtz parameter lambda >= 0
(P:101).  Boundaries are homogeneous Dirichlet.
"""
from dataclasses import dataclass, field
import numpy as np


@dataclass
class Grid:
    p: int
    ne: tuple                 # (nx, ny, nz)
    hx: np.ndarray            # element widths along x, len nx
    hy: np.ndarray
    hz: np.ndarray
    lam: float
    origin: tuple = (0.0, 0.0, 0.0)
    name: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def n_elements(self):
        return int(self.ne[0] * self.ne[1] * self.ne[2])

    @property
    def n_lattice(self):
        nx, ny, nz = self.ne
        return (nx * self.p + 1) * (ny * self.p + 1) * (nz * self.p + 1)

    def n_skeleton(self):
        """N_c = N - n_e (p-1)^3 (lattice nodes on some element boundary)."""
        return self.n_lattice - self.n_elements * (self.p - 1) ** 3

    def edges(self, d):
        """Element interface coordinates along direction d (0=x,1=y,2=z)."""
        h = (self.hx, self.hy, self.hz)[d]
        return self.origin[d] + np.concatenate([[0.0], np.cumsum(h)])

    def uniform(self):
        return (np.all(self.hx == self.hx[0]) and np.all(self.hy == self.hy[0])
                and np.all(self.hz == self.hz[0]))


def small_grid(p, ne, lam, lengths=(1.0, 1.0, 1.0), name="small"):
    nx, ny, nz = ne
    return Grid(p=p, ne=(nx, ny, nz),
                hx=np.full(nx, lengths[0] / nx), hy=np.full(ny, lengths[1] / ny),
                hz=np.full(nz, lengths[2] / nz), lam=float(lam), name=name)


def cfg1():
    """BASELINE configs[0]: [0,1]^3, 2^3 elements, p=4, lambda=1."""
    return small_grid(4, (2, 2, 2), 1.0, name="cfg1")


def cfg2():
    """BASELINE configs[1]: [0,1]^3, 8^3 elements, p=8, lambda=0."""
    return small_grid(8, (8, 8, 8), 0.0, name="cfg2")


CFG3_P = (2, 4, 8, 12, 16, 24, 32)


def cfg3(p):
    """BASELINE configs[2]: n per direction = round(594/p), halves rounded up (SURVEY c16:
    p = 4 -> 149), lambda=1."""
    n = int(594.0 / p + 0.5)
    return small_grid(p, (n, n, n), 1.0, name=f"cfg3_p{p}")


def cfg4(ar, n=32):
    """BASELINE configs[3]: [0,AR]x[0,1]^2, 32^3 elements, p=16, lambda=0."""
    g = small_grid(16, (n, n, n), 0.0, lengths=(float(ar), 1.0, 1.0), name=f"cfg4_ar{ar}")
    g.extra["aspect_ratio"] = ar
    return g


def cfg5(n=128):
    """BASELINE configs[4]: [0,1]^3, 128^3 elements, p=8, lambda=1; z-slabs over GPUs."""
    return small_grid(8, (n, n, n), 1.0, name="cfg5")


def nonuniform_grid(p, ne, lam, seed=0, lo=0.3, hi=1.7):
    """Per-element widths drawn uniform[lo, hi) from a seeded generator (test geometry)."""
    rng = np.random.default_rng(seed)
    g = small_grid(p, ne, lam, name=f"nonuniform_s{seed}")
    g.hx = rng.uniform(lo, hi, ne[0])
    g.hy = rng.uniform(lo, hi, ne[1])
    g.hz = rng.uniform(lo, hi, ne[2])
    return g


def graded_widths(n, alpha, length):
    """n widths growing by the constant expansion factor alpha (h_e = h_0 alpha^e), summing to
    `length` (8 elements, alpha in {1, 1.5, 2}, AR_max = alpha^7 = 1 / 17 / 128)."""
    w = np.asarray([alpha ** e for e in range(n)], dtype=np.float64)
    return w * (length / w.sum())


def e3_grid(p, alpha, n=8, lam=0.0):
    """The paper's solver benchmark E3: Omega = (0, 2 pi)^3, n^3 elements graded with
    expansion factor alpha in every direction (reading R15), lambda = 0."""
    L = 2.0 * np.pi
    h = graded_widths(n, alpha, L)
    return Grid(p=p, ne=(n, n, n), hx=h.copy(), hy=h.copy(), hz=h.copy(), lam=float(lam),
                name=f"e3_p{p}_a{alpha}", extra={"alpha": alpha, "dirichlet": "e3"})
