"""Manufactured solutions of BASELINE.json configs (input data only).

u = sin(pi x) sin(pi y) sin(pi z) vanishes on the boundary of [0,A]x[0,1]^2 for
integer A, and f = lambda u - Laplace(u) = (lambda + 3 pi^2) u (PAPER.md
P:96-101, Eq. eq:helmholtz_equation).  Coordinates are passed in by the
caller (each side computes GLL lattice coordinates with its own basis code).
"""
import numpy as np


def sine_u(x, y, z):
    return np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)


def sine_f(x, y, z, lam):
    return (lam + 3.0 * np.pi ** 2) * sine_u(x, y, z)


# ---- PAPER.md Eq. eq:solution, the solver benchmark E3 -------------------------
# u_ex = cos(k(x1 - 3x2 + 2x3)) sin(k(1 + x1)) sin(k(1 - x2)) sin(k(2x1 + x2)) sin(k(3x1 - 2x2 + 2x3))
# on (0, 2 pi)^3 with k = 5, inhomogeneous Dirichlet data u_ex on the boundary, and
# f = lambda u_ex - Laplace(u_ex) evaluated analytically.  Each factor is
# g_m(theta_m), theta_m = k (a_m . x + c_m); for a product of such factors
#   Laplace(u) = k^2 [ -(sum_m |a_m|^2) u + 2 sum_{m<n} (a_m . a_n) g_m' g_n' prod_{l != m,n} g_l ].
_E3_FACTORS = (  # (a, c, kind)
    ((1.0, -3.0, 2.0), 0.0, "cos"),
    ((1.0, 0.0, 0.0), 1.0, "sin"),
    ((0.0, -1.0, 0.0), 1.0, "sin"),
    ((2.0, 1.0, 0.0), 0.0, "sin"),
    ((3.0, -2.0, 2.0), 0.0, "sin"),
)


def _e3_terms(x, y, z, k):
    g, dg = [], []
    for a, c, kind in _E3_FACTORS:
        th = k * (a[0] * x + a[1] * y + a[2] * z + c)
        if kind == "sin":
            g.append(np.sin(th)); dg.append(np.cos(th))
        else:
            g.append(np.cos(th)); dg.append(-np.sin(th))
    return g, dg


def e3_u(x, y, z, k=5.0):
    g, _ = _e3_terms(x, y, z, k)
    out = np.ones_like(np.asarray(x, dtype=np.float64))
    for v in g:
        out = out * v
    return out


def e3_f(x, y, z, lam, k=5.0):
    g, dg = _e3_terms(x, y, z, k)
    a = [np.array(f[0]) for f in _E3_FACTORS]
    u = e3_u(x, y, z, k)
    lap = -sum(float(v @ v) for v in a) * u
    m = len(g)
    for i in range(m):
        for j in range(i + 1, m):
            rest = np.ones_like(u)
            for l in range(m):
                if l != i and l != j:
                    rest = rest * g[l]
            lap = lap + 2.0 * float(a[i] @ a[j]) * dg[i] * dg[j] * rest
    lap = k * k * lap
    return lam * u - lap
