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
