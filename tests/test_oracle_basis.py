"""Pins of oracle/basis.py against closed forms and an independent construction.

PAPER.md P:119-123 (M, K definitions), P:156-158 (GLL nodal basis, lumped
mass), P:302 (generalized eigenproblem).
"""
import math

import numpy as np
import pytest
from numpy.polynomial import Polynomial

from oracle import basis
from conftest import read_golden

G = read_golden("basis_1d.txt")


def test_gll_closed_forms():
    x, w = basis.gll(1)
    assert np.allclose(x, [-1, 1], atol=0) and np.allclose(w, [1, 1], atol=0)
    x, w = basis.gll(2)
    assert np.allclose(x, [-1, 0, 1], atol=1e-16)
    assert np.allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=1e-15)
    x, w = basis.gll(3)
    assert np.allclose(x, G["p3_nodes"], atol=1e-15)
    assert np.allclose(w, [float(v) for v in G["p3_weights"]], rtol=1e-14)
    x, w = basis.gll(4)
    assert np.allclose(x, G["p4_nodes"], atol=1e-15)
    assert np.allclose(w, [float(v) for v in G["p4_weights"]], rtol=1e-14)


@pytest.mark.parametrize("p", [2, 5, 8, 13, 16, 24, 32])
def test_gll_quadrature_exactness(p):
    """GLL with p+1 points integrates degree <= 2p-1 exactly, and not degree 2p."""
    x, w = basis.gll(p)
    assert abs(w.sum() - 2.0) < 1e-13
    assert np.allclose(x, -x[::-1], atol=1e-15)
    rng = np.random.default_rng(p)
    for deg in (2 * p - 1, 2 * p - 2, p):
        c = rng.uniform(-1, 1, deg + 1)
        P = Polynomial(c)
        exact = P.integ()(1.0) - P.integ()(-1.0)
        assert abs(np.dot(w, P(x)) - exact) < 1e-12 * max(1.0, np.abs(c).sum())
    # degree 2p is NOT integrated exactly: the Lobatto sum of L_p^2 is 2/p, the integral 2/(2p+1)
    Lp = np.polynomial.legendre.Legendre.basis(p)
    assert abs(np.dot(w, Lp(x) ** 2) - 2.0 / p) < 1e-12


@pytest.mark.parametrize("p", [1, 2, 3, 6, 11, 17])
def test_derivative_matrix_exact_on_polynomials(p):
    x, _ = basis.gll(p)
    Dm = basis.lagrange_derivative_matrix(x)
    P = Polynomial(np.random.default_rng(1).uniform(-1, 1, p + 1))
    assert np.allclose(Dm @ P(x), P.deriv()(x), atol=1e-11 * p * p)


def test_stiffness_closed_forms():
    _, _, K = basis.mass_stiffness(1)
    assert np.allclose(K, [[0.5, -0.5], [-0.5, 0.5]], atol=1e-16)
    _, _, K = basis.mass_stiffness(2)
    assert np.allclose(K * 6, [[7, -8, 1], [-8, 16, -8], [1, -8, 7]], atol=1e-13)
    assert abs(K[1, 1] - 8 / 3) < 1e-14


@pytest.mark.parametrize("p", [2, 3, 4, 7, 10, 16])
def test_stiffness_vs_independent_integration(p):
    """K_ij = int phi_i' phi_j' with phi_i = prod (x-x_m)/(x_i-x_m) built as numpy
    polynomials and integrated by Gauss-Legendre (exact for degree 2p-2)."""
    x, _, K = basis.mass_stiffness(p)
    gx, gw = np.polynomial.legendre.leggauss(p + 2)
    dphi = []
    for i in range(p + 1):
        others = np.delete(x, i)
        phi = Polynomial.fromroots(others) / np.prod(x[i] - others)
        dphi.append(phi.deriv()(gx))
    dphi = np.array(dphi)
    Kref = (dphi * gw[None, :]) @ dphi.T
    assert np.allclose(K, Kref, atol=1e-11 * p ** 2)
    assert np.allclose(K.sum(axis=1), 0.0, atol=1e-11 * p ** 2)
    assert np.allclose(K, K.T, atol=0)
    # reflection symmetry K_{ij} = K_{p-i, p-j}
    assert np.allclose(K, K[::-1, ::-1], atol=1e-11 * p ** 2)


def test_interior_eigen_closed_forms():
    for p, key in ((2, "p2_lambda"), (3, "p3_lambda"), (4, "p4_lambda")):
        lam, S = basis.interior_eigen(p)
        assert np.allclose(lam, G[key], rtol=1e-13)
    _, S = basis.interior_eigen(2)
    assert abs(abs(S[0, 0]) - math.sqrt(3) / 2) < 1e-15


@pytest.mark.parametrize("p", [2, 3, 5, 8, 16, 32])
def test_interior_eigen_invariants(p):
    x, w, K = basis.mass_stiffness(p)
    lam, S = basis.interior_eigen(p)
    MII = np.diag(w[1:p])
    KII = K[1:p, 1:p]
    scale = lam.max()
    assert np.allclose(S @ MII @ S.T, np.eye(p - 1), atol=1e-12)
    assert np.allclose(S @ KII @ S.T, np.diag(lam), atol=1e-12 * scale)
    assert np.all(np.diff(lam) > 0) and lam[0] > 0
    a0 = S @ K[1:p, 0]
    assert np.all(a0 > 0)                                   # SURVEY c2 sign rule
    if p >= 8:
        assert abs(lam[0] - G["lambda1_limit"]) < 1e-6
