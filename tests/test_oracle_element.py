"""Pins of oracle/element.py: metric coefficients, element matrix, Schur complement.

PAPER.md P:125-137 (Eq. eq:helmholtz_operator, eq:metriccoeffelement),
P:198-225 (static condensation), P:406-440 (transformed system, Table 2).
"""
import itertools
import math

import numpy as np
import pytest

from oracle import basis, element
from conftest import read_golden

P2 = read_golden("p2_single_element.txt")


def test_metric_coefficients_spec_examples():
    # SPEC S:206-208
    assert np.allclose(element.metric_coefficients((2, 2, 2), 0.0), [0, 1, 1, 1])
    assert np.allclose(element.metric_coefficients((2, 2, 2), math.pi), [math.pi, 1, 1, 1])
    assert np.allclose(element.metric_coefficients((1, 2, 4), 0.0), [0, 4, 1, 0.25])
    with pytest.raises(ValueError):
        element.metric_coefficients((1, 1, 1), -1.0)
    with pytest.raises(ValueError):
        element.metric_coefficients((1, 0, 1), 1.0)


def _element_matrix_by_quadrature(p, h, lam):
    """Brute-force definition: H[a,b] = sum_q W_q J (lam phi_a phi_b + sum_d (2/h_d)^2 d_d phi_a d_d phi_b)
    over the 3-D GLL points q (nodal basis: phi_a(q) = delta_aq), loop form."""
    x, w = basis.gll(p)
    Dm = basis.lagrange_derivative_matrix(x)       # Dm[q, a] = phi_a'(x_q)
    n = p + 1
    J = h[0] * h[1] * h[2] / 8.0
    idx = lambda i, j, k: i + n * j + n * n * k
    H = np.zeros((n ** 3, n ** 3))
    nodes = list(itertools.product(range(n), repeat=3))
    for (qk, qj, qi) in nodes:
        W = w[qi] * w[qj] * w[qk] * J
        for (ak, aj, ai) in nodes:
            va = 1.0 if (ai, aj, ak) == (qi, qj, qk) else 0.0
            ga = (Dm[qi, ai] * (aj == qj) * (ak == qk) * 2 / h[0],
                  Dm[qj, aj] * (ai == qi) * (ak == qk) * 2 / h[1],
                  Dm[qk, ak] * (ai == qi) * (aj == qj) * 2 / h[2])
            if va == 0.0 and ga == (0.0, 0.0, 0.0):
                continue
            for (bk, bj, bi) in nodes:
                vb = 1.0 if (bi, bj, bk) == (qi, qj, qk) else 0.0
                gb = (Dm[qi, bi] * (bj == qj) * (bk == qk) * 2 / h[0],
                      Dm[qj, bj] * (bi == qi) * (bk == qk) * 2 / h[1],
                      Dm[qk, bk] * (bi == qi) * (bj == qj) * 2 / h[2])
                H[idx(ai, aj, ak), idx(bi, bj, bk)] += W * (lam * va * vb + sum(a * b for a, b in zip(ga, gb)))
    return H


@pytest.mark.parametrize("p,h,lam", [(2, (2.0, 2.0, 2.0), 0.0), (2, (0.5, 1.3, 2.2), 1.7), (3, (0.7, 0.4, 1.9), 3.1)])
def test_element_matrix_vs_quadrature_definition(p, h, lam):
    """Pins the Kronecker order (rightmost factor = x) and the metric scaling."""
    H = element.element_matrix(p, element.metric_coefficients(h, lam), sparse=False)
    Href = _element_matrix_by_quadrature(p, h, lam)
    assert np.allclose(H, Href, atol=1e-12 * np.abs(Href).max())


@pytest.mark.parametrize("p", [2, 4, 7])
def test_element_matrix_constant_nullspace(p):
    H = element.element_matrix(p, element.metric_coefficients((0.3, 0.9, 0.5), 0.0), sparse=False)
    assert np.abs(H @ np.ones(H.shape[0])).max() < 1e-11 * np.abs(H).max()


def _loc(ce, p, i, j, k):
    return int(np.nonzero(ce.bidx == element.local_index(p, i, j, k))[0][0])


def test_schur_p2_closed_forms():
    ce = element.CondensedElement(2, element.metric_coefficients((2, 2, 2), 0.0))
    Hh = ce.explicit()
    L = lambda i, j, k: _loc(ce, 2, i, j, k)
    assert abs(Hh[L(0, 1, 1), L(0, 1, 1)] - float(P2["schur_face_diag"])) < 1e-13
    assert abs(Hh[L(0, 1, 1), L(2, 1, 1)] - float(P2["schur_face_w_e"])) < 1e-13
    assert abs(Hh[L(0, 1, 1), L(1, 0, 1)] - float(P2["schur_face_w_s"])) < 1e-13
    assert abs(Hh[L(0, 0, 1), L(0, 0, 1)] - float(P2["schur_edge_diag"])) < 1e-13
    assert abs(Hh[L(0, 0, 0), L(0, 0, 0)] - float(P2["schur_vertex_diag"])) < 1e-13
    # interior block of H itself
    H = element.element_matrix(2, [0, 1, 1, 1], sparse=False)
    c = element.local_index(2, 1, 1, 1)
    assert abs(H[c, c] - float(P2["H_II"])) < 1e-13


@pytest.mark.parametrize("p,h,lam", [(3, (0.7, 0.4, 1.9), 3.1), (4, (1.0, 1.0, 1.0), 0.0), (5, (0.2, 0.2, 3.0), 1.0)])
def test_schur_symmetry_definiteness_nullspace(p, h, lam):
    ce = element.CondensedElement(p, element.metric_coefficients(h, lam))
    Hh = ce.explicit()
    assert np.allclose(Hh, Hh.T, atol=1e-12 * np.abs(Hh).max())
    ev = np.linalg.eigvalsh(Hh)
    if lam > 0:
        assert ev.min() > 0
    else:
        # single element, lambda = 0: constants are the (only) null space
        assert abs(ev[0]) < 1e-10 * ev[-1] and ev[1] > 1e-8 * ev[-1]
        assert np.abs(Hh @ np.ones(len(Hh))).max() < 1e-10 * np.abs(Hh).max()


@pytest.mark.parametrize("p", [2, 3, 5])
def test_schur_equals_inverse_of_inverse_block(p):
    """Schur complement identity ((H^{-1})_BB)^{-1} = H_BB - H_BI H_II^{-1} H_IB (lambda > 0)."""
    d = element.metric_coefficients((0.6, 1.1, 0.8), 2.0)
    ce = element.CondensedElement(p, d)
    H = element.element_matrix(p, d, sparse=False)
    Hinv = np.linalg.inv(H)
    ref = np.linalg.inv(Hinv[np.ix_(ce.bidx, ce.bidx)])
    assert np.allclose(ce.explicit(), ref, atol=1e-9 * np.abs(ref).max())


def test_schur_apply_matches_explicit_and_large_p_path():
    d = element.metric_coefficients((0.5, 0.5, 0.5), 1.0)
    for p in (6, 17):
        ce = element.CondensedElement(p, d)
        X = np.random.default_rng(p).uniform(-1, 1, (len(ce.bidx), 3))
        Y = ce.apply(X)
        if p == 6:
            assert np.allclose(Y, ce.explicit() @ X, atol=1e-12 * np.abs(Y).max())
        # symmetry of the operator form: x^T (A y) = y^T (A x)
        assert abs(X[:, 0] @ Y[:, 1] - X[:, 1] @ Y[:, 0]) < 1e-11 * np.abs(Y).max() * len(X)


def _transform_element(p, Hh, bidx):
    """T_BB Hh T_BB^T with T = S(x)S(x)S, S = diag(1, S_II, 1)."""
    _, S_II = basis.interior_eigen(p)
    S = np.eye(p + 1)
    S[1:p, 1:p] = S_II
    T = np.kron(S, np.kron(S, S))
    TBB = T[np.ix_(bidx, bidx)]
    return TBB @ Hh @ TBB.T


def test_transformed_p2_closed_forms():
    ce = element.CondensedElement(2, element.metric_coefficients((2, 2, 2), 0.0))
    Ht = _transform_element(2, ce.explicit(), ce.bidx)
    L = lambda i, j, k: _loc(ce, 2, i, j, k)
    assert abs(Ht[L(0, 1, 1), L(0, 1, 1)] - float(P2["t_face_diag"])) < 1e-13
    assert abs(Ht[L(0, 1, 1), L(2, 1, 1)] - float(P2["t_face_w_e"])) < 1e-13
    assert abs(Ht[L(0, 1, 1), L(1, 0, 1)] - float(P2["t_face_w_s"])) < 1e-13
    assert abs(Ht[L(0, 0, 1), L(0, 0, 1)] - float(P2["t_edge_diag"])) < 1e-13
    assert abs(Ht[L(0, 0, 0), L(0, 0, 0)] - float(P2["t_vertex_diag"])) < 1e-13


@pytest.mark.parametrize("p", [3, 5, 6])
def test_transformed_structure_table2(p):
    """Paper claims checked on the dense oracle:
    the face self-blocks of the transformed condensed operator are diagonal (Eq. 26 plus
    the rank-1 condensed part), and opposite faces couple diagonally."""
    ce = element.CondensedElement(p, element.metric_coefficients((0.4, 0.9, 1.3), 0.7))
    Ht = _transform_element(p, ce.explicit(), ce.bidx)
    n = p + 1
    bl = ce.bidx
    i, j, k = bl % n, (bl // n) % n, bl // (n * n)
    inner = lambda a: (a > 0) & (a < p)
    w_face = np.nonzero((i == 0) & inner(j) & inner(k))[0]
    e_face = np.nonzero((i == p) & inner(j) & inner(k))[0]
    blk = Ht[np.ix_(w_face, w_face)]
    assert np.abs(blk - np.diag(np.diag(blk))).max() < 1e-12 * np.abs(blk).max()
    blk = Ht[np.ix_(w_face, e_face)]
    assert np.abs(blk - np.diag(np.diag(blk))).max() < 1e-12 * np.abs(Ht).max()


def test_edges_do_not_couple_to_interior():
    """Only faces map into the element interior (diagonal mass)."""
    p = 5
    ce = element.CondensedElement(p, element.metric_coefficients((0.4, 0.9, 1.3), 0.7))
    n = p + 1
    bl = ce.bidx
    i, j, k = bl % n, (bl // n) % n, bl // (n * n)
    onb = lambda a: (a == 0) | (a == p)
    edge_or_vertex = (onb(i).astype(int) + onb(j) + onb(k)) >= 2
    assert np.abs(ce.H_IB.toarray()[:, edge_or_vertex]).max() == 0.0
