"""Pins of the inhomogeneous-Dirichlet pipeline (the paper's solver benchmark E3):
oracle/solve.py dirichlet_rhs + recover(dirichlet=...), and the E3 inputs in synth/.

* the condensed solve with Dirichlet data + interior recovery equals the uncondensed direct
  solve u_F = A_FF^{-1} (F_F - A_FD g_D) of the assembled element matrices (S:351 generalised);
* e3_f = lambda u - Laplace(u) of Eq. eq:solution against 4th-order finite differences of e3_u;
* graded widths: expansion factor alpha, AR_max = alpha^7 on 8 elements.
"""
import numpy as np
import pytest

from oracle import element, mesh, operator, pcg, solve
from synth import small_grid, e3_grid, e3_u, e3_f, graded_widths


def _dense_dirichlet_solve(g, f, gval):
    """Uncondensed SEM system with u = g on the domain boundary, by dense assembly."""
    G = mesh.element_global_indices(g)
    N = g.n_lattice
    A = np.zeros((N, N))
    widths = mesh.element_widths(g)
    for e in range(g.n_elements):
        H = element.element_matrix(g.p, element.metric_coefficients(widths[e], g.lam), sparse=False)
        A[np.ix_(G[e], G[e])] += H
    F = mesh.gather(g, solve.element_load(g, f), G)
    D = mesh.dirichlet_mask(g)
    Fr = ~D
    u = np.where(D, gval, 0.0)
    u[Fr] = np.linalg.solve(A[np.ix_(Fr, Fr)], F[Fr] - A[np.ix_(Fr, D)] @ gval[D])
    return u


@pytest.mark.parametrize("p,alpha,lam", [(3, 2.0, 0.0), (4, 1.5, 0.3)])
def test_dirichlet_condensed_solve_equals_full_solve(p, alpha, lam):
    g = e3_grid(p, alpha, n=3, lam=lam)
    X, Y, Z = mesh.lattice_coordinates(g)
    k = 0.7
    f = e3_f(X, Y, Z, lam, k=k)
    gval = e3_u(X, Y, Z, k=k)
    u_ref = _dense_dirichlet_solve(g, f, gval)
    op = operator.AssembledCondensedOperator(g)
    b = solve.dirichlet_rhs(op, f, gval)
    fr = op.free
    n = g.n_lattice
    Ac = np.stack([op.apply(np.eye(n)[i]) for i in np.nonzero(fr)[0]], axis=1)[fr]
    ub = np.zeros(n)
    ub[fr] = np.linalg.solve(Ac, b[fr])
    u = solve.recover(op, f, ub, dirichlet=gval)
    assert np.abs(u - u_ref).max() < 1e-11 * np.abs(u_ref).max()
    # a solve that ignores the lifting is visibly wrong (the pin discriminates)
    b0 = solve.condensed_rhs(op, f)
    ub0 = np.zeros(n)
    ub0[fr] = np.linalg.solve(Ac, b0[fr])
    assert np.abs(solve.recover(op, f, ub0, dirichlet=gval) - u_ref).max() > 1e-3 * np.abs(u_ref).max()


def test_e3_rhs_matches_finite_differences():
    rng = np.random.default_rng(0)
    P = rng.uniform(0.3, 2 * np.pi - 0.3, (3, 40))
    h = 1e-3
    lap = np.zeros(P.shape[1])
    for d in range(3):
        e = np.zeros((3, 1))
        e[d] = h
        u = lambda s: e3_u(*(P + s * e))
        lap += (-u(2) + 16 * u(1) - 30 * u(0) + 16 * u(-1) - u(-2)) / (12 * h * h)
    lam = 0.4
    f = e3_f(*P, lam)
    ref = lam * e3_u(*P) - lap
    assert np.abs(f - ref).max() < 2e-5 * np.abs(ref).max()


def test_graded_widths_expansion_factor():
    for alpha, ar in ((1.0, 1.0), (1.5, 1.5 ** 7), (2.0, 128.0)):
        w = graded_widths(8, alpha, 2 * np.pi)
        assert abs(w.sum() - 2 * np.pi) < 1e-14
        assert np.allclose(w[1:] / w[:-1], alpha)
        assert abs(w.max() / w.min() - ar) < 1e-9 * ar
    assert abs(1.5 ** 7 - 17.0859375) < 1e-12      # "AR_max ~ 17"


def test_e3_dirichlet_spectral_convergence():
    """Alg. 1 with Dirichlet data on a 2^3 graded grid: the nodal max error against u_ex drops
    geometrically in p (smooth k = 0.5 variant of Eq. eq:solution)."""
    errs = []
    for p in (3, 4, 5, 6, 7):
        g = e3_grid(p, 1.5, n=2, lam=0.0)
        X, Y, Z = mesh.lattice_coordinates(g)
        f = e3_f(X, Y, Z, 0.0, k=0.5)
        gval = e3_u(X, Y, Z, k=0.5)
        op = operator.AssembledCondensedOperator(g)
        b = solve.dirichlet_rhs(op, f, gval)
        P = solve.BlockJacobi(op)
        res = pcg.pcg(op.apply, P.apply, b, rtol=1e-13, norm=solve.transformed_norm(g, op.skel))
        assert res.converged
        u = solve.recover(op, f, res.x, dirichlet=gval)
        errs.append(np.abs(u - gval).max())
    errs = np.array(errs)
    # measured 0.69, 0.24, 0.11, 0.044, 0.016 (p = 3..7): every step >= 2x, overall >= 40x
    assert np.all(errs[1:] < errs[:-1] / 2.0), errs
    assert errs[-1] < errs[0] / 40.0, errs
