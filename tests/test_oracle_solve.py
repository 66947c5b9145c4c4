"""Pins of oracle/mesh.py, operator.py, pcg.py, solve.py.

PAPER.md P:105-110 (gather/scatter), P:226-246 (Alg. 1), P:594-607 (CG and the
block preconditioner), SPEC S:224-235 (DOF counts, adjointness), S:351 (recovery
== full solve), S:418 (identity operator converges in one iteration).
"""
import numpy as np
import pytest

from oracle import basis, mesh, operator, pcg, solve
from synth import small_grid, sine_f, sine_u, lattice_random


def test_dof_counts_spec():
    g = small_grid(2, (1, 1, 1), 0.0)
    assert g.n_lattice == 27 and mesh.skeleton_mask(g).sum() == 26
    g = small_grid(3, (2, 2, 2), 0.0)
    assert mesh.skeleton_mask(g).sum() == 279
    assert g.n_skeleton() == 279


def test_gather_scatter_adjoint_and_multiplicity():
    g = small_grid(3, (3, 2, 2), 0.0)
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, g.n_lattice)
    Y = rng.uniform(-1, 1, ((g.p + 1) ** 3, g.n_elements))
    assert abs(np.sum(mesh.scatter(g, x) * Y) - np.dot(x, mesh.gather(g, Y))) < 1e-10
    mult = mesh.gather(g, mesh.scatter(g, np.ones(g.n_lattice)))
    gx, gy, gz = mesh.lattice_ijk(g)
    nx1, ny1, nz1 = mesh.lattice_dims(g)
    cnt = lambda c, n1: np.where((c % g.p == 0) & (c > 0) & (c < n1 - 1), 2, 1)
    assert np.array_equal(mult, cnt(gx, nx1) * cnt(gy, ny1) * cnt(gz, nz1))


def test_pcg_identity_one_iteration_and_dense_spd():
    b = np.random.default_rng(1).uniform(-1, 1, 40)
    r = pcg.pcg(lambda v: v.copy(), lambda v: v.copy(), b, rtol=1e-12)
    assert r.iters == 1 and r.converged and np.allclose(r.x, b)
    rng = np.random.default_rng(2)
    A = rng.uniform(-1, 1, (30, 30))
    A = A @ A.T + 30 * np.eye(30)
    r = pcg.pcg(lambda v: A @ v, lambda v: v / np.diag(A), b[:30], rtol=1e-13)
    assert r.converged and r.iters <= 31
    assert np.allclose(r.x, np.linalg.solve(A, b[:30]), atol=1e-10)


def test_pcg_breakdown_on_indefinite():
    A = np.diag([1.0, -1.0])
    r = pcg.pcg(lambda v: A @ v, lambda v: v.copy(), np.array([0.0, 1.0]))
    assert r.breakdown


@pytest.mark.parametrize("p,lam", [(3, 1.0), (4, 0.0)])
def test_condensed_solve_plus_recovery_equals_full_solve(p, lam):
    """SPEC S:351 / Alg. 1: interior recovery reproduces the uncondensed direct solve."""
    g = small_grid(p, (2, 2, 2), lam)
    X, Y, Z = mesh.lattice_coordinates(g)
    f = np.cos(X + 2 * Y) * np.exp(Z) + 1.0
    A, F, free = solve.full_system(g, f)
    ufull = np.zeros(g.n_lattice)
    ufull[free] = np.linalg.solve(A, F)
    op = operator.AssembledCondensedOperator(g)
    b = solve.condensed_rhs(op, f)
    fr = op.free
    Ac = np.stack([op.apply(np.eye(g.n_lattice)[i]) for i in np.nonzero(fr)[0]], axis=1)[fr]
    ub = np.zeros(g.n_lattice)
    ub[fr] = np.linalg.solve(Ac, b[fr])
    u = solve.recover(op, f, ub)
    assert np.abs(u - ufull).max() < 1e-11 * np.abs(ufull).max()


def test_assembled_operator_symmetric_spd_on_free_set():
    g = small_grid(3, (2, 2, 1), 0.0)
    op = operator.AssembledCondensedOperator(g)
    fr = np.nonzero(op.free)[0]
    A = np.stack([op.apply(np.eye(g.n_lattice)[i]) for i in fr], axis=1)[fr]
    assert np.allclose(A, A.T, atol=1e-12 * np.abs(A).max())
    assert np.linalg.eigvalsh(A).min() > 0


def test_apply_at_matches_apply():
    g = small_grid(4, (3, 2, 2), 0.5, lengths=(1.5, 1.0, 0.7))
    op = operator.AssembledCondensedOperator(g)
    x = lattice_random(7, g.ne, g.p).ravel()
    y = op.apply(x)
    tg = np.nonzero(op.free)[0][::13]
    assert np.allclose(op.apply_at(x, tg), y[tg], atol=1e-13 * np.abs(y).max())


def test_spectral_convergence_cfg1_like():
    """Manufactured sine on 2^3 elements, lambda=1 (BASELINE configs[0] family):
    nodal max error drops >= 10x per +1 in p (c9)."""
    errs = []
    for p in (2, 3, 4, 5, 6):
        g = small_grid(p, (2, 2, 2), 1.0)
        op = operator.AssembledCondensedOperator(g)
        X, Y, Z = mesh.lattice_coordinates(g)
        f = sine_f(X, Y, Z, 1.0)
        b = solve.condensed_rhs(op, f)
        P = solve.BlockJacobi(op)
        res = pcg.pcg(op.apply, P.apply, b, rtol=1e-12, norm=solve.transformed_norm(g, op.skel))
        assert res.converged
        u = solve.recover(op, f, res.x)
        errs.append(np.abs(u - sine_u(X, Y, Z)).max())
    errs = np.array(errs)
    assert np.all(errs[1:] < errs[:-1] / 10.0), errs
    assert errs[-1] < 1e-7


def test_block_jacobi_is_diagonal_in_transformed_system():
    """block preconditioning 'reduces to the application of a diagonal matrix in
    the transformed system' -- every assembled self-block is diagonal after Shat."""
    g = small_grid(4, (3, 2, 2), 0.3, lengths=(2.0, 1.0, 1.0))
    op = operator.AssembledCondensedOperator(g)
    P = solve.BlockJacobi(op)
    _, S = basis.interior_eigen(g.p)
    nx1, ny1, _ = mesh.lattice_dims(g)
    nI = g.p - 1
    for idx, Binv in P.diagonal_blocks():
        B = np.linalg.inv(Binv)
        m = len(idx)
        if m == 1:
            continue
        T = S if m == nI else np.kron(S, S)
        Bt = T @ B @ T.T
        assert np.abs(Bt - np.diag(np.diag(Bt))).max() < 1e-12 * np.abs(Bt).max()


def test_transform_roundtrip_and_duality():
    g = small_grid(5, (2, 3, 2), 0.0)
    skel = mesh.skeleton_mask(g)
    rng = np.random.default_rng(3)
    x = np.where(skel, rng.uniform(-1, 1, g.n_lattice), 0.0)
    y = np.where(skel, rng.uniform(-1, 1, g.n_lattice), 0.0)
    assert np.allclose(solve.transform(g, solve.transform(g, x, "dual"), "dual_inv"), x, atol=1e-13)
    assert np.allclose(solve.transform(g, solve.transform(g, x, "primal"), "primal_inv"), x, atol=1e-13)
    xt = solve.transform(g, x, "primal")
    yt = solve.transform(g, y, "dual")
    assert abs(np.dot(xt, yt) - np.dot(x, y)) < 1e-12 * g.n_lattice


def _assembled_dense(op):
    """The assembled condensed matrix by applying the oracle operator to unit vectors."""
    n = op.grid.n_lattice
    return np.stack([op.apply(np.eye(n)[i]) for i in range(n)], axis=1)


def test_transform_through_p2_closed_forms():
    """solve.transform pinned by the hand-derived p = 2 transformed entries (tests/golden/
    p2_single_element.txt): on a 2x2x2 grid of reference elements (h = 2,
    lambda = 0), the assembled transformed operator Shat A Shat^T, formed as
    transform(A transform(e, 'primal_inv'), 'dual'), has diagonal 2 x 41/18 at an interior face
    (2 elements), 4 x 1 at an interior edge, 8 x 7/18 at the centre vertex, and the face w -> face s
    coupling -2/9 (one element holds both).  A swapped primal / dual pair scales face entries by
    (S M)^2 / S^2 = 16/9 and fails."""
    from conftest import read_golden
    G = read_golden("p2_single_element.txt")
    g = small_grid(2, (2, 2, 2), 0.0, lengths=(4.0, 4.0, 4.0))
    op = operator.AssembledCondensedOperator(g)
    nx1, ny1, _ = mesh.lattice_dims(g)
    idx = lambda gx, gy, gz: gx + nx1 * (gy + ny1 * gz)

    def At(i, j):
        e = np.zeros(g.n_lattice)
        e[j] = 1.0
        return solve.transform(g, op.apply(solve.transform(g, e, "primal_inv")), "dual")[i]

    xface = idx(2, 1, 1)          # x-face fx = 1 of elements (0,0,0) | (1,0,0), node (j,k) = (1,1)
    yface = idx(1, 2, 1)          # y-face fy = 1 of elements (0,0,0) | (0,1,0)
    zedge = idx(2, 2, 1)          # z-edge (fx, fy) = (1, 1), layer 0: 4 elements
    vert = idx(2, 2, 2)           # centre vertex: 8 elements
    assert abs(At(xface, xface) - 2 * float(G["t_face_diag"])) < 1e-13
    assert abs(At(zedge, zedge) - 4 * float(G["t_edge_diag"])) < 1e-13
    assert abs(At(vert, vert) - 8 * float(G["t_vertex_diag"])) < 1e-13
    assert abs(At(xface, yface) - float(G["t_face_w_s"])) < 1e-13
    # transformed_norm: || Shat e || for a face unit vector is S_II^2 = 3/4 at p = 2
    norm = solve.transformed_norm(g, op.skel)
    e = np.zeros(g.n_lattice)
    e[xface] = 1.0
    assert abs(norm(e) - 0.75) < 1e-14
    e[xface] = 0.0
    e[zedge] = 1.0
    assert abs(norm(e) - np.sqrt(0.75)) < 1e-14


def test_block_jacobi_blocks_are_assembled_diagonal_blocks():
    """BlockJacobi pinned against the explicitly assembled condensed matrix: every block is the
    inverse of the assembled matrix restricted to one face / edge / vertex, the blocks
    partition the free skeleton nodes, and a block that dropped a neighbour element's
    contribution would differ from the assembled entries (non-uniform widths make the
    contributions of the elements around an entity differ)."""
    g = small_grid(3, (3, 2, 2), 0.4, lengths=(1.5, 1.0, 0.8))
    g.hx = np.array([0.3, 0.7, 0.5])
    g.hz = np.array([0.35, 0.45])
    op = operator.AssembledCondensedOperator(g)
    A = _assembled_dense(op)
    P = solve.BlockJacobi(op)
    seen = np.zeros(g.n_lattice, dtype=int)
    for idx, Binv in P.diagonal_blocks():
        B = A[np.ix_(idx, idx)]
        assert np.allclose(np.linalg.inv(Binv), B, rtol=0, atol=1e-12 * np.abs(B).max())
        seen[idx] += 1
    assert np.array_equal(seen, op.free.astype(int))


def test_multi_geometry_grouping_recovery_equals_full_solve():
    """Non-uniform widths (several Schur matrices, operator.py's np.unique grouping over
    mesh.element_widths): condensed solve + interior recovery equals the uncondensed direct
    solve, and the operator equals the dense assembly of per-element full matrices
    condensed one element at a time."""
    g = small_grid(3, (3, 2, 2), 0.7)
    g.hx = np.array([0.2, 0.5, 0.3])
    g.hy = np.array([0.6, 0.4])
    g.hz = np.array([0.25, 0.75])
    w = mesh.element_widths(g)
    assert w.shape == (12, 3)
    assert np.allclose(w[1 + 3 * (0 + 2 * 1)], (0.5, 0.6, 0.75))       # e = ex + nx (ey + ny ez)
    op = operator.AssembledCondensedOperator(g)
    assert len(op.groups) == 12
    X, Y, Z = mesh.lattice_coordinates(g)
    f = np.sin(3 * X + Y) * np.cos(2 * Z) + 0.5
    A, F, free = solve.full_system(g, f)
    ufull = np.zeros(g.n_lattice)
    ufull[free] = np.linalg.solve(A, F)
    b = solve.condensed_rhs(op, f)
    fr = op.free
    Ac = _assembled_dense(op)[np.ix_(fr, fr)]
    ub = np.zeros(g.n_lattice)
    ub[fr] = np.linalg.solve(Ac, b[fr])
    u = solve.recover(op, f, ub)
    assert np.abs(u - ufull).max() < 1e-11 * np.abs(ufull).max()


def test_assembled_diagonal_p2_closed_forms_and_dense():
    """solve.assembled_diagonal (solver DC) pinned by the hand-derived nodal p = 2 Schur
    diagonal (tests/golden/p2_single_element.txt): on a 2x2x2 grid of reference elements an interior
    face sums 2 x 328/81, an interior edge 4 x 4/3, the centre vertex 8 x 7/18; and on a non-uniform
    grid it equals the diagonal of the explicitly assembled matrix (a dropped neighbour fails)."""
    from conftest import read_golden
    G = read_golden("p2_single_element.txt")
    g = small_grid(2, (2, 2, 2), 0.0, lengths=(4.0, 4.0, 4.0))
    op = operator.AssembledCondensedOperator(g)
    d = solve.assembled_diagonal(op)
    nx1, ny1, _ = mesh.lattice_dims(g)
    idx = lambda gx, gy, gz: gx + nx1 * (gy + ny1 * gz)
    assert abs(d[idx(2, 1, 1)] - 2 * float(G["schur_face_diag"])) < 1e-13
    assert abs(d[idx(2, 2, 1)] - 4 * float(G["schur_edge_diag"])) < 1e-13
    assert abs(d[idx(2, 2, 2)] - 8 * float(G["schur_vertex_diag"])) < 1e-13
    assert d[idx(0, 1, 1)] == 0.0                 # Dirichlet face node
    g = small_grid(3, (3, 2, 2), 0.4, lengths=(1.5, 1.0, 0.8))
    g.hx = np.array([0.3, 0.7, 0.5])
    g.hz = np.array([0.35, 0.45])
    op = operator.AssembledCondensedOperator(g)
    A = _assembled_dense(op)
    ref = np.where(op.free, np.diag(A), 0.0)
    assert np.allclose(solve.assembled_diagonal(op), ref, rtol=0, atol=1e-13 * np.abs(ref).max())
