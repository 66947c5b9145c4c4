"""Every p <= 8 operator family against the oracle, each selected explicitly (SC_OP) and checked to be
the one that ran (sc_operator_kernel): v6 (halo-recompute tile columns, uniform class lanes, both
tile heights), v3 (tile columns with look-back), rw (row-warp p = 3, 4).  Multi-tile ragged grids,
z-segments, z-slab ranks, PCG with the fused p . q partials, bitwise repeatability."""
import numpy as np
import pytest
import torch

from oracle import operator, pcg, solve
from synth import small_grid, lattice_random

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()
    assert torch.cuda.is_available()


def _ctx(g, monkeypatch, op, h=None, **kw):
    from paper_1601_08179_b200 import Context
    monkeypatch.setenv("SC_OP", op)
    if h is not None:
        monkeypatch.setenv("SC_V6_H", str(h))
    ctx = Context(g.p, g.ne, (g.hx, g.hy, g.hz), g.lam, device=0, **kw)
    want = {"v6": "v6h8" if h == 8 else "v6", "v3": "v3", "rw": "rw", "v7": "v7"}[op]
    assert ctx.operator_kernel() == want, (ctx.operator_kernel(), want)
    return ctx


def _apply_nodal(ctx, x_lat):
    from paper_1601_08179_b200 import SC_PRIMAL, SC_DUAL
    xt = ctx.skeleton()
    ctx.sc_to_transformed(torch.from_numpy(np.ascontiguousarray(x_lat)).cuda(), xt, SC_PRIMAL)
    yt = ctx.skeleton()
    ctx.sc_apply_condensed(xt, yt)
    y = ctx.lattice()
    ctx.sc_from_transformed(yt, y, SC_DUAL)
    return y.cpu().numpy()


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


CASES = [(3, (17, 9, 3), "rw", None), (3, (17, 9, 3), "v6", None), (4, (9, 8, 3), "rw", None),
         (4, (9, 8, 3), "v6", None), (5, (15, 7, 3), "v6", None), (5, (15, 7, 3), "v3", None),
         (6, (9, 10, 2), "v6", None), (7, (16, 4, 3), "v6", None), (7, (16, 4, 3), "v3", None),
         (8, (9, 7, 3), "v6", None), (8, (9, 7, 3), "v3", None), (7, (8, 15, 2), "v6", 8),
         (5, (15, 16, 2), "v6", 8)]


@pytest.mark.parametrize("p,ne,op,h", CASES)
def test_family_operator_parity(p, ne, op, h, monkeypatch):
    g = small_grid(p, ne, 0.7, lengths=(1.2, 0.9, 0.6))
    ref_op = operator.AssembledCondensedOperator(g)
    x = lattice_random(90 + p, g.ne, g.p).ravel()
    ctx = _ctx(g, monkeypatch, op, h)
    assert _rel(_apply_nodal(ctx, x), ref_op.apply(x)) <= 1e-12


@pytest.mark.parametrize("p,ne,op,h,zseg", [(6, (10, 5, 7), "v6", None, "3"), (7, (9, 8, 6), "v6", 8, "2"),
                                             (8, (9, 4, 7), "v6", None, "4")])
def test_family_zsegments(p, ne, op, h, zseg, monkeypatch):
    monkeypatch.setenv("SC_ZSEG", zseg)
    g = small_grid(p, ne, 0.5, lengths=(1.1, 0.8, 1.3))
    ref_op = operator.AssembledCondensedOperator(g)
    x = lattice_random(7, g.ne, g.p).ravel()
    ctx = _ctx(g, monkeypatch, op, h)
    assert _rel(_apply_nodal(ctx, x), ref_op.apply(x)) <= 1e-12


@pytest.mark.parametrize("p,ne,op,h", [(5, (15, 7, 4), "v6", None), (8, (10, 6, 3), "v6", None),
                                       (7, (9, 9, 3), "v6", 8), (8, (10, 6, 3), "v3", None)])
def test_family_pcg_fused_dot(p, ne, op, h, monkeypatch):
    """BT-PCG with p . q from the operator's per-CTA x . A x partials (the default)."""
    from paper_1601_08179_b200 import SC_DUAL
    g = small_grid(p, ne, 1.0, lengths=(1.3, 0.7, 0.5))
    ref_op = operator.AssembledCondensedOperator(g)
    ctx = _ctx(g, monkeypatch, op, h)
    bt = ctx.skeleton()
    ctx.sc_fill_random(8, bt)
    lat = ctx.lattice()
    ctx.sc_from_transformed(bt, lat, SC_DUAL)
    b = lat.cpu().numpy()
    P = solve.BlockJacobi(ref_op)
    norm = solve.transformed_norm(g, ref_op.skel)
    res = pcg.pcg(ref_op.apply, P.apply, b, rtol=1e-10, norm=norm)
    xt = ctx.skeleton()
    rep = ctx.sc_pcg_solve(bt, xt, rtol=1e-10, maxit=2000)
    assert rep.converged and abs(rep.iters - res.iters) <= 1, (rep.iters, res.iters)
    ref = res.x if rep.iters == res.iters else pcg.pcg(ref_op.apply, P.apply, b, rtol=0, norm=norm,
                                                       fixed_iters=rep.iters).x
    assert _rel(ctx.to_lattice_nodal(xt).cpu().numpy(), ref) <= 1e-10


@pytest.mark.parametrize("p,ne,R,h", [(6, (9, 5, 5), 2, None), (7, (10, 7, 6), 3, None), (5, (9, 10, 5), 2, 8)])
def test_family_v6_slab_ranks(p, ne, R, h, monkeypatch):
    """z-slab ranks (SC_TEST_LOCAL_SLAB: local partial sums on the interface planes) against the
    oracle's slab operator with non-Dirichlet interface planes."""
    import copy
    monkeypatch.setenv("SC_TEST_LOCAL_SLAB", "1")
    g = small_grid(p, ne, 0.9, lengths=(1.2, 0.8, 1.1))
    for r in range(R):
        ctx = _ctx(g, monkeypatch, "v6", h, rank=r, nranks=R)
        z0, z1 = ctx.layout.z_begin, ctx.layout.z_end
        gs = copy.deepcopy(g)
        gs.ne = (g.ne[0], g.ne[1], z1 - z0)
        gs.hz = g.hz[z0:z1]
        gs.extra = dict(g.extra, dirichlet_z=(r == 0, r == R - 1))
        xg = lattice_random(70 + p, g.ne, g.p)
        xs = np.ascontiguousarray(xg[z0 * p:z1 * p + 1])
        ref = operator.AssembledCondensedOperator(gs).apply(xs.ravel())
        assert _rel(_apply_nodal(ctx, xs.ravel()), ref) <= 1e-12, (r, z0, z1)


@pytest.mark.parametrize("h", [None, 8])
def test_family_v6_bitwise_repeatable(h, monkeypatch):
    g = small_grid(7, (30, 13, 9), 1.0)
    ctx = _ctx(g, monkeypatch, "v6", h)
    x = ctx.skeleton()
    ctx.sc_fill_random(3, x)
    y0 = ctx.skeleton()
    ctx.sc_apply_condensed(x, y0)
    for _ in range(4):
        y = ctx.skeleton(fill=float("nan"))
        ctx.sc_apply_condensed(x, y)
        torch.cuda.synchronize()
        assert torch.equal(y, y0)


@pytest.mark.parametrize("ne,lam", [((2, 2, 2), 1.0), ((37, 5, 4), 0.3), ((33, 32, 3), 0.0), ((1, 1, 3), 1.0)])
def test_p2_owner_stencil(ne, lam, monkeypatch):
    """p = 2 owner-computes stencil (kernels_p2s.cu, the default on one rank) against the oracle and
    against the colour-scheduled kernel (SC_P2_COLOUR=1); every entry written once (stale y
    overwritten, padding 0), repeated applications bitwise equal."""
    from paper_1601_08179_b200 import Context
    g = small_grid(2, ne, lam, lengths=(1.3, 0.9, 0.7))
    x = lattice_random(33, g.ne, g.p).ravel()
    ctx = Context(g.p, g.ne, (g.hx, g.hy, g.hz), g.lam, device=0)
    assert ctx.operator_kernel() == "p2s"
    ref = operator.AssembledCondensedOperator(g).apply(x)
    assert _rel(_apply_nodal(ctx, x), ref) <= 1e-12
    xt = ctx.skeleton()
    ctx.sc_fill_random(4, xt)
    y1 = ctx.skeleton(fill=float("nan"))
    ctx.sc_apply_condensed(xt, y1)
    y2 = ctx.skeleton(fill=5.0)
    ctx.sc_apply_condensed(xt, y2)
    assert torch.equal(y1, y2)
    monkeypatch.setenv("SC_P2_COLOUR", "1")
    ctx2 = Context(g.p, g.ne, (g.hx, g.hy, g.hz), g.lam, device=0)
    assert ctx2.operator_kernel() == "p2"
    y3 = ctx2.skeleton()
    ctx2.sc_apply_condensed(xt, y3)
    assert (y1 - y3).norm() <= 1e-13 * y3.norm()


V7_CASES = [(3, (1, 1, 1)), (8, (1, 1, 1)), (4, (40, 1, 1)), (6, (1, 37, 2)), (16, (1, 1, 3)), (3, (17, 9, 3)), (4, (9, 8, 3)), (5, (15, 7, 3)), (6, (9, 10, 2)), (7, (16, 4, 3)), (8, (9, 7, 3)),
            (8, (33, 5, 4)), (8, (1, 1, 2)), (5, (2, 17, 3)), (9, (9, 4, 3)), (10, (5, 3, 3)), (11, (3, 4, 2)),
            (12, (4, 3, 2)), (13, (3, 2, 3)), (14, (2, 3, 2)), (15, (3, 2, 2)), (16, (2, 3, 2)), (18, (3, 2, 2)),
            (24, (2, 2, 2))]


@pytest.mark.parametrize("p,ne", V7_CASES)
def test_family_v7_operator_parity(p, ne, monkeypatch):
    """v7 (two passes: unassembled condensed part, then entity-wise assembly + primary part) against
    the oracle on ragged multi-run grids; every entry overwritten (stale y), repeatable bitwise."""
    g = small_grid(p, ne, 0.7, lengths=(1.2, 0.9, 0.6))
    ref_op = operator.AssembledCondensedOperator(g)
    x = lattice_random(90 + p, g.ne, g.p).ravel()
    ctx = _ctx(g, monkeypatch, "v7")
    y, ref = _apply_nodal(ctx, x), ref_op.apply(x)
    if np.linalg.norm(ref) == 0.0:   # a single element: every skeleton entity is Dirichlet
        assert np.linalg.norm(y) == 0.0
    else:
        assert _rel(y, ref) <= 1e-12
    xt = ctx.skeleton()
    ctx.sc_fill_random(2, xt)
    y1 = ctx.skeleton(fill=float("nan"))
    ctx.sc_apply_condensed(xt, y1)
    y2 = ctx.skeleton(fill=3.0)
    ctx.sc_apply_condensed(xt, y2)
    assert torch.equal(y1, y2)


@pytest.mark.parametrize("p,ne,R,z", [(8, (9, 5, 5), 2, None), (5, (10, 7, 6), 3, "2"), (3, (17, 4, 4), 2, None),
                                      (12, (3, 2, 4), 2, "1"), (7, (9, 4, 9), 3, "2")])
def test_family_v7_slab_ranks(p, ne, R, z, monkeypatch):
    """v7 on z-slab ranks (SC_TEST_LOCAL_SLAB: no halo exchange): every entry off the interface planes
    against the oracle's slab operator (non-Dirichlet interface planes), every z-segment split.  On the
    interface planes v7 splits an edge's face-line couplings between the two ranks differently from
    the oracle's element-by-element split (each line goes to one of the two elements of its face, see
    kernels_v7.cu), so only the halo-summed value is comparable there: test_gpu_loopback checks it
    against the global oracle."""
    import copy
    monkeypatch.setenv("SC_TEST_LOCAL_SLAB", "1")
    if z:
        monkeypatch.setenv("SC_V7_Z", z)
    g = small_grid(p, ne, 0.9, lengths=(1.2, 0.8, 1.1))
    for r in range(R):
        ctx = _ctx(g, monkeypatch, "v7", rank=r, nranks=R)
        z0, z1 = ctx.layout.z_begin, ctx.layout.z_end
        gs = copy.deepcopy(g)
        gs.ne = (g.ne[0], g.ne[1], z1 - z0)
        gs.hz = g.hz[z0:z1]
        gs.extra = dict(g.extra, dirichlet_z=(r == 0, r == R - 1))
        xg = lattice_random(75 + p, g.ne, g.p)
        xs = np.ascontiguousarray(xg[z0 * p:z1 * p + 1])
        ref = operator.AssembledCondensedOperator(gs).apply(xs.ravel()).reshape(xs.shape)
        y = _apply_nodal(ctx, xs.ravel()).reshape(xs.shape)
        keep = np.ones(xs.shape[0], bool)
        if r > 0:
            keep[0] = False
        if r < R - 1:
            keep[-1] = False
        assert _rel(y[keep], ref[keep]) <= 1e-12, (r, z0, z1)


@pytest.mark.parametrize("p,ne,z", [(8, (9, 7, 5), "2"), (8, (17, 3, 7), "3"), (5, (33, 4, 6), "4"),
                                    (3, (65, 3, 5), "2"), (4, (17, 2, 9), "1"), (6, (9, 5, 4), "4"),
                                    (10, (5, 3, 5), "2"), (12, (3, 2, 4), "3")])
def test_family_v7_z_segments(p, ne, z, monkeypatch):
    """v7 pass A assembles the z-faces inside a column of Z layers (and the x-faces inside a run); the
    segment-boundary z-faces and run-boundary x-faces keep their second part in U1: every Z, incl. a
    ragged last segment, and runs split in x (R = 8 / 16 / 32 elements)."""
    monkeypatch.setenv("SC_V7_Z", z)
    g = small_grid(p, ne, 0.9, lengths=(1.1, 0.8, 1.3))
    ref_op = operator.AssembledCondensedOperator(g)
    x = lattice_random(70 + p, g.ne, g.p).ravel()
    ctx = _ctx(g, monkeypatch, "v7")
    assert _rel(_apply_nodal(ctx, x), ref_op.apply(x)) <= 1e-12


@pytest.mark.parametrize("p,ne,want", [(4, (33, 5, 4), "rw"), (8, (21, 6, 5), "v3"), (6, (9, 5, 4), "v6"),
                                       (12, (5, 3, 3), "v4")])
def test_v7_out_of_memory_falls_back(p, ne, want, monkeypatch):
    """Without the memory for v7's two face-part vectors (SC_TEST_V7_NOMEM simulates the failed
    allocation) the context falls back to the one-pass family of that p, still exact."""
    from paper_1601_08179_b200 import Context
    monkeypatch.setenv("SC_TEST_V7_NOMEM", "1")
    g = small_grid(p, ne, 0.7, lengths=(1.2, 0.9, 0.6))
    ref_op = operator.AssembledCondensedOperator(g)
    x = lattice_random(97 + p, g.ne, g.p).ravel()
    ctx = Context(g.p, g.ne, (g.hx, g.hy, g.hz), g.lam, device=0)
    assert ctx.operator_kernel() == want, ctx.operator_kernel()
    assert _rel(_apply_nodal(ctx, x), ref_op.apply(x)) <= 1e-12


@pytest.mark.parametrize("p,ne", [(4, (33, 5, 4)), (8, (21, 6, 5)), (12, (5, 3, 3))])
def test_family_v7_two_stage_variant(p, ne, monkeypatch):
    """The opt-in two-stage pass A (SC_V7_STAGES=2: one element group per item, the next item's loads in
    flight while this one computes) against the oracle."""
    monkeypatch.setenv("SC_V7_STAGES", "2")
    g = small_grid(p, ne, 0.7, lengths=(1.2, 0.9, 0.6))
    ref_op = operator.AssembledCondensedOperator(g)
    x = lattice_random(95 + p, g.ne, g.p).ravel()
    ctx = _ctx(g, monkeypatch, "v7")
    assert _rel(_apply_nodal(ctx, x), ref_op.apply(x)) <= 1e-12


@pytest.mark.parametrize("p,ne", [(5, (15, 7, 4)), (8, (10, 6, 3)), (12, (3, 3, 3))])
def test_family_v7_pcg_fused_dot(p, ne, monkeypatch):
    """BT-PCG on v7 with p . q from pass B's per-block x . y partials, against the oracle."""
    from paper_1601_08179_b200 import SC_DUAL
    g = small_grid(p, ne, 1.0, lengths=(1.3, 0.7, 0.5))
    ref_op = operator.AssembledCondensedOperator(g)
    ctx = _ctx(g, monkeypatch, "v7")
    bt = ctx.skeleton()
    ctx.sc_fill_random(8, bt)
    lat = ctx.lattice()
    ctx.sc_from_transformed(bt, lat, SC_DUAL)
    b = lat.cpu().numpy()
    P = solve.BlockJacobi(ref_op)
    norm = solve.transformed_norm(g, ref_op.skel)
    res = pcg.pcg(ref_op.apply, P.apply, b, rtol=1e-10, norm=norm)
    xt = ctx.skeleton()
    rep = ctx.sc_pcg_solve(bt, xt, rtol=1e-10, maxit=2000)
    assert rep.converged and abs(rep.iters - res.iters) <= 1, (rep.iters, res.iters)
    ref = res.x if rep.iters == res.iters else pcg.pcg(ref_op.apply, P.apply, b, rtol=0, norm=norm,
                                                       fixed_iters=rep.iters).x
    assert _rel(ctx.to_lattice_nodal(xt).cpu().numpy(), ref) <= 1e-10
