"""GPU parity of the paper's operator variants TPC and MMC (§7, Table 3)
against the CPU oracle's dense Schur complement (nodal basis, no conversion: both variants take
and return nodal skeleton vectors, SC_PERM only re-orders lattice <-> skeleton layout).

Tolerance: relative L2 <= 1e-12 for one application (BASELINE.json north_star, as for TPT).
At p = 24, 32 (where the dense oracle setup takes minutes) the variants are compared with the TPT
path converted to the nodal basis, which tests/test_gpu_parity.py pins against the oracle.
"""
import numpy as np
import pytest
import torch

from oracle import operator
from synth import small_grid, lattice_random

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()
    assert torch.cuda.is_available()


def ctx_for(g):
    from paper_1601_08179_b200 import context_for_grid
    return context_for_grid(g, device=0)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def nonuniform(p, ne, lam, seed=0):
    rng = np.random.default_rng(seed)
    g = small_grid(p, ne, lam)
    g.hx = rng.uniform(0.3, 1.7, ne[0]); g.hy = rng.uniform(0.3, 1.7, ne[1]); g.hz = rng.uniform(0.3, 1.7, ne[2])
    return g


def variant_apply(ctx, variant, x_lat):
    """Nodal lattice vector -> nodal skeleton -> variant -> nodal lattice vector."""
    from paper_1601_08179_b200 import SC_PERM
    xs = ctx.skeleton()
    ctx.sc_to_transformed(torch.from_numpy(np.ascontiguousarray(x_lat)).cuda(), xs, SC_PERM)
    ys = ctx.skeleton(fill=7.0)           # stale values must be overwritten
    if variant == "tpc":
        ctx.sc_apply_tpc(xs, ys)
    else:
        ctx.sc_apply_mmc(xs, ys)
    y = ctx.lattice()
    ctx.sc_from_transformed(ys, y, SC_PERM)
    return y.cpu().numpy(), ys


def tpt_apply_nodal(ctx, x_lat):
    from paper_1601_08179_b200 import SC_PRIMAL, SC_DUAL
    xt = ctx.skeleton()
    ctx.sc_to_transformed(torch.from_numpy(np.ascontiguousarray(x_lat)).cuda(), xt, SC_PRIMAL)
    yt = ctx.skeleton()
    ctx.sc_apply_condensed(xt, yt)
    y = ctx.lattice()
    ctx.sc_from_transformed(yt, y, SC_DUAL)
    return y.cpu().numpy()


CASES = [(2, (2, 2, 2), 1.0), (3, (3, 2, 2), 0.0), (4, (2, 3, 2), 1.0), (5, (2, 2, 3), 0.7),
         (8, (3, 3, 3), 0.0), (8, (1, 2, 3), 1.0), (9, (2, 2, 2), 0.3), (12, (2, 2, 2), 1.0),
         (16, (2, 2, 2), 0.0)]


@pytest.mark.parametrize("variant", ["tpc", "mmc"])
@pytest.mark.parametrize("p,ne,lam", CASES)
def test_variant_parity_uniform(variant, p, ne, lam):
    g = small_grid(p, ne, lam, lengths=(1.0, 1.5, 0.8))
    ref = operator.AssembledCondensedOperator(g).apply(lattice_random(21 + p, g.ne, g.p).ravel())
    ctx = ctx_for(g)
    if variant == "mmc":
        ctx.sc_mmc_bind()
    y, _ = variant_apply(ctx, variant, lattice_random(21 + p, g.ne, g.p).ravel())
    assert rel(y, ref) <= 1e-12


@pytest.mark.parametrize("variant", ["tpc", "mmc"])
@pytest.mark.parametrize("p", [3, 6, 10])
def test_variant_parity_nonuniform(variant, p):
    """Per-element widths: TPC recomputes D^{-1} per element; MMC stores one matrix per element."""
    g = nonuniform(p, (3, 2, 2), 0.4, seed=p)
    x = lattice_random(4, g.ne, g.p).ravel()
    ref = operator.AssembledCondensedOperator(g).apply(x)
    ctx = ctx_for(g)
    if variant == "mmc":
        ctx.sc_mmc_bind()
    y, _ = variant_apply(ctx, variant, x)
    assert rel(y, ref) <= 1e-12


@pytest.mark.parametrize("p", [24, 32])
def test_variants_high_p_against_tpt(p):
    g = small_grid(p, (2, 1, 2), 1.0)
    x = lattice_random(9, g.ne, g.p).ravel()
    ctx = ctx_for(g)
    ref = tpt_apply_nodal(ctx, x)
    y_tpc, _ = variant_apply(ctx, "tpc", x)
    assert rel(y_tpc, ref) <= 1e-12
    ctx.sc_mmc_bind()
    y_mmc, _ = variant_apply(ctx, "mmc", x)
    assert rel(y_mmc, ref) <= 1e-12


def test_mmc_deterministic_and_symmetric():
    """Entity-centric assembly in a fixed order: repeated applications are bitwise equal; the
    assembled operator is symmetric (x . A y == y . A x to rounding)."""
    g = small_grid(6, (3, 3, 2), 1.0)
    ctx = ctx_for(g)
    ctx.sc_mmc_bind()
    x = lattice_random(1, g.ne, g.p).ravel()
    z = lattice_random(2, g.ne, g.p).ravel()
    y1, ys1 = variant_apply(ctx, "mmc", x)
    y2, ys2 = variant_apply(ctx, "mmc", x)
    assert torch.equal(ys1, ys2)
    w, _ = variant_apply(ctx, "mmc", z)
    a, b = float(z @ y1), float(x @ w)
    assert abs(a - b) <= 1e-12 * max(abs(a), 1.0)


def test_mmc_memory_guard_and_state():
    """sc_mmc_bind with a buffer smaller than sc_mmc_bytes -> SC_ENOMEM (the paper's memory
    argument); sc_apply_mmc before any bind -> SC_ESTATE."""
    from paper_1601_08179_b200 import capi
    g = nonuniform(5, (2, 2, 2), 1.0, seed=3)
    ctx = ctx_for(g)
    need = ctx.sc_mmc_bytes()
    nB = 6 * 16 + 12 * 4 + 8
    assert need >= 8 * nB * nB * 8          # one matrix per element (8 elements)
    x, y = ctx.skeleton(), ctx.skeleton()
    with pytest.raises(capi.ScError) as ei:
        ctx.sc_apply_mmc(x, y)
    assert ei.value.status == capi.SC_ESTATE
    small = torch.empty(need // 16, dtype=torch.float64, device="cuda")
    st = ctx.lib.sc_mmc_bind(ctx.ctx, small.data_ptr(), small.numel() * 8, None)
    assert st == capi.SC_ENOMEM
    ctx.sc_mmc_bind()
    ctx.sc_apply_mmc(x, y)


def test_tpc_multitile_launch_count():
    """TPC is one kernel launch per application (after the memset); MMC three (gather, DGEMM,
    assemble) -- the counts the variant sweep reports."""
    g = small_grid(4, (4, 3, 2), 1.0)
    ctx = ctx_for(g)
    x, y = ctx.skeleton(), ctx.skeleton()
    ctx.sc_fill_random(3, x)
    n0 = ctx.launch_count()
    ctx.sc_apply_tpc(x, y)
    assert ctx.launch_count() - n0 == 1
    ctx.sc_mmc_bind()
    n0 = ctx.launch_count()
    ctx.sc_apply_mmc(x, y)
    assert ctx.launch_count() - n0 == 3


# ---------------------------------------------------------------- solvers UC / DC / BC
def _nodal_skel(ctx, v_lat):
    from paper_1601_08179_b200 import SC_PERM
    s = ctx.skeleton()
    ctx.sc_to_transformed(torch.from_numpy(np.ascontiguousarray(v_lat)).cuda(), s, SC_PERM)
    return s


def _nodal_lat(ctx, v_skel):
    from paper_1601_08179_b200 import SC_PERM
    lat = ctx.lattice()
    ctx.sc_from_transformed(v_skel, lat, SC_PERM)
    return lat.cpu().numpy()


@pytest.mark.parametrize("prec", ["none", "diag", "block"])
@pytest.mark.parametrize("p,ne,aniso", [(4, (3, 2, 2), 1.0), (6, (2, 3, 2), 8.0), (9, (2, 2, 2), 1.0)])
def test_nodal_solvers_against_oracle(prec, p, ne, aniso):
    """UC / DC / BC with the TPC operator against the oracle's PCG with the same preconditioner
    (identity / assembled diagonal / BlockJacobi), nodal Euclidean residual norm (DESIGN R18):
    iteration count within +-1, iterate at the GPU's count within 1e-10 (readings R7, R8)."""
    from oracle import pcg, solve
    g = small_grid(p, ne, 1.0, lengths=(aniso, 1.0, 1.0))
    op = operator.AssembledCondensedOperator(g)
    b = lattice_random(17, g.ne, g.p).ravel()
    P = {"none": lambda r: np.where(op.free, r, 0.0),
         "diag": (lambda dg: lambda r: np.where(op.free, r / np.where(op.free, dg, 1.0), 0.0))(
             solve.assembled_diagonal(op)),
         "block": solve.BlockJacobi(op).apply}[prec]
    ref = pcg.pcg(op.apply, P, np.where(op.free, b, 0.0), rtol=1e-10, maxit=2000)
    ctx = ctx_for(g)
    bs, xs = _nodal_skel(ctx, b), ctx.skeleton()
    rep = ctx.sc_pcg_solve_nodal(bs, xs, op="tpc", prec=prec, rtol=1e-10, maxit=2000)
    assert rep.converged and abs(rep.iters - ref.iters) <= 1
    ref_k = pcg.pcg(op.apply, P, np.where(op.free, b, 0.0), fixed_iters=rep.iters)
    assert rel(_nodal_lat(ctx, xs), ref_k.x) <= 1e-10


def test_bc_equals_bt_iterates_and_mmc_solver():
    """BC (nodal, block preconditioner) and BT (transformed, diagonal) produce the same iterates
    (x_BC = Shat^T x~_BT: the block preconditioner reduces to a diagonal in the
    transformed system); the MMC operator gives the same BC solve as TPC."""
    from paper_1601_08179_b200 import SC_PRIMAL, SC_DUAL
    g = small_grid(5, (3, 3, 2), 0.5)
    ctx = ctx_for(g)
    b = lattice_random(3, g.ne, g.p).ravel()
    bs, xs = _nodal_skel(ctx, b), ctx.skeleton()
    ctx.sc_pcg_solve_nodal(bs, xs, op="tpc", prec="block", rtol=0.0, maxit=15)
    bt = ctx.skeleton()
    ctx.sc_to_transformed(torch.from_numpy(b).cuda(), bt, SC_DUAL)
    xt = ctx.skeleton()
    ctx.sc_pcg_solve(bt, xt, rtol=0.0, maxit=15)
    x_bt = ctx.lattice()
    ctx.sc_from_transformed(xt, x_bt, SC_PRIMAL)
    assert rel(_nodal_lat(ctx, xs), x_bt.cpu().numpy()) <= 1e-10
    ctx.sc_mmc_bind()
    xm = ctx.skeleton()
    rep = ctx.sc_pcg_solve_nodal(bs, xm, op="mmc", prec="block", rtol=1e-10, maxit=500)
    rep2 = ctx.sc_pcg_solve_nodal(bs, xs, op="tpc", prec="block", rtol=1e-10, maxit=500)
    assert rep.converged and abs(rep.iters - rep2.iters) <= 1
    assert rel(_nodal_lat(ctx, xm), _nodal_lat(ctx, xs)) <= 1e-9
