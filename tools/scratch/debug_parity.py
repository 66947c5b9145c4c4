"""Quick GPU-vs-oracle parity sweep (debug aid): operator rel. error per p / grid, and the
spectral-convergence PCG runs with their iteration counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_1601_08179_b200 import context_for_grid, SC_PRIMAL, SC_DUAL
from oracle import mesh, operator
from synth import small_grid, lattice_random, sine_f, sine_u


def apply_nodal(ctx, x):
    xt = ctx.skeleton(); ctx.sc_to_transformed(torch.from_numpy(x).cuda(), xt, SC_PRIMAL)
    yt = ctx.skeleton(); ctx.sc_apply_condensed(xt, yt)
    y = ctx.lattice(); ctx.sc_from_transformed(yt, y, SC_DUAL)
    return y.cpu().numpy()


for p in range(2, 10):
    for ne in [(2, 2, 2), (9, 5, 2)]:
        g = small_grid(p, ne, 1.0)
        op = operator.AssembledCondensedOperator(g)
        x = lattice_random(3, g.ne, g.p).ravel()
        ref = op.apply(x)
        y = apply_nodal(context_for_grid(g, device=0), x)
        print(f"p={p} ne={ne}: rel {np.linalg.norm(y - ref) / np.linalg.norm(ref):.2e}", flush=True)
for p in (2, 3, 4, 5, 6, 7):
    g = small_grid(p, (2, 2, 2), 1.0)
    X, Y, Z = mesh.lattice_coordinates(g)
    f = torch.from_numpy(sine_f(X, Y, Z, 1.0)).cuda()
    ctx = context_for_grid(g, device=0)
    bt, xt, u = ctx.skeleton(), ctx.skeleton(), ctx.lattice()
    ctx.sc_condense_rhs(f, bt)
    try:
        rep = ctx.sc_pcg_solve(bt, xt, rtol=1e-13, maxit=1000)
        ctx.sc_recover(f, xt, u)
        print(f"spectral p={p}: iters {rep.iters} conv {rep.converged} err {np.abs(u.cpu().numpy() - sine_u(X, Y, Z)).max():.2e}")
    except Exception as e:
        print(f"spectral p={p}: {e}")
