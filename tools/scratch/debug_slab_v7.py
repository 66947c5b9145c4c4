import copy, os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import __graft_entry__
__graft_entry__.build()
from oracle import operator
from synth import small_grid, lattice_random
from paper_1601_08179_b200 import Context, SC_PRIMAL, SC_DUAL
os.environ["SC_TEST_LOCAL_SLAB"] = "1"; os.environ["SC_SMALL_V1"] = "0"
p, ne, R = 4, (3, 3, 4), 2
for op in ("v6", "v7"):
    os.environ["SC_OP"] = op
    g = small_grid(p, ne, 0.9, lengths=(1.2, 0.8, 1.1))
    for r in range(R):
        ctx = Context(g.p, g.ne, (g.hx, g.hy, g.hz), g.lam, device=0, rank=r, nranks=R)
        z0, z1 = ctx.layout.z_begin, ctx.layout.z_end
        gs = copy.deepcopy(g); gs.ne = (g.ne[0], g.ne[1], z1 - z0); gs.hz = g.hz[z0:z1]
        gs.extra = dict(g.extra, dirichlet_z=(r == 0, r == R - 1))
        xg = lattice_random(75 + p, g.ne, g.p)
        xs = np.ascontiguousarray(xg[z0 * p:z1 * p + 1])
        ref = operator.AssembledCondensedOperator(gs).apply(xs.ravel()).reshape(xs.shape)
        xt = ctx.skeleton(); ctx.sc_to_transformed(torch.from_numpy(xs.ravel()).cuda(), xt, SC_PRIMAL)
        yt = ctx.skeleton(); ctx.sc_apply_condensed(xt, yt)
        yl = ctx.lattice(); ctx.sc_from_transformed(yt, yl, SC_DUAL)
        y = yl.cpu().numpy().reshape(xs.shape)
        d = np.abs(y - ref)
        print(op, ctx.operator_kernel(), "rank", r, "rel", np.linalg.norm(d) / np.linalg.norm(ref))
        nz1 = xs.shape[0]
        for k in range(nz1):
            if d[k].max() > 1e-10:
                pl = d[k]
                idx = np.argwhere(pl > 1e-10)
                kinds = set()
                for (j, i) in idx[:400]:
                    t = (i % p == 0) + (j % p == 0) + (k % p == 0)
                    kinds.add({1: "face", 2: "edge", 3: "vertex", 0: "interior"}[int(t)])
                print("  plane k", k, "max", pl.max(), "n", len(idx), kinds)
        ctx.close()
# detail: rank 0 top interface plane, entries with error
os.environ["SC_OP"] = "v7"
g = small_grid(p, ne, 0.9, lengths=(1.2, 0.8, 1.1))
r = 0
ctx = Context(g.p, g.ne, (g.hx, g.hy, g.hz), g.lam, device=0, rank=r, nranks=R)
z0, z1 = ctx.layout.z_begin, ctx.layout.z_end
gs = copy.deepcopy(g); gs.ne = (g.ne[0], g.ne[1], z1 - z0); gs.hz = g.hz[z0:z1]
gs.extra = dict(g.extra, dirichlet_z=(True, False))
for trial in range(3):
    xs = np.zeros(((z1 - z0) * p + 1, g.ne[1] * p + 1, g.ne[0] * p + 1))
    k = (z1 - z0) * p
    if trial == 0: xs[k, 5, 5] = 1.0          # interface face interior node
    if trial == 1: xs[k - p, 5, 5] = 1.0      # plane below (opposite face)
    if trial == 2: xs[k - 1, 5, 5] = 1.0      # interior node (not skeleton) -> ignored
    ref = operator.AssembledCondensedOperator(gs).apply(xs.ravel()).reshape(xs.shape)
    xt = ctx.skeleton(); ctx.sc_to_transformed(torch.from_numpy(xs.ravel()).cuda(), xt, SC_PRIMAL)
    yt = ctx.skeleton(); ctx.sc_apply_condensed(xt, yt)
    yl = ctx.lattice(); ctx.sc_from_transformed(yt, yl, SC_DUAL)
    y = yl.cpu().numpy().reshape(xs.shape)
    d = y - ref
    print("trial", trial, "max err", np.abs(d).max())
    for kk in range(xs.shape[0]):
        if np.abs(d[kk]).max() > 1e-12:
            print("  k", kk, np.round(d[kk][4:9, 4:9], 6).tolist(), "ref", np.round(ref[kk][4:9, 4:9], 6).tolist())
