"""Diagnose the 16^3 p=16 AR=128 PCG iteration gap (GPU 54 vs oracle 52): residual histories,
operator parity at AR=128, and the true residual of both iterates."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ.setdefault("SC_SMALL_V1", "0")
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from oracle import operator, solve, pcg, mesh
from synth import small_grid, sine_f, lattice_random
from paper_1601_08179_b200 import context_for_grid, SC_PRIMAL, SC_DUAL

def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)

# operator parity at AR = 128 (small grid) and AR = 1
for ar in (1, 128):
    g = small_grid(16, (3, 3, 3), 0.0, lengths=(float(ar) * 3 / 16, 3 / 16, 3 / 16))
    op = operator.AssembledCondensedOperator(g)
    x = lattice_random(5, g.ne, g.p).ravel()
    ctx = context_for_grid(g, device=0)
    xt = ctx.skeleton(); ctx.sc_to_transformed(torch.from_numpy(x).cuda(), xt, SC_PRIMAL)
    yt = ctx.skeleton(); ctx.sc_apply_condensed(xt, yt)
    y = ctx.lattice(); ctx.sc_from_transformed(yt, y, SC_DUAL)
    print("operator AR", ar, "rel", rel(y.cpu().numpy(), op.apply(x)), flush=True)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
g = small_grid(16, (n, n, n), 0.0, lengths=(128.0, 1.0, 1.0))
X, Y, Z = mesh.lattice_coordinates(g)
f = sine_f(X, Y, Z, 0.0)
t = time.time()
op = operator.AssembledCondensedOperator(g)
b = solve.condensed_rhs(op, f)
P = solve.BlockJacobi(op)
res = pcg.pcg(op.apply, P.apply, b, rtol=1e-10, norm=solve.transformed_norm(g, op.skel))
print("oracle iters", res.iters, "time", time.time() - t, flush=True)
h0 = np.array(res.history) / res.history[0]
ctx = context_for_grid(g, device=0)
fd = torch.from_numpy(f).cuda()
bt = ctx.skeleton(); ctx.sc_condense_rhs(fd, bt)
lat = ctx.lattice(); ctx.sc_from_transformed(bt, lat, SC_DUAL)
print("rhs rel", rel(lat.cpu().numpy(), b), flush=True)
hist = []
for k in range(1, 60):
    xt = ctx.skeleton()
    rep = ctx.sc_pcg_solve(bt, xt, rtol=0.0, maxit=k)
    hist.append(rep.relres)
for k in range(1, 60):
    o = h0[k] if k < len(h0) else float('nan')
    print(k, f"gpu {hist[k-1]:.6e} oracle {o:.6e}", flush=True)
# run the oracle with the GPU's rhs (transformed back) to separate rhs vs operator effects
res2 = pcg.pcg(op.apply, P.apply, lat.cpu().numpy(), rtol=1e-10, norm=solve.transformed_norm(g, op.skel))
print("oracle iters with GPU rhs", res2.iters, flush=True)
