import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_1601_08179_b200 import context_for_grid, capi
from oracle import mesh
from synth import small_grid, sine_f
lib = capi.load()
for trial in range(4):
    for p in (2, 3, 4):
        g = small_grid(p, (2, 2, 2), 1.0)
        X, Y, Z = mesh.lattice_coordinates(g)
        f = torch.from_numpy(sine_f(X, Y, Z, 1.0)).cuda()
        ctx = context_for_grid(g, device=0)
        bt, xt = ctx.skeleton(), ctx.skeleton()
        ctx.sc_condense_rhs(f, bt)
        h = bt.cpu().numpy()
        for it_chunk in (1, 8):
            ctx.sc_pcg_start(bt, xt, rtol=1e-13, maxit=1000)
            hist = []
            for k in range(24 // it_chunk):
                ctx.sc_pcg_iterate(it_chunk)
                rep = capi.ScPcgReport()
                st = lib.sc_pcg_status(ctx.ctx, ctypes.byref(rep), None)
                hist.append((rep.iters, f"{rep.relres:.2e}", st))
            print(trial, p, it_chunk, "b-sum", float(np.abs(h).sum()), hist[:6], flush=True)
