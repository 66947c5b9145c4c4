"""BASELINE configs[3] / SURVEY c15 (cfg4): anisotropic grid, 32^3 elements of degree p=16 on
[0, AR] x [0, 1]^2 (x element length scaled), lambda = 0, homogeneous Dirichlet, manufactured
u = sin(pi x) sin(pi y) sin(pi z) (AR integer, so u vanishes on x = AR), f = 3 pi^2 u.
For AR in {1, 8, 32, 128}: condense the RHS (Alg. 4 pre), BT-PCG to rtol = 1e-10, recover the
interiors (Alg. 4 post); report iterations, solve time (CUDA events around sc_pcg_solve) and the
max nodal error against u.

    python tools/cfg4_aniso.py [--ars 1,8,32,128] [--n 32] [--out profiles/cfg4_r1.json]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gll_nodes(p):
    """GLL nodes on [-1, 1]: endpoints and the roots of P_p' (numpy Legendre, for the input only)."""
    inner = np.polynomial.legendre.Legendre.basis(p).deriv().roots()
    return np.concatenate([[-1.0], np.sort(inner.real), [1.0]])


def lattice_1d(n, length, p):
    """Lattice coordinates of n equal elements on [0, length] (shared element ends once)."""
    x = gll_nodes(p)
    h = length / n
    pts = [0.0]
    for e in range(n):
        pts.extend((e * h + 0.5 * h * (x[1:] + 1.0)).tolist())
    return np.array(pts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ars", default="1,8,32,128")
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import context_for_grid
    from synth import cfg4
    rows = []
    for ar in [int(s) for s in a.ars.split(",")]:
        g = cfg4(ar, n=a.n)
        if a.p != 16:
            g.p = a.p
        ctx = context_for_grid(g)
        X = torch.from_numpy(lattice_1d(a.n, float(ar), g.p)).cuda()
        Y = torch.from_numpy(lattice_1d(a.n, 1.0, g.p)).cuda()
        Z = Y.clone()
        sx, sy, sz = torch.sin(math.pi * X), torch.sin(math.pi * Y), torch.sin(math.pi * Z)
        u_ex = (sz[:, None, None] * sy[None, :, None] * sx[None, None, :]).reshape(-1)
        f = (g.lam + 3.0 * math.pi ** 2) * u_ex
        b, x, u = ctx.skeleton(), ctx.skeleton(), ctx.lattice()
        ctx.sc_condense_rhs(f, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.sc_pcg_solve(b, x, rtol=1e-10, maxit=20000)   # warm-up solve (module load, graph capture); the second is timed
        torch.cuda.synchronize()
        e0.record()
        rep = ctx.sc_pcg_solve(b, x, rtol=1e-10, maxit=20000)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ctx.sc_recover(f, x, u)
        err = float((u - u_ex).abs().max())
        row = {"aspect_ratio": ar, "p": g.p, "elements": a.n ** 3, "N": int(u.numel()), "iters": rep.iters,
               "converged": bool(rep.converged), "relres": rep.relres, "solve_ms": ms,
               "ms_per_iter": ms / max(rep.iters, 1), "max_nodal_error": err}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del ctx, b, x, u, f, u_ex
        torch.cuda.empty_cache()
    out = {"config": f"cfg4: {a.n}^3 elements p={a.p} on [0,AR]x[0,1]^2, lambda=0, sine manufactured solution, "
                     "BT-PCG rtol 1e-10", "rows": rows}
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
