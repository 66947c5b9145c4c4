"""SURVEY §8(f) f4 (the paper's E4): BT-PCG iteration count and solve time against the
element count at p = 16, n_e = n^3 for n = 2, 4, 8, 16, 32.  Stand-in for the paper's alpha = 1
case (whose inhomogeneous Dirichlet lifting is out of scope here): the unit cube,
lambda = 0, homogeneous Dirichlet, manufactured u = sin(pi x) sin(pi y) sin(pi z), rtol 1e-12 (the
paper's tolerance).  Reports the log-log slope of iterations against n_e (paper: < 1/3).

    python tools/ne_scaling.py [--ns 2,4,8,16,32] [--p 16] [--out profiles/ne_scaling_r1.json]
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="2,4,8,16,32")
    ap.add_argument("--p", type=int, default=16)
    ap.add_argument("--rtol", type=float, default=1e-12)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import context_for_grid
    from synth import small_grid
    from cfg4_aniso import lattice_1d
    rows = []
    for n in [int(s) for s in a.ns.split(",")]:
        g = small_grid(a.p, (n, n, n), 0.0, name=f"ne{n}")
        ctx = context_for_grid(g)
        X = torch.from_numpy(lattice_1d(n, 1.0, g.p)).cuda()
        s1 = torch.sin(math.pi * X)
        u_ex = (s1[:, None, None] * s1[None, :, None] * s1[None, None, :]).reshape(-1)
        f = (g.lam + 3.0 * math.pi ** 2) * u_ex
        b, x, u = ctx.skeleton(), ctx.skeleton(), ctx.lattice()
        ctx.sc_condense_rhs(f, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.sc_pcg_solve(b, x, rtol=a.rtol, maxit=50000)   # warm-up solve (module load, graph capture); the second is timed
        torch.cuda.synchronize()
        e0.record()
        rep = ctx.sc_pcg_solve(b, x, rtol=a.rtol, maxit=50000)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        ctx.sc_recover(f, x, u)
        row = {"n_e": n ** 3, "n": n, "p": g.p, "N": int(u.numel()), "iters": rep.iters,
               "converged": bool(rep.converged), "solve_ms": ms,
               "max_nodal_error": float((u - u_ex).abs().max())}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del ctx, b, x, u, f, u_ex
        torch.cuda.empty_cache()
    ne = np.array([r["n_e"] for r in rows], dtype=float)
    it = np.array([r["iters"] for r in rows], dtype=float)
    slope = float(np.polyfit(np.log(ne[1:]), np.log(it[1:]), 1)[0]) if len(rows) > 2 else None
    out = {"config": f"p={a.p}, unit cube, lambda=0, sine manufactured solution, BT-PCG rtol {a.rtol}",
           "rows": rows, "iteration_slope_vs_n_e": slope}
    print(json.dumps({"iteration_slope_vs_n_e": slope}))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
