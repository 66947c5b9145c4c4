"""The paper's solver benchmark E3: Omega = (0, 2 pi)^3,
8^3 elements graded with constant expansion factor alpha in {1, 1.5, 2} (AR_max 1 / 17 / 128,
DESIGN.md reading R15), lambda = 0, the manufactured solution Eq. eq:solution with k = 5 and its
inhomogeneous Dirichlet data, residual reduced by 1e-12.

Per (alpha, p) one solve = sc_setup + workspace (precomputation is included) +
sc_condense_rhs_dirichlet + BT-PCG + sc_recover_dirichlet, repeated --reps times; the first
repetition is dropped and the rest averaged (11 runs, last 10 averaged).  Reports
iterations, per-solve and per-iteration time, and the max nodal error against u_ex.  The
summary gives iterations(alpha = 2) / iterations(alpha = 1) per p, the paper's "about 1.5x"
(P:684).  Timing is host wall clock around a synchronised solve (it includes host setup work),
so it is a study number, not a bench value.

    python tools/e3_study.py [--ps 2,4,6,8,12,16,24,32] [--alphas 1,1.5,2] [--reps 11] [--out f.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def gll_nodes(p):
    """GLL nodes on [-1, 1]: endpoints and the roots of P_p' (input generation only)."""
    inner = np.polynomial.legendre.Legendre.basis(p).deriv().roots()
    return np.concatenate([[-1.0], np.sort(inner.real), [1.0]])


def lattice_1d(widths, p):
    x = gll_nodes(p)
    pts = [0.0]
    a = 0.0
    for h in widths:
        pts.extend((a + 0.5 * h * (x[1:] + 1.0)).tolist())
        a += h
    return np.array(pts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ps", default="2,4,6,8,12,16,24,32")
    ap.add_argument("--alphas", default="1,1.5,2")
    ap.add_argument("--reps", type=int, default=11)
    ap.add_argument("--k", type=float, default=5.0)
    ap.add_argument("--ns", default="8", help="elements per direction (E4: --ps 16 --alphas 1 --ns 2,4,8,16)")
    ap.add_argument("--solvers", default="bt", help="bt,bc,dc,uc (P:602-607; UC/DC/BC use TPC, nodal system)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import context_for_grid
    from synth import e3_grid, e3_u, e3_f
    rows = []
    from paper_1601_08179_b200 import SC_PERM, SC_PRIMAL, SC_DUAL
    cases = [(p, alpha, n, sv) for n in [int(s) for s in a.ns.split(",")] for p in [int(s) for s in a.ps.split(",")]
             for alpha in [float(s) for s in a.alphas.split(",")] for sv in a.solvers.split(",")]
    for p, alpha, n, solver in cases:
        g = e3_grid(p, alpha, n=n)
        xs, ys, zs = lattice_1d(g.hx, p), lattice_1d(g.hy, p), lattice_1d(g.hz, p)
        Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
        f = torch.from_numpy(e3_f(X, Y, Z, 0.0, k=a.k).ravel()).cuda()
        gd = torch.from_numpy(e3_u(X, Y, Z, k=a.k).ravel()).cuda()
        times, its, kern = [], None, ""
        for rep in range(a.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ctx = context_for_grid(g)
            bt = ctx.skeleton()
            ctx.sc_condense_rhs_dirichlet(f, gd, bt)
            xt = ctx.skeleton()
            if solver == "bt":
                r = ctx.sc_pcg_solve(bt, xt, rtol=1e-12, maxit=20000)
            else:   # nodal system: b = Shat^{-1} b~, x~ = Shat^{-T} x (untimed conversions around the solve)
                lat = ctx.lattice()
                ctx.sc_from_transformed(bt, lat, SC_DUAL)
                bs, xs = ctx.skeleton(), ctx.skeleton()
                ctx.sc_to_transformed(lat, bs, SC_PERM)
                r = ctx.sc_pcg_solve_nodal(bs, xs, op="tpc", prec={"bc": "block", "dc": "diag", "uc": "none"}[solver],
                                           rtol=1e-12, maxit=20000)
                ctx.sc_from_transformed(xs, lat, SC_PERM)
                ctx.sc_to_transformed(lat, xt, SC_PRIMAL)
            u = ctx.lattice()
            ctx.sc_recover_dirichlet(f, gd, xt, u)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            its, conv, t_pcg, kern = r.iters, bool(r.converged), r.t_solve_s, ctx.operator_kernel()
            err = float((u - gd).abs().max())
            ctx.close()
            del ctx
        t = float(np.mean(times[1:])) if len(times) > 1 else times[0]
        row = dict(solver=solver, p=p, alpha=alpha, n=n, ar_max=float(alpha ** (n - 1)), iters=its, converged=conv,
                   s_per_solve=t, s_pcg=t_pcg, s_per_iter=t_pcg / max(its, 1), max_err=err, kernel=kern,
                   N=int(len(xs) * len(ys) * len(zs)))
        rows.append(row)
        print(json.dumps(row), flush=True)
    summary = {}
    for sv, p, n in sorted({(r["solver"], r["p"], r["n"]) for r in rows}):
        it = {r["alpha"]: r["iters"] for r in rows if r["p"] == p and r["n"] == n and r["solver"] == sv}
        if 1.0 in it and 2.0 in it:
            summary[f"{sv}_p{p}_n{n}"] = dict(iters=it, growth_a2_over_a1=it[2.0] / it[1.0])
    out = dict(study="E3 (P:625-687): 8^3 graded, k = 5, lambda = 0, inhomogeneous Dirichlet, rtol 1e-12",
               k=a.k, ns=a.ns, reps=a.reps, rows=rows, iteration_growth=summary,
               paper="iterations grow by about 1.5x from AR_max 1 to 128 for BC and BT (P:684)",
               gpu=torch.cuda.get_device_name(0))
    print(json.dumps(dict(iteration_growth=summary)))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
