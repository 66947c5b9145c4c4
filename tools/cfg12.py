"""BASELINE configs[0], [1] (cfg1: 2^3 elements p=4 lambda=1; cfg2: 8^3 elements p=8 lambda=0):
operator applications (mean of 100 after one warm-up) and the sine manufactured PCG solve to
rtol 1e-10 (iterations, solve time, per-iteration time, max nodal error).  Launch-bound sizes.

    python tools/cfg12.py [--out profiles/cfg12_r1.json]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import context_for_grid
    from synth import cfg1, cfg2
    from cfg4_aniso import lattice_1d
    rows = []
    for name, g in (("cfg1", cfg1()), ("cfg2", cfg2())):
        ctx = context_for_grid(g)
        x, y = ctx.skeleton(), ctx.skeleton()
        ctx.sc_fill_random(1 if name == "cfg1" else 2, x)
        ctx.sc_apply_condensed(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100):
            ctx.sc_apply_condensed(x, y)
        e1.record()
        torch.cuda.synchronize()
        op_us = e0.elapsed_time(e1) * 10.0
        n = g.ne[0]
        X = torch.from_numpy(lattice_1d(n, 1.0, g.p)).cuda()
        s1 = torch.sin(math.pi * X)
        u_ex = (s1[:, None, None] * s1[None, :, None] * s1[None, None, :]).reshape(-1)
        f = (g.lam + 3.0 * math.pi ** 2) * u_ex
        b, xs, u = ctx.skeleton(), ctx.skeleton(), ctx.lattice()
        ctx.sc_condense_rhs(f, b)
        ctx.sc_pcg_solve(b, xs, rtol=1e-10, maxit=1000)     # warm-up (graph capture, caches)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = ctx.sc_pcg_solve(b, xs, rtol=1e-10, maxit=1000)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        ctx.sc_recover(f, xs, u)
        row = {"config": name, "p": g.p, "elements": g.n_elements, "N": int(u.numel()), "op_us_per_apply": op_us,
               "pcg_iters": rep.iters, "solve_ms_wall": ms, "us_per_iter": 1e3 * ms / max(rep.iters, 1),
               "max_nodal_error": float((u - u_ex).abs().max())}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as fh:
            json.dump({"rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
