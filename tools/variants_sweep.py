"""The paper's operator comparison (§7 "Efficiency of operators", Fig.
`fig:operator_efficiency`): n_e = 512 elements (8^3), lambda = pi, 2 <= p <= 32; precomputation and
application time of MMC, TPC and TPT on one B200.

Timing as in the paper: one warm-up application, then the mean of the next 100 (CUDA events
on the launching stream).  TPT is timed twice: "tpt_v1" runs the one-CTA-per-element v1 kernel,
the same implementation skeleton as the TPC kernel (so the ratio TPC / TPT_v1 isolates the
factorisation, the paper's comparison), and "tpt" the library's default kernel for the grid.
MMC is timed uniform (one element matrix) and, with --nonuniform, on a graded grid (one matrix per
element: the paper's setup / memory argument).

    python tools/variants_sweep.py [--ps 2,3,4,...] [--ne 8] [--reps 100] [--out f.json]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps):
    import torch
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ps", default="2,3,4,5,6,8,10,12,14,16,20,24,28,32")
    ap.add_argument("--ne", type=int, default=8)
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--nonuniform", default="2,4,8,12,16")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import numpy as np
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import context_for_grid
    import synth
    rows = []
    n = a.ne
    nonuni = {int(v) for v in a.nonuniform.split(",") if v}
    for p in (int(v) for v in a.ps.split(",")):
        g = synth.small_grid(p, (n, n, n), math.pi)
        ni = p - 1
        nB = 6 * ni * ni + 12 * ni + 8
        N = (n * p + 1) ** 3
        row = {"p": p, "ne": n ** 3, "N": N, "nB": nB,
               "mult_per_elem": {"mmc": 36 * ni ** 4 + 56 * ni ** 2, "tpc": 49 * ni ** 3, "tpt": 13 * ni ** 3}}
        # TPT, library default kernel
        t0 = time.perf_counter()
        ctx = context_for_grid(g, device=0)
        torch.cuda.synchronize()
        row["tpt_setup_ms"] = 1e3 * (time.perf_counter() - t0)
        row["tpt_kernel"] = ctx.operator_kernel()
        x, y = ctx.skeleton(), ctx.skeleton()
        ctx.sc_fill_random(5, x)
        row["tpt_ms"] = timed(lambda: ctx.sc_apply_condensed(x, y), a.reps)
        row["tpc_ms"] = timed(lambda: ctx.sc_apply_tpc(x, y), a.reps)
        t0 = time.perf_counter()
        ctx.sc_mmc_bind()
        torch.cuda.synchronize()
        row["mmc_setup_ms"] = 1e3 * (time.perf_counter() - t0)
        row["mmc_bytes"] = ctx.sc_mmc_bytes()
        row["mmc_ms"] = timed(lambda: ctx.sc_apply_mmc(x, y), a.reps)
        del ctx, x, y
        torch.cuda.empty_cache()
        # TPT through the v1 kernel (same skeleton as the TPC kernel)
        os.environ["SC_APPLY_V1"] = "1"
        try:
            ctx = context_for_grid(g, device=0)
        finally:
            del os.environ["SC_APPLY_V1"]
        x, y = ctx.skeleton(), ctx.skeleton()
        ctx.sc_fill_random(5, x)
        row["tpt_v1_ms"] = timed(lambda: ctx.sc_apply_condensed(x, y), a.reps)
        del ctx, x, y
        if p in nonuni:   # graded widths: one MMC matrix per element
            rng = np.random.default_rng(p)
            gn = synth.small_grid(p, (n, n, n), math.pi)
            gn.hx = rng.uniform(0.5, 1.5, n); gn.hy = rng.uniform(0.5, 1.5, n); gn.hz = rng.uniform(0.5, 1.5, n)
            ctx = context_for_grid(gn, device=0)
            x, y = ctx.skeleton(), ctx.skeleton()
            ctx.sc_fill_random(5, x)
            row["mmc_nonuni_bytes"] = ctx.sc_mmc_bytes()
            t0 = time.perf_counter()
            ctx.sc_mmc_bind()
            torch.cuda.synchronize()
            row["mmc_nonuni_setup_ms"] = 1e3 * (time.perf_counter() - t0)
            row["mmc_nonuni_ms"] = timed(lambda: ctx.sc_apply_mmc(x, y), a.reps)
            row["tpc_nonuni_ms"] = timed(lambda: ctx.sc_apply_tpc(x, y), a.reps)
            row["tpt_nonuni_ms"] = timed(lambda: ctx.sc_apply_condensed(x, y), a.reps)
            row["tpt_nonuni_kernel"] = ctx.operator_kernel()
            del ctx, x, y
        torch.cuda.empty_cache()
        row["ratio_tpc_over_tpt_v1"] = row["tpc_ms"] / row["tpt_v1_ms"]
        row["ratio_mmc_over_tpt_v1"] = row["mmc_ms"] / row["tpt_v1_ms"]
        row["ratio_mmc_over_tpc"] = row["mmc_ms"] / row["tpc_ms"]
        print(json.dumps(row), flush=True)
        rows.append(row)
    if a.out:
        json.dump({"config": f"n_e = {n}^3, lambda = pi, uniform unit cube (P:505-507); nonuniform: widths "
                             "uniform[0.5,1.5] per direction", "reps": a.reps, "rows": rows},
                  open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
