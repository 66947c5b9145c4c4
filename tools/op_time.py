"""Time one condensed-operator application (CUDA events, mean of --reps after 2 warm-ups) for the
p <= 8 operator families selected by SC_OP (v5 / v3 / rw) on cfg5 and cfg3-shaped grids.

    python tools/op_time.py [--ops v5,v3] [--cases cfg5,cfg3:4,cfg3:8] [--reps 10] [--out f.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", default="v5,v3")
    ap.add_argument("--cases", default="cfg5,cfg3:4,cfg3:8")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import context_for_grid
    import synth
    rows = []
    for case in a.cases.split(","):
        if case == "cfg5":
            g = synth.cfg5()
        elif case.startswith("cfg3:"):
            g = synth.cfg3(int(case.split(":")[1]))
        else:   # "p<degree>:<n>": n^3 elements on the unit cube, lambda = 1
            p, n = (int(v) for v in case[1:].split(":"))
            g = synth.small_grid(p, (n, n, n), 1.0)
        for op in a.ops.split(","):
            if op == "rw" and g.p not in (3, 4):
                continue
            os.environ["SC_OP"] = op
            ctx = context_for_grid(g, device=0)
            x, y = ctx.skeleton(), ctx.skeleton()
            ctx.sc_fill_random(3, x)
            for _ in range(2):
                ctx.sc_apply_condensed(x, y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                ctx.sc_apply_condensed(x, y)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            L = ctx.layout
            nx, ny, nz = L.ne_local
            nc = (nx * g.p + 1) * (ny * g.p + 1) * (nz * g.p + 1) - nx * ny * nz * (g.p - 1) ** 3
            gbs = 16.0 * nc / (ms * 1e-3) / 1e9
            r = {"case": case, "op": op, "p": g.p, "ne": list(g.ne), "ms": ms, "alg_GBs": gbs,
                 "hbm_frac": gbs / 6549.8, "ynorm": float(y.norm())}
            print(json.dumps(r), flush=True)
            rows.append(r)
            del ctx, x, y
            torch.cuda.empty_cache()
    if a.out:
        json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
