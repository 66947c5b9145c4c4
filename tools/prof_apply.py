"""Run the condensed operator a few times on a given grid (for ncu captures).

    python tools/prof_apply.py --p 8 --n 64 --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--nz", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--pcg", type=int, default=0, help="also run this many PCG iterations")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import context_for_grid
    from synth import small_grid
    nz = a.nz or a.n
    g = small_grid(a.p, (a.n, a.n, nz), 1.0)
    ctx = context_for_grid(g)
    x, y = ctx.skeleton(), ctx.skeleton()
    ctx.sc_fill_random(5, x)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        ctx.sc_apply_condensed(x, y)
    ev0.record()
    for _ in range(a.reps):
        ctx.sc_apply_condensed(x, y)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / a.reps
    n_c = g.n_skeleton()
    print(f"p={a.p} n={a.n}x{a.n}x{nz}: {ms:.3f} ms/apply, {16 * n_c / ms / 1e6:.1f} GB/s algorithmic, "
          f"{g.n_lattice / ms / 1e6:.2f} GDOF/s")
    if a.pcg:
        b = ctx.skeleton()
        ctx.sc_fill_random(7, b)
        ctx.sc_pcg_start(b, y, rtol=0.0)
        ev0.record()
        ctx.sc_pcg_iterate(a.pcg)
        ev1.record()
        torch.cuda.synchronize()
        print(f"pcg: {ev0.elapsed_time(ev1) / a.pcg:.3f} ms/iter")


if __name__ == "__main__":
    main()
