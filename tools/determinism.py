"""Repeat the operator on fixed inputs and check bitwise reproducibility (race detector)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_1601_08179_b200 import context_for_grid
from synth import small_grid
for p, ne in [(2, (2, 2, 2)), (3, (2, 2, 2)), (8, (9, 5, 2)), (4, (17, 9, 5)), (8, (33, 17, 6))]:
    g = small_grid(p, ne, 1.0)
    ctx = context_for_grid(g, device=0)
    x = ctx.skeleton(); ctx.sc_fill_random(3, x)
    y0 = ctx.skeleton(); ctx.sc_apply_condensed(x, y0)
    bad = 0; maxd = 0.0
    ys = [ctx.skeleton() for _ in range(8)]
    for rep in range(50):
        for y in ys:
            y.fill_(float("nan"))
            ctx.sc_apply_condensed(x, y)
        torch.cuda.synchronize()
        for y in ys:
            d = (y - y0).abs().max().item()
            if not (d == 0.0):
                bad += 1; maxd = max(maxd, d) if d == d else float("nan")
    print(f"p={p} ne={ne}: {bad} / 400 differ, max diff {maxd}", flush=True)
