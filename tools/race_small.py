"""Small operator + PCG run for compute-sanitizer (racecheck / synccheck / memcheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1601_08179_b200 import context_for_grid
from synth import small_grid
for p, ne in [(2, (2, 2, 2)), (8, (9, 5, 2))]:
    g = small_grid(p, ne, 1.0)
    ctx = context_for_grid(g, device=0)
    x, y = ctx.skeleton(), ctx.skeleton()
    ctx.sc_fill_random(3, x)
    ctx.sc_apply_condensed(x, y)
    ctx.sc_pcg_start(x, y, rtol=0.0, maxit=4)
    ctx.sc_pcg_iterate(4)
    torch.cuda.synchronize()
    print(p, ne, "ok", float(y.norm()))
