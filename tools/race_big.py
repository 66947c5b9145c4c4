"""v4 operator (n_I >= 8) on small multi-colour grids, for compute-sanitizer racecheck /
synccheck (kernels_big.cu had an index form that 'gave wrong vertex values in some
builds').  python tools/race_big.py [p ...]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SC_SMALL_V1", "0")
import torch
from paper_1601_08179_b200 import context_for_grid
from synth import small_grid, nonuniform_grid

ps = [int(a) for a in sys.argv[1:]] or [9, 12, 16, 17, 24, 25, 32]
for p in ps:
    for g in (small_grid(p, (3, 2, 2), 1.0), nonuniform_grid(p, (2, 2, 3), 0.5, seed=7)):
        ctx = context_for_grid(g, device=0)
        x, y = ctx.skeleton(), ctx.skeleton()
        ctx.sc_fill_random(3, x)
        ctx.sc_apply_condensed(x, y)
        torch.cuda.synchronize()
        print(p, g.ne, g.uniform(), "ok", float(y.norm()), flush=True)
