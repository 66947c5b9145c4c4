"""Small operator / PCG runs for compute-sanitizer (racecheck / synccheck / memcheck)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import __graft_entry__
__graft_entry__.build()
from paper_1601_08179_b200 import context_for_grid
import synth
os.environ["SC_SMALL_V1"] = "0"
for op, p, ne in [("v7", 5, (20, 5, 4)), ("v7", 8, (9, 4, 5)), ("v7", 12, (3, 3, 3)), ("big", 12, (3, 3, 3)),
                  ("big", 20, (2, 2, 2)), ("big", 32, (2, 2, 2))]:
    os.environ["SC_OP"] = op
    g = synth.small_grid(p, ne, 1.0)
    ctx = context_for_grid(g, device=0)
    x, y = ctx.skeleton(), ctx.skeleton()
    ctx.sc_fill_random(1, x)
    ctx.sc_apply_condensed(x, y)
    rep = ctx.sc_pcg_solve(x, y, rtol=1e-8, maxit=5)
    torch.cuda.synchronize()
    print(op, p, ctx.operator_kernel(), float(y.norm()), flush=True)
