"""Operator time on a graded (non-uniform) grid: v4 per-CTA coefficients vs the v1 kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_1601_08179_b200 import context_for_grid
from synth import small_grid
for p, n in ((16, 32), (12, 40)):
    g = small_grid(p, (n, n, n), 0.0)
    r = np.random.default_rng(1)
    g.hx = r.uniform(0.5, 1.5, n) / n; g.hy = r.uniform(0.5, 1.5, n) / n; g.hz = r.uniform(0.5, 1.5, n) / n
    for v1 in ("0", "1"):
        os.environ["SC_APPLY_V1"] = v1
        ctx = context_for_grid(g)
        x, y = ctx.skeleton(), ctx.skeleton()
        ctx.sc_fill_random(3, x)
        ctx.sc_apply_condensed(x, y); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): ctx.sc_apply_condensed(x, y)
        e1.record(); torch.cuda.synchronize()
        print(f"p={p} n={n} graded, {'v1' if v1 == '1' else 'v4'}: {e0.elapsed_time(e1) / 5:.3f} ms/apply", flush=True)
        del ctx, x, y
        torch.cuda.empty_cache()
