import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1601_08179_b200 import context_for_grid, capi
from synth import small_grid
g = small_grid(8, (128, 128, 128), 1.0)
ctx = context_for_grid(g)
x, y = ctx.skeleton(), ctx.skeleton()
ctx.sc_fill_random(5, x)
ctx.sc_apply_condensed(x, y)
torch.cuda.synchronize()
lib = capi.load()
buf = (ctypes.c_ulonglong * 16)()
lib.sc_exp_phase_cycles(buf)
names = ["wait loads", "zero+sD", "volume loop", "volume E/N out", "z-output", "reductions", "edge primary", "publish", "owned+park+finish"]
tot = sum(buf[i] for i in range(9))
for i in range(9):
    print(f"{names[i]:14s} {buf[i] / tot * 100:5.1f}%")
