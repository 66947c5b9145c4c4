"""Per-phase cycle split of the tile-column operator (build with SC_EXP=9; thread 0 of each CTA
accumulates clock64 deltas between the SC_PHASE marks)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1601_08179_b200 import context_for_grid, capi
from synth import small_grid
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = small_grid(8, (n, n, n), 1.0)
ctx = context_for_grid(g)
x, y = ctx.skeleton(), ctx.skeleton()
ctx.sc_fill_random(5, x)
ctx.sc_apply_condensed(x, y)
torch.cuda.synchronize()
lib = capi.load()
buf = (ctypes.c_ulonglong * 16)()
lib.sc_exp_phase_cycles(buf)
names = {0: "wait loads", 1: "zero+edge sums", 2: "condensed+faces", 6: "edge primary", 7: "publish",
         8: "owned+park+finish"}
tot = sum(buf[i] for i in range(16))
for i in range(16):
    if buf[i]:
        print(f"{names.get(i, str(i)):18s} {buf[i] / tot * 100:5.1f}%")
