"""Per-warp, per-phase cycle split of the tile-column operator (build with SC_EXP=9; lane 0 of
each warp accumulates clock64 deltas between the SC_PHASE marks)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1601_08179_b200 import context_for_grid, capi
from synth import small_grid
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
pdeg = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = small_grid(pdeg, (n, n, n), 1.0)
ctx = context_for_grid(g)
x, y = ctx.skeleton(), ctx.skeleton()
ctx.sc_fill_random(5, x)
ctx.sc_apply_condensed(x, y)
torch.cuda.synchronize()
lib = capi.load()
buf = (ctypes.c_ulonglong * 128)()
lib.sc_exp_phase_cycles(buf)
names = {0: "wait loads", 1: "zero+edgesum", 3: "phase A", 4: "phase B", 5: "bar r0", 10: "round 0",
         11: "bar r1", 12: "round 1", 2: "sync", 6: "edges", 7: "finalize", 8: "finish"}
steps = None
tot0 = sum(buf[k] for k in range(16))
print(f"{'phase':14s}" + "".join(f"  w{w:d}" for w in range(8)) + "   (% of warp-0 total)")
for k in (0, 1, 3, 4, 5, 10, 11, 12, 2, 6, 7, 8):
    print(f"{names[k]:14s}" + "".join(f"{100 * buf[w * 16 + k] / tot0:5.1f}" for w in range(8)))
