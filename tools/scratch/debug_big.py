"""Debug aid: v4 (n_I >= 8) against v1 per entity class (faces x/y/z, edges x/y/z, vertices)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_1601_08179_b200 import context_for_grid
from synth import small_grid

for p, ne in [(12, (2, 2, 2)), (12, (3, 3, 3)), (20, (3, 3, 3)), (17, (3, 3, 3))]:
    g = small_grid(p, ne, 1.0)
    os.environ["SC_APPLY_V1"] = "1"
    c1 = context_for_grid(g, device=0)
    del os.environ["SC_APPLY_V1"]
    c4 = context_for_grid(g, device=0)
    x0 = c4.skeleton()
    c4.sc_fill_random(3, x0)
    L = c4.layout
    ni = L.n_i
    for part in ("faces", "edges", "vertices"):
      x = torch.zeros_like(x0)
      lo, hi = {"faces": (L.off_face[0], L.off_edge[0]), "edges": (L.off_edge[0], L.off_vertex),
                "vertices": (L.off_vertex, L.off_vertex + L.n_vertices)}[part]
      x[lo:hi] = x0[lo:hi]
      y1, y4 = c1.skeleton(), c4.skeleton()
      c1.sc_apply_condensed(x, y1)
      c4.sc_apply_condensed(x, y4)
      torch.cuda.synchronize()
      o, n = L.off_vertex, L.n_vertices
      print(p, ne, part, "vertex max diff", float((y1[o:o+n] - y4[o:o+n]).abs().max()), "ref", float(y1[o:o+n].abs().max()))
    continue
    segs = [("fx", L.off_face[0], L.n_faces[0] * ni * ni), ("fy", L.off_face[1], L.n_faces[1] * ni * ni),
            ("fz", L.off_face[2], L.n_faces[2] * ni * ni), ("ex", L.off_edge[0], L.n_edges[0] * ni),
            ("ey", L.off_edge[1], L.n_edges[1] * ni), ("ez", L.off_edge[2], L.n_edges[2] * ni),
            ("v", L.off_vertex, L.n_vertices)]
    out = [f"p={p} ne={ne} total rel {float((y1 - y4).norm() / y1.norm()):.2e}"]
    for nm, o, n in segs:
        a, b = y1[o:o + n], y4[o:o + n]
        d = (a - b).abs()
        out.append(f"{nm}: max {float(d.max()):.2e} (ref max {float(a.abs().max()):.2e}) nbad {int((d > 1e-10 * float(a.abs().max() + 1e-300)).sum())}/{n}")
    print("\n  ".join(out), flush=True)
