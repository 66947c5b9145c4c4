"""BASELINE configs[2] / SURVEY §8(d) cfg3: condensed-operator time per unknown against p.

    python tools/p_sweep.py [--ps 2,4,8,12,16,24,32] [--reps 20] [--out profiles/p_sweep.json]

For each p the uniform cube has n = round(594/p) elements per direction (about 2.1e8 GLL
unknowns), lambda = 1, and a seeded uniform[-1,1] skeleton vector (counter-based generator).
Times `reps` back-to-back applications with CUDA events after warm-up (inputs of 0.2-1.5 GB
per vector exceed L2).  Reports ms per application, GDOF/s = N / t, s per unknown, and the
roofline: HBM floor = 16 N_c bytes / measured copy bandwidth (MEASURED_PEAKS.json),
FP64 floor = the paper's 13 multiplications + 11 additions per interior point (24 n_e n_I^3 flop,
P:413 / Table 3) / the measured DFMA peak (profiles/fp64_peak.json); fraction of roofline =
max(the two floors) / t, each floor's own fraction reported too.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ps", default="2,4,8,12,16,24,32")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_1601_08179_b200 import context_for_grid
    from synth import cfg3
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    fpath = os.path.join(ROOT, "profiles", "fp64_peak.json")
    fp64 = json.load(open(fpath))["fp64_tflops"] if os.path.exists(fpath) else 37.2
    rows = []
    for p in [int(s) for s in a.ps.split(",")]:
        g = cfg3(p)
        ctx = context_for_grid(g)
        x, y = ctx.skeleton(), ctx.skeleton()
        ctx.sc_fill_random(3, x)
        for _ in range(3):
            ctx.sc_apply_condensed(x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.reps):
            ctx.sc_apply_condensed(x, y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        n_c = g.n_skeleton()
        t_hbm = 16.0 * n_c / (hbm * 1e9) * 1e3                                   # ms
        t_fp64 = 24.0 * g.n_elements * (p - 1) ** 3 / (fp64 * 1e12) * 1e3       # ms
        row = {"p": p, "n": g.ne[0], "N": g.n_lattice, "N_c": n_c, "ms_per_apply": ms,
               "gdofs": g.n_lattice / ms / 1e6, "s_per_unknown": ms * 1e-3 / g.n_lattice,
               "hbm_floor_ms": t_hbm, "fp64_floor_ms": t_fp64,
               "hbm_frac": t_hbm / ms, "fp64_frac": t_fp64 / ms,
               "bound": "hbm" if t_hbm >= t_fp64 else "fp64", "roofline_frac": max(t_hbm, t_fp64) / ms,
               "kernel": ctx.operator_kernel()}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del ctx, x, y
        torch.cuda.empty_cache()
    out = {"config": "cfg3: uniform cube, n = round(594/p) (halves up), lambda = 1, seeded uniform[-1,1] x",
           "hbm_peak_gbs": hbm, "fp64_peak_tflops": fp64, "fp64_peak_source": "profiles/fp64_peak.json (measured)",
           "sweep": rows}
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
