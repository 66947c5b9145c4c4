#!/usr/bin/env python
"""Benchmark of the hot path: BT-PCG iterations of the condensed SEM Helmholtz solver.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg5]

A "step" is one BT-PCG iteration (scatter, TPT condensed
operator, gather, dot products, vector updates, diagonal preconditioner) on the
BASELINE configs[4] workload (128^3 elements, p=8, lambda=1, seeded uniform[-1,1]
right-hand side in the transformed basis, z-slabs over the ranks).  value = GLL
unknowns N x iterations / second over all ranks (GDOF/s; equivalently PCG
s/iter/unknown = 1e-9 / value).  Inputs (2.9 GB per vector) are far larger than L2,
so no flush is needed between iterations.

--impl reference times the CPU oracle (oracle/, the paper's method as a dense Schur
complement + block-Jacobi PCG) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "condensed-operator GDOF/s (fp64) and PCG s/iter/unknown at 1/2/4/8 B200 vs roofline"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=20, help="elements per direction of the oracle sample")
    return ap.parse_args()


def workload(name):
    import synth
    if name == "cfg5":
        return synth.cfg5()
    if name == "cfg2":
        return synth.cfg2()
    if name.startswith("cfg3:"):
        return synth.cfg3(int(name.split(":")[1]))
    if name.startswith("cfg4:"):
        return synth.cfg4(int(name.split(":")[1]))
    raise SystemExit(f"unknown config {name}")


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            mp = json.load(fh)
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def oracle_sample(grid, n_side, iters=None, budget_s=15.0, threads=None):
    """Time the oracle's PCG iteration on a bounded sample (n_side^3 elements, same p / lambda).
    threads: limit the BLAS threads (threadpoolctl), e.g. 1 for the paper's single core."""
    if threads is not None:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=threads):
            res = oracle_sample(grid, n_side, iters, budget_s, None)
        res["cores"] = threads
        return res
    import numpy as np
    from oracle import operator, solve, pcg
    from synth import small_grid, lattice_random
    g = small_grid(grid.p, (n_side, n_side, n_side), grid.lam)
    op = operator.AssembledCondensedOperator(g)
    P = solve.BlockJacobi(op)
    b = lattice_random(5, g.ne, g.p).ravel()
    pcg.pcg(op.apply, P.apply, b, rtol=0, fixed_iters=1)      # warm-up
    t0 = time.perf_counter()
    n = 0
    while True:
        pcg.pcg(op.apply, P.apply, b, rtol=0, fixed_iters=2)
        n += 2
        if iters is not None and n >= iters:
            break
        if iters is None and time.perf_counter() - t0 > budget_s:
            break
    t = (time.perf_counter() - t0) / n
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    return {"value": g.n_lattice / t / 1e9, "unit": "GDOF/s", "cores": int(cores), "kind": "oracle",
            "sample": f"{n_side}^3 elements p={g.p} lambda={g.lam} (N={g.n_lattice}), {n} BT-equivalent "
                      f"block-Jacobi PCG iterations of the dense-Schur oracle, {t * 1e3:.1f} ms/iter",
            "s_per_iter": t}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    grid = workload(args.config)
    n_side = args.cpu_sample
    # oracle_sample runs one untimed warm-up iteration itself (it includes the dense Schur setup)
    res = oracle_sample(grid, n_side, iters=max(2, args.steps // 2 * 2))
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": "GDOF/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["s_per_iter"] * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} oracle sample {n_side}^3 elements", "p": grid.p,
                       "lambda": grid.lam},
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": res["value"], "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import __graft_entry__
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier(device_ids=[local])      # every rank loads the library rank 0 just built
    from paper_1601_08179_b200 import capi
    from paper_1601_08179_b200.solver import Context
    if world > 1:
        lib = capi.load()
        idbuf = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            import ctypes
            raw = ctypes.create_string_buffer(128)
            assert lib.sc_nccl_unique_id(raw) == 0
            idbuf.copy_(torch.frombuffer(bytearray(raw.raw), dtype=torch.uint8))
        dist.broadcast(idbuf, 0)
        import ctypes
        comm = ctypes.c_void_p()
        st = lib.sc_nccl_comm_init(bytes(idbuf.cpu().numpy().tobytes()), world, rank, local, ctypes.byref(comm))
        assert st == 0, st
        comm = comm.value
    else:
        comm = None

    grid = workload(args.config)
    ctx = Context(grid.p, grid.ne, (grid.hx, grid.hy, grid.hz), grid.lam, device=local, nccl_comm=comm,
                  rank=rank, nranks=world)
    L = ctx.layout
    N_global = int(L.n_lattice_global)
    n_c_local = int(L.n_total)
    nI = grid.p - 1
    ne_local = L.ne_local[0] * L.ne_local[1] * L.ne_local[2]
    # exact skeleton length of the slab (the algorithmic N_c, no padding)
    nx, ny, nz = L.ne_local
    N_c_local = (nx * grid.p + 1) * (ny * grid.p + 1) * (nz * grid.p + 1) - ne_local * nI ** 3
    stream = torch.cuda.current_stream(dev)

    b = ctx.skeleton()
    x = ctx.skeleton()
    ctx.sc_fill_random(5, b)           # cfg5: b~ seed 5, uniform[-1,1] on free skeleton DOFs
    torch.cuda.synchronize(dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- BT-PCG iterations (the step) ----
    ctx.sc_pcg_start(b, x, rtol=0.0, maxit=1 << 30)
    ctx.sc_pcg_iterate(args.warmup)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    clocks = Clocks(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = ctx.launch_count()
    ctx.sc_profile_enable(True)
    ev0.record(stream)
    ctx.sc_pcg_iterate(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    launches = ctx.launch_count() - n0
    op_ms_total, op_n = ctx.sc_profile_read()
    ctx.sc_profile_enable(False)
    t_ms = max_over_ranks(ev0.elapsed_time(ev1))
    rep = ctx.sc_pcg_status()
    ms_step = t_ms / args.steps
    value = N_global * args.steps / (t_ms * 1e-3) / 1e9

    # ---- operator alone (K applications, p -> q), for the operator GDOF/s ----
    q = ctx.skeleton()
    for _ in range(2):
        ctx.sc_apply_condensed(b, q)
    torch.cuda.synchronize(dev)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ctx.sc_apply_condensed(b, q)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    op_apply_ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps

    # ---- roofline of the dominant kernel (condensed operator), inside the PCG step ----
    hbm, hbm_src = peaks()
    kern_ms = op_ms_total / max(op_n, 1)
    alg_bytes = 16.0 * N_c_local                     # skeleton read once + written once
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.config}:n{world}")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic, "kernel": "k_apply (TPT condensed operator + assembly)",
                "kernel_ms": kern_ms, "kernel_share_of_step": kern_ms / ms_step,
                "algorithmic_bytes_per_launch": alg_bytes, "peak_source": f"{hbm_src} hbm_gbs"}

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        hb = torch.empty(ctx.n_total, dtype=torch.float64, pin_memory=True)
        hx = torch.empty(ctx.n_total, dtype=torch.float64, pin_memory=True)
        hb.copy_(b.cpu())
        torch.cuda.synchronize(dev)
        barrier()
        t0 = time.perf_counter()
        ctx.sc_pcg_solve_host(hb, hx, rtol=0.0, maxit=args.steps)
        torch.cuda.synchronize(dev)
        t_e2e = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": N_global * args.steps / t_e2e / 1e9, "unit": "GDOF/s",
               "h2d_bytes_per_step": 8 * ctx.n_total * world, "d2h_bytes_per_step": 8 * ctx.n_total * world,
               "note": f"one sc_pcg_solve_host call of {args.steps} iterations incl. H2D of b and D2H of x "
                       f"(pinned), wall clock"}
        del hb, hx

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = oracle_sample(grid, args.cpu_sample)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        # the paper ran on one core: the same oracle with one BLAS thread
        one = oracle_sample(grid, max(4, args.cpu_sample // 2), budget_s=8.0, threads=1)
        cpu["one_core"] = {k: one[k] for k in ("value", "unit", "cores", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {grid.ne[0]}x{grid.ne[1]}x{grid.ne[2]} elements p={grid.p} "
                                   f"lambda={grid.lam}, BT-PCG iterations, seeded uniform[-1,1] rhs",
                       "p": grid.p, "elements": grid.n_elements, "N": N_global, "N_c": grid.n_skeleton(),
                       "parallelism": f"z-slab x{world}", "l2": "inputs larger than L2 (no flush)"},
            "pcg_s_per_iter_per_unknown": ms_step * 1e-3 / N_global,
            "operator": {"gdofs": N_global / (op_apply_ms * 1e-3) / 1e9, "ms_per_apply": op_apply_ms,
                         "kernel_ms_in_step": kern_ms},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk, "pcg_iters_done": rep.iters,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` without a torchrun environment: re-exec as N ranks on this node
    (the driver's own launch sets WORLD_SIZE and never gets here)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
