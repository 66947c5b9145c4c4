"""Summarise ncu outputs (launch list CSV + one --set full report) into profiles/.

    python tools/ncu_summary.py --tag r1a --launches gpurun_out/launches_r1a.csv \
        --full gpurun_out/prof_cfg5_r1a.ncu-rep --config cfg5:n1 --n-c 357567489

Writes profiles/<tag>_summary.md and updates profiles/traffic.json (dram bytes per launch of
the condensed-operator kernel, keyed by bench config).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem, CTAs/SM)"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "ns")
                scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(unit, 1e-6)
                out.append((d["Kernel Name"].split("(")[0], v * scale))
    return out


def full(path):
    """Every kernel of the capture (one operator application: v7 = pass A + pass B): name and metrics."""
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        res = {}
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                res[k] = (name, v[i], u[i])
        out.append((v[h.index("Kernel Name")] if "Kernel Name" in h else "?", res))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--config", default="cfg5:n1")
    ap.add_argument("--n-c", type=float, default=0.0, help="skeleton length N_c (algorithmic bytes 16 N_c)")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary {a.tag}", ""]
    if a.note:
        lines += [a.note, ""]
    if a.launches:
        ls = launches(a.launches)
        tot = sum(t for _, t in ls)
        agg = collections.OrderedDict()
        for k, t in ls:
            c = agg.setdefault(k, [0, 0.0])
            c[0] += 1
            c[1] += t
        lines += ["## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold, serialised)", "",
                  f"source: `{os.path.basename(a.launches)}`, {len(ls)} launches, {tot:.3f} ms total", "",
                  "| kernel | launches | total ms | mean ms | share |", "|---|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {n} | {t:.3f} | {t / n:.4f} | {t / tot * 100:.1f}% |")
        lines.append("")
    if a.full:
        traffic = 0.0
        dsec_tot = 0.0
        for kname, res in full(a.full):
            lines += [f"## `--set full` capture of `{kname[:90]}`", "", f"source: `{os.path.basename(a.full)}`", "",
                      "| metric | value | unit |", "|---|---|---|"]
            for k, (name, v, u) in res.items():
                lines.append(f"| {name} (`{k}`) | {v} | {u} |")
            lines.append("")
            try:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                rd = float(res["dram__bytes_read.sum"][1].replace(",", "")) * scale.get(res["dram__bytes_read.sum"][2], 1)
                wr = float(res["dram__bytes_write.sum"][1].replace(",", "")) * scale.get(res["dram__bytes_write.sum"][2], 1)
                dur = float(res["gpu__time_duration.sum"][1].replace(",", ""))
                dunit = res["gpu__time_duration.sum"][2]
                dsec = dur * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(dunit, 1e-9)
                traffic += rd + wr
                dsec_tot += dsec
                lines += [f"DRAM traffic of this kernel: {(rd + wr) / 1e9:.3f} GB in {dsec * 1e3:.3f} ms "
                          f"({(rd + wr) / dsec / 1e9:.1f} GB/s)", ""]
            except Exception as e:  # pragma: no cover
                lines.append(f"(traffic not computed: {e})")
        if traffic > 0:
            lines += [f"## One operator application (all kernels above)", "",
                      f"DRAM traffic per application: {traffic / 1e9:.3f} GB, {dsec_tot * 1e3:.3f} ms under ncu"]
            if a.n_c:
                alg = 16 * a.n_c
                lines += [f"algorithmic bytes (16 N_c): {alg / 1e9:.3f} GB -> traffic / algorithmic = {traffic / alg:.3f}",
                          f"achieved DRAM bandwidth under ncu (cold, clock-control none): {traffic / dsec_tot / 1e9:.1f} GB/s"]
            tpath = os.path.join(ROOT, "profiles", "traffic.json")
            tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
            tj[a.config] = traffic
            json.dump(tj, open(tpath, "w"), indent=1)
    out = os.path.join(ROOT, "profiles", f"{a.tag}_summary.md")
    open(out, "w").write("\n".join(lines) + "\n")
    print(out)


if __name__ == "__main__":
    main()
