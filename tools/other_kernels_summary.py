"""Summary of the non-cfg5 operator kernels (p2, rw, v4) from tools/gpu_prof_others.sh output:
per-apply duration and DRAM traffic (8 colour launches, ncu launch metrics) against the
algorithmic 16 N_c bytes, plus one --set full capture per kernel (issue, FP64 pipe, stalls).

    python tools/other_kernels_summary.py r1p > profiles/r1p_other_kernels.md
"""
import csv
import io
import subprocess
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r1p"
CASES = [(2, 297, "p2 row-warp"), (4, 148, "rw row-warp"), (16, 37, "v4 colour element-CTA"),
         (32, 19, "v4 colour element-CTA")]


def n_c(p, n):
    ni = p - 1
    faces = 3 * (n + 1) * n * n * ni * ni
    edges = 3 * n * (n + 1) * (n + 1) * ni
    return faces + edges + (n + 1) ** 3


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    mi, vi = h.index("Metric Name"), h.index("Metric Value")
    tot = {}
    for r in rows[1:]:
        tot[r[mi]] = tot.get(r[mi], 0.0) + float(r[vi].replace(",", ""))
    return tot


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    d = dict(zip(r[0], r[2]))
    st = sorted(((float(d[k]), k) for k in r[0] if k.startswith("smsp__average_warps_issue_stalled")
                 and k.endswith("per_issue_active.ratio") and d[k] not in ("", "n/a")), reverse=True)[:5]
    stalls = ", ".join("%s %.2f" % (k.replace("smsp__average_warps_issue_stalled_", "")
                                    .replace("_per_issue_active.ratio", ""), v) for v, k in st)
    return d, stalls


print(f"# Non-cfg5 operator kernels ({TAG}), cfg3 sizes\n")
print("Per apply = the 8 colour launches (ncu `--metrics gpu__time_duration.sum,dram__bytes_*`, cold,")
print("serialised); algorithmic bytes = 16 N_c. Full capture: one colour launch.\n")
print("| p | n | kernel | ms / apply (ncu) | DRAM GB / apply | traffic / algorithmic | DRAM TB/s | issue % | FP64 pipe % | warps / SM | regs | top stalls (per issue) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for p, n, name in CASES:
    t = launches(f"gpurun_out/traffic_{TAG}_p{p}.csv")
    ms = t["gpu__time_duration.sum"] / 1e6
    gb = (t["dram__bytes_read.sum"] + t["dram__bytes_write.sum"]) / 1e9
    alg = 16 * n_c(p, n) / 1e9
    d, stalls = full(f"gpurun_out/prof_{TAG}_p{p}.ncu-rep")
    print(f"| {p} | {n} | {name} | {ms:.3f} | {gb:.2f} | {gb / alg:.2f} | {gb / ms:.2f} | "
          f"{float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} | "
          f"{float(d['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']):.1f} | "
          f"{float(d['sm__warps_active.avg.per_cycle_active']):.1f} | {d['launch__registers_per_thread']} | {stalls} |")
