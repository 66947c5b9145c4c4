"""Quick summary of an ncu --set full report: duration, DRAM, issue, warps, stall reasons."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    print(d.get("Kernel Name", "")[:60])
    for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
              "launch__grid_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sass__inst_executed_local_loads"]:
        if k in d:
            print(f"  {k:62s} {d[k]} {units[hdr.index(k)]}")
    st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("per_issue_active.ratio") and v not in ("", "n/a")]
    for k, v in sorted(st, key=lambda kv: -kv[1])[:8]:
        print(f"  stall {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v:.3f}")
