"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source line:
instructions executed and stall samples, top N lines.
    ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = []
for r in rows:
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Line No") and r[0].isdigit():
        ie = hdr.index("Instructions Executed")
        ss = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            out.append((int(r[ie]), int(r[ss]), int(r[0]), r[1][:110]))
        except ValueError:
            pass
tot_i = sum(o[0] for o in out) or 1
tot_s = sum(o[1] for o in out) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"total warp-instr {tot_i}, samples {tot_s}")
for ie, ss, ln, src in sorted(out, key=lambda o: -o[1])[:n]:
    print(f"{ln:5d} instr {100 * ie / tot_i:5.1f}%  stall {100 * ss / tot_s:5.1f}%  {src.strip()}")
