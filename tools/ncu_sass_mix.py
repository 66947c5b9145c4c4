"""Instruction mix of one kernel from an ncu --set full report (source page, cuda+sass view):
warp instructions executed per SASS opcode and per CUDA source line.
    python tools/ncu_sass_mix.py rep.ncu-rep [N]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True).stdout.decode("utf-8", "replace")
op = collections.Counter(); line = collections.Counter(); stall = collections.Counter()
hdr = None; fname = ""; cur = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0]:
        cur = f"{fname}:{r[0]} {r[1].strip()[:90]}"
    if r[2]:
        try:
            ie = int(r[hdr.index("Instructions Executed")] or 0)
            ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        opc = r[3].strip().split()
        o = opc[0] if opc else "?"
        if o.startswith("@"): o = opc[1] if len(opc) > 1 else o
        op[o.split(".")[0]] += ie
        line[cur] += ie; stall[cur] += ss
tot = sum(op.values()) or 1; tots = sum(stall.values()) or 1
print(f"total warp instructions {tot}")
for o, v in op.most_common(n): print(f"  {o:12s} {v:14d} {100*v/tot:5.1f}%")
print("top lines by instructions:")
for l, v in line.most_common(n): print(f"  {100*v/tot:5.1f}% instr {100*stall[l]/tots:5.1f}% stall  {l}")
