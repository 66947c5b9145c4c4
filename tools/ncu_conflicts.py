import collections, csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True).stdout.decode("utf-8", "replace")
hdr=None; fname=""; cur=None
agg = collections.defaultdict(lambda: [0,0,0,0])
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0]: cur = f"{fname}:{r[0]} {r[1].strip()[:80]}"
    if r[2]:
        def g(k):
            try: return float(r[hdr.index(k)] or 0)
            except: return 0.0
        a = agg[cur]
        a[0] += g("L1 Wavefronts Shared Excessive"); a[1] += g("L1 Wavefronts Shared"); a[2] += g("Instructions Executed"); a[3] += g("Warp Stall Sampling (All Samples)")
tot = sum(v[0] for v in agg.values()); tots=sum(v[3] for v in agg.values())
print("excess wavefronts total", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv)>2 else 20]:
    print(f"{100*v[0]/max(tot,1):5.1f}% excess  {v[1]:12.0f} wf  {100*v[3]/tots:5.1f}% stall  {k}")
