"""Measured FP64 (DFMA) peak of this B200, for the FP64 roofline of the p >= 16 operator
(VERDICT r1 asked for it in a committed JSON with its clock record).

    python tools/fp64_peak.py [--out profiles/fp64_peak.json]

Compiles tools/microbench.cu (DFMA loop: 8 independent FMA chains per thread, 8 x 148 CTAs of
256 threads, best of 10 launches) and samples nvidia-smi clocks while it runs.
"""
import argparse
import json
import os
import re
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "fp64_peak.json"))
    a = ap.parse_args()
    exe = os.path.join(tempfile.mkdtemp(), "microbench")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                           os.path.join(ROOT, "tools", "microbench.cu")])
    sys.path.insert(0, ROOT)
    from bench import Clocks
    clk = Clocks(0)
    time.sleep(0.3)
    out = subprocess.check_output([exe], text=True)
    c = clk.stop()
    m = re.search(r"DFMA: ([0-9.]+) TFLOP/s fp64 \(([0-9.]+) FMA/clk/SM at ([0-9.]+) MHz", out)
    rec = {"fp64_tflops": float(m.group(1)), "fma_per_clk_per_sm_at_nominal": float(m.group(2)),
           "nominal_mhz": float(m.group(3)), "clocks": c, "raw": out.strip().splitlines(),
           "how": "tools/microbench.cu k_dfma: 8 x 148 CTAs x 256 threads, 8 independent DFMA chains, "
                  "16-way unrolled, 2000 iterations, best of 10 launches (CUDA events)",
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    with open(a.out, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
