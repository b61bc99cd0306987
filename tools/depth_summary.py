"""Summarise tools/depth_sweep.sh output: Gcell/s per depth (bench lines) and
ncu DRAM bytes per cell-update of the step kernels (all launches of the
profiled run: warm-up + timed steps).
usage: python tools/depth_summary.py DIR  (DIR = gpurun_out/sweep)"""
import csv
import json
import os
import sys

D = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep"
CELLS = 1024 * 1024 * 256
STEPS = 8  # --steps 4 --warmup 4 in the ncu pass
ALG = {"naive": 88, "fused": 64, "tb2": 32, "tb4": 16}
DEPTH = {"naive": 1, "fused": 2, "tb2": 4, "tb4": 8}
STEP_KERNELS = ("k_naive_", "k_fused", "k_tb2", "k_tb4")
for v in ("naive", "fused", "tb2", "tb4"):
    bp = os.path.join(D, f"bench_{v}.json")
    bp = bp if os.path.exists(bp) else os.path.join(D, f"bench_c5_{v}.json")
    b = json.loads(open(bp).read().strip().splitlines()[-1])
    tot = 0.0
    with open(os.path.join(D, f"ncu_{v}.csv")) as f:
        rows = [r for r in csv.reader(ln for ln in f if ln.startswith('"'))]
    hdr = rows[0]
    kn, mn, mv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    mu = hdr.index("Metric Unit")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for r in rows[1:]:
        if any(k in r[kn] for k in STEP_KERNELS) and r[mn] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[mv].replace(",", "")) * scale[r[mu]]
    print(f"| {DEPTH[v]} | {v} | {b['value']:.1f} | {ALG[v]} | {tot / (CELLS * STEPS):.1f} | "
          f"{b['ms_per_step']:.2f} ms/step |")
