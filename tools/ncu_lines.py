"""Per-source-line instruction / stall attribution of one ncu report
(--page source, cuda+sass): python tools/ncu_lines.py report.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = collections.defaultdict(lambda: [0, 0, collections.Counter(), ""])
ops = collections.Counter()
cur = curline = hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        iE = hdr.index("Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if r[0] != "":
        curline = (cur, r[0])
        agg[curline][3] = r[1].strip()[:80]
        continue
    try:
        n = int(r[iE] or 0)
        s = int(r[iS] or 0)
    except (ValueError, IndexError):
        continue
    a = agg[curline]
    a[0] += n
    a[1] += s
    o = r[3].strip().split()
    if o:
        op = (o[1] if o[0].startswith("@") else o[0]).split(".")[0]
        a[2][op] += n
        ops[op] += n
tot = sum(v[0] for v in agg.values()) or 1
stot = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot}")
print("opcodes:", ", ".join(f"{o} {n / tot * 100:.1f}%" for o, n in ops.most_common(16)))
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}% st{v[1] / stot * 100:5.1f}% {k[0]}:{k[1]} {v[3][:60]} | "
          f"{dict(v[2].most_common(4))}")
