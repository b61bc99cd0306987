"""A/B of the two-step kernel's TMA stage count on a large grid (env YB_STAGES2
is read at the first launch, so each setting runs in its own process).

usage: python tools/stage_ab2.py NX NY NZ [EPS_SEED]   (EPS_SEED < 0: vacuum, no per-cell array)"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 5 and sys.argv[5] == "child":
    import paper_1301_4539_b200 as yb
    nx, ny, nz, es = (int(a) for a in sys.argv[1:5])
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        if es >= 0:
            s.generate_medium(es, -1)
        s.fill(3)
        s.run(8)
        s.synchronize()
        ms = min(s.run_timed(20) for _ in range(3))
        print(f"{nx}x{ny}x{nz} eps={es} stages={s.info()['stages']} {nx * ny * nz * 20 / ms / 1e6:.1f} Gcell/s")
    sys.exit(0)
args = sys.argv[1:4] + [sys.argv[4] if len(sys.argv) > 4 else "-1"]
for rep in range(2):
    for st in ("2", "3"):
        env = dict(os.environ, YB_STAGES2=st)
        r = subprocess.run([sys.executable, __file__, *args, "child"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or ("failed: " + r.stderr.strip()[-300:]))
