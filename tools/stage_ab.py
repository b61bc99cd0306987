"""A/B of the two-step kernel's stage count on a vacuum grid (env YB_STAGES2
is read at first launch, so each setting runs in its own process)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1:
    import paper_1301_4539_b200 as yb
    n = int(sys.argv[1])
    with yb.Simulation(n, n, n, variant=yb.VARIANT_TB2) as s:
        s.fill(3)
        s.run(8)
        s.synchronize()
        ms = min(s.run_timed(40) for _ in range(3))
        print(f"n={n} stages={s.info()['stages']} {n ** 3 * 40 / ms / 1e6:.1f} Gcell/s")
    sys.exit(0)
for n in (256, 384):
    for st in ("2", "3"):
        env = dict(os.environ, YB_STAGES2=st)
        print(subprocess.run([sys.executable, __file__, str(n)], env=env, capture_output=True, text=True).stdout.strip() or "failed")
