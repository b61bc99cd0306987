"""A/B of the two-step kernel's L2 prefetch distance (YB_TB2_PF) and stage
count (YB_STAGES2), each setting in its own process (read at the first launch).

usage: python tools/pf_ab.py [REPS]   (configs 4, 3, 2 geometry and media, random fields)"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

GRIDS = {"c4": (1024, 1024, 512, 4, -1), "c3": (512, 512, 512, 2, 2), "c2": (256, 256, 256, 1, -1)}

if len(sys.argv) > 2 and sys.argv[1] == "child":
    import paper_1301_4539_b200 as yb
    nx, ny, nz, es, ss = GRIDS[sys.argv[2]]
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        s.generate_medium(es, ss)
        s.fill(3)
        s.run(8)
        s.synchronize()
        ms = min(s.run_timed(20) for _ in range(3))
        print(f"{sys.argv[2]} stages={s.info()['stages']} {nx * ny * nz * 20 / ms / 1e6:.1f}")
    sys.exit(0)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
settings = os.environ.get("PF_SET", "0 1 2 3 4").split()
for rep in range(reps):
    for cfg in GRIDS:
        row = []
        for pf in settings:
            env = dict(os.environ, YB_TB2_PF=pf)
            r = subprocess.run([sys.executable, __file__, "child", cfg], env=env, capture_output=True, text=True)
            row.append(f"pf={pf}: " + (r.stdout.strip().split()[-1] if r.returncode == 0 else "FAIL"))
        print(cfg, " | ".join(row), flush=True)
