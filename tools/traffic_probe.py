"""DRAM bytes per cell-update of the two-step kernel vs grid shape (run under
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_tb2).

usage: python tools/traffic_probe.py NX NY NZ [STEPS]  (eps medium seed 4, random fields)
Separates the x-halo from the y-halo share of the read excess: a grid one
tile wide (NX = 128) has no x-neighbours, one tile tall (NY = 8) none in y."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4539_b200 as yb  # noqa: E402

nx, ny, nz = (int(a) for a in sys.argv[1:4])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 8
variant = yb.VARIANT_FUSED if os.environ.get("TP_VARIANT") == "fused" else yb.VARIANT_TB2
with yb.Simulation(nx, ny, nz, variant=variant) as s:
    s.generate_medium(4, -1)
    s.fill(3)
    s.run(4)
    s.synchronize()
    ms = s.run_timed(steps)
    print(f"{nx}x{ny}x{nz} {steps} steps: {nx * ny * nz * steps / ms / 1e6:.1f} Gcell/s, cell-updates {nx * ny * nz * steps}")
