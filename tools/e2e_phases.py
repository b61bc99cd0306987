"""Where the end-to-end time of config 2 goes: coefficient upload, field upload,
the 500 steps, field download (pinned host buffers, as bench.py's e2e)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4539_b200 as Y  # noqa: E402

n, steps = int(os.environ.get("N", "256")), int(os.environ.get("STEPS", "500"))


def pin(shape):
    return torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()


shapes = [Y.comp_extents(n, n, n, c)[::-1] for c in range(6)]
host_f = [pin(sh) for sh in shapes]
host_o = [pin(sh) for sh in shapes]
for a in host_f:
    a[...] = 0.0
med = Y.host_medium_slab(n, n, n, 0, n, 1, -1, [pin((n, n, n)) if q == Y.CB else None for q in range(4)])
t = np.arange(steps + 16, dtype=np.float64)
tab = np.exp(-((t - 40.0) / 12.0) ** 2).astype(np.float32)
for rep in range(3):
    s = Y.Simulation(n, n, n, variant=Y.VARIANT_TB2)
    s.add_source(Y.EZ, n // 2, n // 2, n // 2, tab)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.set_cell_coeffs(Y.CB, med[Y.CB])
    s.synchronize()
    t1 = time.perf_counter()
    s.upload(host_f)
    s.synchronize()
    t2 = time.perf_counter()
    s.run(steps)
    t3 = time.perf_counter()
    s.download(out=host_o)
    t4 = time.perf_counter()
    s.close()
    print(f"coeffs {1e3*(t1-t0):.2f} ms, fields up {1e3*(t2-t1):.2f} ms, run {1e3*(t3-t2):.2f} ms, "
          f"down {1e3*(t4-t3):.2f} ms, total {1e3*(t4-t0):.2f} ms -> {n**3*steps/(t4-t0)/1e9:.1f} Gcell/s")
