"""Where the end-to-end time goes: coefficient upload, field upload, the steps,
field download (pinned host buffers, as bench.py's e2e). Env: N (cube edge) or
NX/NY/NZ, STEPS, ZERO_START=1 (no field upload: configs 2 / 4)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4539_b200 as Y  # noqa: E402

n, steps = int(os.environ.get("N", "256")), int(os.environ.get("STEPS", "500"))
nx, ny, nz = (int(os.environ.get(k, n)) for k in ("NX", "NY", "NZ"))
zero_start = os.environ.get("ZERO_START") == "1"


def pin(shape):
    return torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()


shapes = [Y.comp_extents(nx, ny, nz, c)[::-1] for c in range(6)]
host_f = [pin(sh) for sh in shapes]
host_o = [pin(sh) for sh in shapes]
for a in host_f:
    a[...] = 0.0
med = Y.host_medium_slab(nx, ny, nz, 0, nz, 1, -1, [pin((nz, ny, nx)) if q == Y.CB else None for q in range(4)])
t = np.arange(steps + 16, dtype=np.float64)
tab = np.exp(-((t - 40.0) / 12.0) ** 2).astype(np.float32)
for rep in range(3):
    s = Y.Simulation(nx, ny, nz, variant=Y.VARIANT_TB2)
    s.add_source(Y.EZ, nx // 2, ny // 2, nz // 2, tab)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.set_cell_coeffs(Y.CB, med[Y.CB])
    s.synchronize()
    t1 = time.perf_counter()
    if not zero_start:
        s.upload(host_f)
    s.synchronize()
    t2 = time.perf_counter()
    s.run(steps)
    t3 = time.perf_counter()
    s.download(out=host_o)
    t4 = time.perf_counter()
    s.close()
    print(f"coeffs {1e3*(t1-t0):.2f} ms, fields up {1e3*(t2-t1):.2f} ms, run {1e3*(t3-t2):.2f} ms, "
          f"down {1e3*(t4-t3):.2f} ms, total {1e3*(t4-t0):.2f} ms -> {nx*ny*nz*steps/(t4-t0)/1e9:.1f} Gcell/s")
