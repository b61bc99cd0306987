"""Streamed readback phases (yb_run_to_host) on one config shape: the plain
multi-sweep run, the readback alone, and run_to_host with YB_DRAIN_TRACE=1
(kernel time of the skewed launch and when each tile row's copies ended).
Env: NX/NY/NZ (default config 4), STEPS (200), CELLS=1|4 (per-cell arrays),
FIELDS=1 (seeded initial fields). Medium generated on the device."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4539_b200 as Y  # noqa: E402

nx, ny, nz = (int(os.environ.get(k, d)) for k, d in (("NX", 1024), ("NY", 1024), ("NZ", 512)))
steps = int(os.environ.get("STEPS", "200"))
four = os.environ.get("CELLS", "1") == "4"
fields = os.environ.get("FIELDS") == "1"
os.environ["YB_DRAIN_TRACE"] = "1"
out = [torch.empty(Y.comp_extents(nx, ny, nz, c)[::-1], dtype=torch.float32, pin_memory=True).numpy()
       for c in range(6)]
t = np.arange(steps + 16, dtype=np.float64)
tab = np.exp(-((t - 40.0) / 12.0) ** 2).astype(np.float32)


def sim():
    s = Y.Simulation(nx, ny, nz, variant=Y.VARIANT_TB2)
    s.generate_medium(5 if four else 4, 5 if four else -1)
    if fields:
        s.fill(6)
    else:
        s.add_source(Y.EZ, nx // 2, ny // 2, nz // 2, tab)
    s.synchronize()
    return s


cells = nx * ny * nz * steps
for rep in range(2):
    s = sim()
    t0 = time.perf_counter()
    s.run(steps)
    t1 = time.perf_counter()
    s.download(out=out)
    t2 = time.perf_counter()
    s.close()
    s = sim()
    t3 = time.perf_counter()
    s.run_to_host(steps, out=out)
    t4 = time.perf_counter()
    streamed = s.info()["streamed_readbacks"]
    s.close()
    print(f"rep {rep}: run {1e3*(t1-t0):.1f} ms ({cells/(t1-t0)/1e9:.1f} Gcell/s), readback {1e3*(t2-t1):.1f} ms, "
          f"sum {1e3*(t2-t0):.1f}; run_to_host {1e3*(t4-t3):.1f} ms ({cells/(t4-t3)/1e9:.1f} Gcell/s, "
          f"streamed={streamed})", flush=True)
