"""Streamed upload phases (yb_run_streamed) on one config shape: each phase of the
phase-by-phase flow timed alone (coefficient upload, field upload, run, readback), then
yb_run_streamed with a short run (8 steps: transfer-bound, shows what the tile-row copies
cost) and with the full step count. Env: NX/NY/NZ (default config 3), STEPS (100),
CELLS=1|4 (per-cell arrays), FIELDS=1 (seeded initial fields uploaded)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4539_b200 as Y  # noqa: E402

nx, ny, nz = (int(os.environ.get(k, d)) for k, d in (("NX", 512), ("NY", 512), ("NZ", 512)))
steps = int(os.environ.get("STEPS", "100"))
four = os.environ.get("CELLS", "4") == "4"
fields = os.environ.get("FIELDS", "1") == "1"


def pin(shape):
    return torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()


out = [pin(Y.comp_extents(nx, ny, nz, c)[::-1]) for c in range(6)]
want = (0, 1, 2, 3) if four else (1,)
med = Y.host_medium_slab(nx, ny, nz, 0, nz, 5 if four else 4, 5 if four else -1,
                         [pin((nz, ny, nx)) if q in want else None for q in range(4)])
cells = {q: med[q] for q in want}
hf = None
if fields:
    hf = [pin(Y.comp_extents(nx, ny, nz, c)[::-1]) for c in range(6)]
    Y.host_fields_slab(nx, ny, nz, 0, nz, 6, out=hf)
t = np.arange(steps + 16, dtype=np.float64)
tab = np.exp(-((t - 40.0) / 12.0) ** 2).astype(np.float32)
gb_up = (sum(a.nbytes for a in cells.values()) + (sum(a.nbytes for a in hf) if hf else 0)) / 1e9
gb_dn = sum(a.nbytes for a in out) / 1e9
print(f"grid {nx}x{ny}x{nz}, {steps} steps, up {gb_up:.2f} GB, down {gb_dn:.2f} GB", flush=True)


def sim():
    s = Y.Simulation(nx, ny, nz, variant=Y.VARIANT_TB2)
    if not fields:
        s.add_source(Y.EZ, nx // 2, ny // 2, nz // 2, tab)
    s.synchronize()
    return s


cu = nx * ny * nz
for rep in range(2):
    s = sim()
    t0 = time.perf_counter()
    s.set_cell_coeffs_many(cells)
    t1 = time.perf_counter()
    if hf:
        s.upload(hf)
    t2 = time.perf_counter()
    s.run(steps)
    t3 = time.perf_counter()
    s.download(out=out)
    t4 = time.perf_counter()
    s.close()
    print(f"rep {rep} phases: coeffs {1e3*(t1-t0):.1f} ms ({sum(a.nbytes for a in cells.values())/1e9/(t1-t0):.1f} GB/s), "
          f"fields {1e3*(t2-t1):.1f}, run {1e3*(t3-t2):.1f} ({cu*steps/(t3-t2)/1e9:.1f} Gcell/s), readback {1e3*(t4-t3):.1f} "
          f"({gb_dn/(t4-t3):.1f} GB/s), sum {1e3*(t4-t0):.1f} ms ({cu*steps/(t4-t0)/1e9:.1f} Gcell/s)", flush=True)
    for n in (8, steps):
        s = sim()
        t5 = time.perf_counter()
        s.run_streamed(n, cells, hf, out=out)
        t6 = time.perf_counter()
        up = s.info()["streamed_uploads"]
        s.close()
        print(f"rep {rep} run_streamed({n}): {1e3*(t6-t5):.1f} ms ({cu*n/(t6-t5)/1e9:.1f} Gcell/s, streamed={up}; "
              f"{gb_up/(t6-t5):.1f} GB/s up if transfer-bound)", flush=True)
    s = sim()
    t7 = time.perf_counter()
    s.set_cell_coeffs_many(cells)
    if hf:
        s.upload(hf)
    s.run_to_host(steps, out=out)
    t8 = time.perf_counter()
    s.close()
    print(f"rep {rep} upload then run_to_host: {1e3*(t8-t7):.1f} ms ({cu*steps/(t8-t7)/1e9:.1f} Gcell/s)", flush=True)
