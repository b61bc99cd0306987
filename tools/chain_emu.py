"""One-GPU emulation of the multi-GPU schedule with chained exchange periods
(yb_peer_run, k_tb2 MODE 4): a grid split into R z-slabs (R "ranks") that run
in ONE persistent launch — every sweep's boundary items wait in-kernel for the
neighbour slab, store their boundary planes into its ghost planes and signal —
against the same grid as one domain (multi-sweep launches). The ratio is the
schedule's own cost per GPU (extra chunk boundaries, peer stores, waits); over
NVLink the stores of a real run also cross the link, overlapped with the sweep.

usage: python tools/chain_emu.py CONFIG R [STEPS]   (CONFIG c2 | c4 | c5; R = 2..8 slabs)
  c4: strong scaling — the 1024^2 x 512 grid in R slabs (each rank 512/R planes)
  c2 / c5: weak scaling — R slabs of the config's own depth each (c2: 256^3 per rank)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4539_b200 as Y  # noqa: E402
from paper_1301_4539_b200.slabs import partition  # noqa: E402

cfg, R = sys.argv[1], int(sys.argv[2])
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
nx, ny, nzr, es, ss, fs = {"c2": (256, 256, 256, 1, -1, None), "c4": (1024, 1024, 512, 4, -1, None),
                           "c5": (1024, 1024, 256, 5, 5, 6)}[cfg]
nzg = nzr if cfg == "c4" else nzr * R


def make(**kw):
    s = Y.Simulation(nx, ny, kw.pop("nz"), variant=Y.VARIANT_TB2, **kw)
    s.generate_medium(es, ss)
    s.fill(fs if fs is not None else 3)
    return s


def rate(fn, sync):
    fn(4)
    sync()
    best = 1e30
    for _ in range(3):
        t0 = time.perf_counter()
        fn(steps)
        sync()
        best = min(best, time.perf_counter() - t0)
    return nx * ny * nzg * steps / best / 1e9


one = make(nz=nzg)
r_one = rate(lambda k: one.run(k, sync=False), one.synchronize)
r_one_chain = rate(lambda k: Y.peer_run([one], k), one.synchronize)  # the rank's (direct) MODE 4 kernel
one.close()
# the emulation kernel (slab arguments indexed in parameter space) over R unlinked domains: its own cost
doms = [make(nz=nzg // R) for _ in range(R)]
r_emu_free = rate(lambda k: Y.peer_run(doms, k), lambda: [s.synchronize() for s in doms])
for s in doms:
    s.close()
sims = [make(nz=n, z_offset=z0, nz_global=nzg) for z0, n in partition(nzg, R)]
for lo, hi in zip(sims[:-1], sims[1:]):
    lo.peer_link(1, hi)
    hi.peer_link(0, lo)
for s in sims:
    s.peer_push(False)
r_chain = rate(lambda k: Y.peer_run(sims, k), lambda: [s.synchronize() for s in sims])
info = sims[0].info()
for s in sims:
    s.close()
print(f"{cfg} {nx}x{ny}x{nzg} in {R} slabs ({steps} steps): one domain {r_one:.1f} Gcell/s "
      f"(through the rank's MODE 4 kernel {r_one_chain:.1f}); emulation: {R} unlinked domains {r_emu_free:.1f}, "
      f"{R} linked slabs {r_chain:.1f} = {r_chain / r_emu_free:.3f} of the unlinked run, "
      f"{r_chain / r_one:.3f} of one domain (zchunk {info['zchunk']})")
