"""One-GPU emulation of the multi-GPU schedule with chained exchange periods
(yb_peer_run, k_tb2 MODE 4): a grid split into R z-slabs (R "ranks") that run
in ONE persistent launch — every sweep's boundary items wait in-kernel for the
neighbour slab, store their boundary planes into its ghost planes and signal —
against the same grid as one domain (multi-sweep launches, MODE 2).

Each measurement runs in its own process (warm-up + best of 3), the variants
alternate over REPS rounds, and the SM clock is sampled during each: sustained
load on this GPU drifts the clock down, so back-to-back measurements in one
process are biased towards the first.

usage: python tools/chain_emu.py CONFIG R [STEPS] [REPS]   (CONFIG c2 | c4 | c5; R = 2..8)
  c4: strong scaling — the 1024^2 x 512 grid in R slabs (each rank 512/R planes)
  c2 / c5: weak scaling — R slabs of the config's own depth each (c2: 256^3 per rank)
variants: one = one domain, MODE 2; one4 = one domain through the rank's MODE 4 kernel
(yb_peer_run on an unlinked handle); free = R unlinked domains of one slab's size in one
emulation launch; chain = the R linked slabs in one emulation launch."""
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CFG = {"c2": (256, 256, 256, 1, -1, None), "c4": (1024, 1024, 512, 4, -1, None),
       "c5": (1024, 1024, 256, 5, 5, 6)}


def child(cfg, R, steps, variant):
    import paper_1301_4539_b200 as Y
    from paper_1301_4539_b200.slabs import partition
    nx, ny, nzr, es, ss, fs = CFG[cfg]
    nzg = nzr if cfg == "c4" else nzr * R

    def make(nz, **kw):
        s = Y.Simulation(nx, ny, nz, variant=Y.VARIANT_TB2, **kw)
        s.generate_medium(es, ss)
        s.fill(fs if fs is not None else 3)
        return s
    if variant in ("one", "one4"):
        sims = [make(nzg)]
    elif variant == "free":
        sims = [make(nzg // R) for _ in range(R)]
    else:
        sims = [make(n, z_offset=z0, nz_global=nzg) for z0, n in partition(nzg, R)]
        for lo, hi in zip(sims[:-1], sims[1:]):
            lo.peer_link(1, hi)
            hi.peer_link(0, lo)
        for s in sims:
            s.peer_push(False)
    fn = (lambda k: sims[0].run(k, sync=False)) if variant == "one" else (lambda k: Y.peer_run(sims, k))
    cells = nx * ny * sum(s.nz for s in sims)
    fn(4)
    for s in sims:
        s.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits",
                            "-lms", "50"], stdout=subprocess.PIPE, text=True)
    best = 1e30
    for _ in range(3):
        t0 = time.perf_counter()
        fn(steps)
        for s in sims:
            s.synchronize()
        best = min(best, time.perf_counter() - t0)
    smi.terminate()
    mhz = [float(x) for x in smi.stdout.read().split() if x.replace(".", "").isdigit()]
    print(f"{cells * steps / best / 1e9:.2f} {statistics.median(mhz) if mhz else 0:.0f}")


if __name__ == "__main__":
    if sys.argv[1] == "child":
        child(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
        sys.exit(0)
    cfg, R = sys.argv[1], int(sys.argv[2])
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    res = {v: [] for v in ("one", "one4", "free", "chain")}
    for rep in range(reps):
        order = list(res) if rep % 2 == 0 else list(res)[::-1]
        for v in order:
            r = subprocess.run([sys.executable, __file__, "child", cfg, str(R), str(steps), v],
                               capture_output=True, text=True)
            val, mhz = (float(x) for x in r.stdout.split()) if r.returncode == 0 else (float("nan"), 0.0)
            res[v].append((val, mhz))
    best = {v: max(x[0] for x in xs) for v, xs in res.items()}
    print(f"{cfg} R={R} {steps} steps, Gcell/s best of {reps} processes [sm MHz]: " +
          ", ".join(f"{v} {best[v]:.1f} {[int(m) for _, m in xs]}" for v, xs in res.items()) +
          f" | chain/free {best['chain'] / best['free']:.3f}, chain/one {best['chain'] / best['one']:.3f}, "
          f"one4/one {best['one4'] / best['one']:.3f}")
