"""One domain, same work: multi-sweep launches (MODE 2, yb_advance) vs the rank's
chained-period kernel (MODE 4 direct, yb_peer_run on an unlinked handle).
usage: python tools/mode4_ab.py CONFIG   (c2 | c4)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4539_b200 as Y  # noqa: E402

nx, ny, nz, es = {"c2": (256, 256, 256, 1), "c4": (1024, 1024, 512, 4)}[sys.argv[1]]
steps = 20
with Y.Simulation(nx, ny, nz, variant=Y.VARIANT_TB2) as s:
    s.generate_medium(es, -1)
    s.fill(3)

    def rate(fn):
        fn(4)
        s.synchronize()
        best = 1e30
        for _ in range(3):
            t0 = time.perf_counter()
            fn(steps)
            s.synchronize()
            best = min(best, time.perf_counter() - t0)
        return nx * ny * nz * steps / best / 1e9
    b0 = rate(lambda k: Y.peer_run([s], k))
    a = rate(lambda k: s.run(k, sync=False))
    b = rate(lambda k: Y.peer_run([s], k))
    a2 = rate(lambda k: s.run(k, sync=False))
    print(f"{sys.argv[1]} MODE4-direct {b0:.1f} MODE2 {a:.1f} MODE4-direct {b:.1f} MODE2 {a2:.1f} ratio {b / a:.3f}")
