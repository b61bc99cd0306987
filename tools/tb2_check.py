"""Quick TB2 parity probe: compare variant 2 with the oracle on a few cases."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1301_4539_b200 as Y
from oracle import pyoracle as O

def run(nx, ny, nz, steps, es, ss, fs, src, zchunk=0):
    tab = O.gauss_table(steps + 2)
    f = O.fill_fields(nx, ny, nz, fs) if fs is not None else O.zeros_state(nx, ny, nz)
    with Y.Simulation(nx, ny, nz, variant=2, zchunk=zchunk) as sim:
        sim.generate_medium(es, ss)
        if src: sim.add_source(2, nx // 2, ny // 2, nz // 2, tab)
        if fs is not None: sim.fill(fs)
        sim.run(steps)
        got = sim.download()
        info = sim.info()
    co = O.Coeffs(nx, ny, nz)
    if es >= 0 or ss >= 0:
        ca, cb, da, db = O.cell_coeffs(nx, ny, nz, es, ss)
        co = O.Coeffs(nx, ny, nz, ca=ca, cb=cb, da=da, db=db)
    O.run(nx, ny, nz, f, co, steps, sources=[O.Source(2, nx // 2, ny // 2, nz // 2, tab)] if src else None)
    bad = []
    for c in range(6):
        d = np.nonzero(got[c].view(np.uint32) != f[c].view(np.uint32))
        if d[0].size:
            k, j, i = (int(v[0]) for v in d)
            bad.append((O.COMP_NAMES[c], d[0].size, (i, j, k), float(got[c][k, j, i]), float(f[c][k, j, i])))
    print((nx, ny, nz, steps, es, ss, fs, src, zchunk), "OK" if not bad else bad, info["zchunk"], info["stages"], flush=True)
    return not bad

ok = True
for case in [(40, 24, 20, 2, -1, -1, 3, False), (40, 24, 20, 4, -1, -1, 3, False), (40, 24, 20, 2, 2, 2, 3, False),
             (64, 48, 40, 6, 2, 2, 3, False), (48, 40, 36, 10, 1, -1, None, True), (37, 29, 23, 7, 7, 7, 8, True),
             (136, 72, 40, 8, 4, -1, None, True), (200, 64, 40, 6, 3, 3, 4, False)]:
    ok &= run(*case)
for z in (1, 2, 3, 7):
    ok &= run(64, 40, 30, 6, 5, 5, 6, False, zchunk=z)
print("ALL OK" if ok else "FAILURES")
