import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1301_4539_b200 as yb
from paper_1301_4539_b200.slabs import partition
nx, ny, nzg, steps, R = 136, 40, 29, int(sys.argv[1]), 3
src_tab = np.exp(-((np.arange(steps + 4) - 40.0) / 12.0) ** 2).astype(np.float32) if len(sys.argv) > 2 else None
for fold in ("1", "0"):
    if fold == "0":
        os.environ["YB_PEER_NOFOLD"] = "1"
    sims = []
    for z0, n in partition(nzg, R):
        s = yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, variant=0)
        s.generate_medium(7, 7); s.fill(8); sims.append(s)
        if src_tab is not None: s.add_source(2, nx // 2, ny // 2, nzg // 2, src_tab)
    for lo, hi in zip(sims[:-1], sims[1:]):
        lo.peer_link(1, hi); hi.peer_link(0, lo)
    for s in sims: s.peer_push(False)
    done = 0
    while done < steps:
        n = min(2, steps - done)
        for s in sims: s.peer_step(n)
        done += n
    outs = [s.download() for s in sims]
    with yb.Simulation(nx, ny, nzg) as one:
        one.generate_medium(7, 7); one.fill(8)
        if src_tab is not None: one.add_source(2, nx // 2, ny // 2, nzg // 2, src_tab)
        one.run(steps); want = one.download()
    for r, s in enumerate(sims):
        for c in range(6):
            k = s.nz
            a = outs[r][c][:k]; b = want[c][s.z_offset:s.z_offset + k]
            bad = np.argwhere(a.view(np.uint32) != b.view(np.uint32))
            if len(bad):
                print("fold", fold, "rank", r, "comp", c, "nbad", len(bad), "planes", sorted(set(bad[:, 0].tolist()))[:10], "rows", sorted(set(bad[:, 1].tolist()))[:10], "cols", sorted(set(bad[:, 2].tolist()))[:6], s.info()["zchunk"])
    print("fold", fold, "done")
    for s in sims: s.close()
