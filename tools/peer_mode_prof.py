"""One two-step launch of a middle z-slab in peer-store mode (yb_peer_step,
MODE 3) and one plain single-sweep launch (MODE 0) of an identical unlinked
slab — for an ncu comparison of the two kernel modes (run under ncu -k
regex:k_tb2). All on one stream; every in-kernel wait is already satisfied."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4539_b200 as Y  # noqa: E402

n = 256
st = torch.cuda.Stream()
sims = []
for i in range(3):
    s = Y.Simulation(n, n, n, variant=Y.VARIANT_TB2, z_offset=i * n, nz_global=3 * n)
    s.generate_medium(1, -1)
    s.set_stream(st.cuda_stream)
    sims.append(s)
for lo, hi in zip(sims[:-1], sims[1:]):
    lo.peer_link(1, hi)
    hi.peer_link(0, lo)
for s in sims:
    s.peer_push(False)
for _ in range(int(os.environ.get("PERIODS", "2"))):
    for s in sims:
        s.peer_step(2)
plain = Y.Simulation(n, n, n, variant=Y.VARIANT_TB2, z_offset=n, nz_global=3 * n)
plain.generate_medium(1, -1)
plain.set_stream(st.cuda_stream)
plain.run(2)
plain.synchronize()
for s in sims:
    s.synchronize()
print("ok")
