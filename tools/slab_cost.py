"""Single-GPU cost of the slab schedule (no transport): a middle slab of a
3-slab grid advanced with plain sweeps vs split sweeps (boundary + interior
launches), against the single-domain multi-sweep run of the same size."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1301_4539_b200 as Y  # noqa: E402

n, steps = 256, 40


def timed(sim, fn):
    fn(4)
    sim.synchronize()
    t0 = time.perf_counter()
    fn(steps)
    sim.synchronize()
    return n ** 3 * steps / (time.perf_counter() - t0) / 1e9


one = Y.Simulation(n, n, n, variant=Y.VARIANT_TB2)
one.generate_medium(1, -1)
print("single domain (multi-sweep)", round(timed(one, lambda k: one.run(k, sync=False)), 1))
one.close()
sl = Y.Simulation(n, n, n, variant=Y.VARIANT_TB2, z_offset=n, nz_global=3 * n)
sl.generate_medium(1, -1)
print("middle slab, plain sweeps", round(timed(sl, lambda k: sl.run(k, sync=False)), 1))


def split(k):
    for _ in range(k // 2):
        sl.advance_begin(2)
        sl.advance_end()


print("middle slab, split sweeps", round(timed(sl, split), 1))
sl.close()

# serial schedule with a self-exchange (pack, then unpack the same planes)
import torch  # noqa: E402

sl = Y.Simulation(n, n, n, variant=Y.VARIANT_TB2, z_offset=n, nz_global=3 * n)
sl.generate_medium(1, -1)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
sl.set_stream(st.cuda_stream)  # stream-ordered pack / unpack, as bench.py runs them
bufs = [torch.empty(sl.halo_bytes(side, False), dtype=torch.uint8, device="cuda") for side in (0, 1)]
rbufs = [torch.empty(sl.halo_bytes(side, True), dtype=torch.uint8, device="cuda") for side in (0, 1)]


def serial(k):
    for _ in range(k // 2):
        for side in (0, 1):
            sl.halo_pack(side, bufs[side].data_ptr())
        for side in (0, 1):
            sl.halo_unpack(side, rbufs[side].data_ptr())
        sl.run(2, sync=False)


print("middle slab, pack + unpack + sweep", round(timed(sl, serial), 1))


def split_x(k):
    for _ in range(k // 2):
        sl.advance_begin(2)
        for side in (0, 1):
            sl.halo_pack(side, bufs[side].data_ptr())
        sl.advance_end()
        for side in (0, 1):
            sl.halo_unpack(side, rbufs[side].data_ptr())


print("middle slab, split + pack + unpack", round(timed(sl, split_x), 1))
sl.close()

# three linked slabs in one process: plain sweeps (no exchange) vs yb_peer_step
# (boundary planes stored straight into the neighbours' ghost planes)
sims = []
for i in range(3):
    s = Y.Simulation(n, n, n, variant=Y.VARIANT_TB2, z_offset=i * n, nz_global=3 * n)
    s.generate_medium(1, -1)
    sims.append(s)


def plain3(k):
    for s in sims:
        s.run(k, sync=False)


def peer3(k):
    for _ in range(k // 2):
        for s in sims:
            s.peer_step(2)


def timed3(fn):
    fn(4)
    for s in sims:
        s.synchronize()
    t0 = time.perf_counter()
    fn(steps)
    for s in sims:
        s.synchronize()
    return 3 * n ** 3 * steps / (time.perf_counter() - t0) / 1e9


print("3 slabs, plain sweeps", round(timed3(plain3), 1))
shared = torch.cuda.Stream()  # one stream: every device-side wait is already satisfied when it runs
for s in sims:
    s.set_stream(shared.cuda_stream)
for lo, hi in zip(sims[:-1], sims[1:]):
    lo.peer_link(1, hi)
    hi.peer_link(0, lo)
for s in sims:
    s.peer_push(False)
print("3 slabs, peer_step (fused peer stores)", round(timed3(peer3), 1))
for s in sims:
    s.close()
