"""How far apart in time do concurrently processed y-neighbouring work items of the multi-sweep
two-step launch run? Reads the timestamp file a -DYB_TB2_STAMP build writes (tools/stamp_build.sh;
YB_TB2_STAMP_FILE), prints the distribution of |start(ty) - start(ty+1)| for items of the same sweep,
z-chunk and tile column, in planes (an item's duration / its planes), and the same for x neighbours.
usage: python tools/stamp_drift.py file"""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
nitems, nsw, ntx, nty, zchunk, nz = np.frombuffer(raw[:24], np.int32)
t = np.frombuffer(raw[24:], np.uint64).reshape(nsw, nitems, 2).astype(np.float64)
T = ntx * nty
nch = nitems // T
start = t[:, :, 0].reshape(nsw, nch, nty, ntx)
end = t[:, :, 1].reshape(nsw, nch, nty, ntx)
dur = end - start
planes = min(zchunk, nz)
per_plane = np.median(dur) / planes
print(f"items {nitems} ({nch} chunks x {nty} x {ntx}), sweeps {nsw}; median item {np.median(dur)/1e3:.1f} us "
      f"({per_plane:.0f} ns per plane); launch {(end.max()-start.min())/1e6:.2f} ms")
for name, d in (("y neighbours", np.abs(start[:, :, 1:, :] - start[:, :, :-1, :])),
                ("x neighbours", np.abs(start[:, :, :, 1:] - start[:, :, :, :-1]))):
    d = d[1:].ravel() / per_plane  # skip the first sweep (all CTAs start together)
    q = np.percentile(d, [10, 25, 50, 75, 90])
    print(f"{name}: |start difference| in planes: p10 {q[0]:.1f} p25 {q[1]:.1f} median {q[2]:.1f} p75 {q[3]:.1f} "
          f"p90 {q[4]:.1f}; within 4 / 8 / 16 / 32 planes: "
          + " / ".join(f"{100*np.mean(d <= w):.0f}%" for w in (4, 8, 16, 32)))
