"""Caller-memory transfers (yb_xfer.cu): pageable host buffers go through the
pinned staging pipeline (multi-threaded host copies overlapped with the
DMAs), pinned ones straight to cudaMemcpyAsync. Both must move the same
bits: round trips through upload / download and the per-cell coefficient
upload, at sizes that are not multiples of the 32 MiB staging chunk, from
pageable numpy memory and from pinned torch memory."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def seeded(yb, nx, ny, nz, seed):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(yb.comp_extents(nx, ny, nz, c)[::-1]).astype(np.float32) for c in range(6)]


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


# 37 MB+ per component (more than one staging chunk, ragged tail), and one just above the 1 MiB threshold
@pytest.mark.parametrize("dims", [(301, 177, 181), (97, 61, 45)])
def test_pageable_round_trip(yb, dims):
    nx, ny, nz = dims
    f = seeded(yb, nx, ny, nz, 7)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        s.upload(f)
        got = s.download()  # fresh (pageable) numpy arrays
    for c in range(6):
        assert np.array_equal(bits(got[c]), bits(f[c])), c


def test_pageable_equals_pinned(yb):
    torch = pytest.importorskip("torch")
    nx, ny, nz = 257, 131, 150
    f = seeded(yb, nx, ny, nz, 8)
    pinned = [torch.from_numpy(a).pin_memory().numpy() for a in f]
    outs = {}
    for name, src in (("pageable", f), ("pinned", pinned)):
        with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
            s.generate_medium(3, 3)
            s.upload(src)
            s.run(4)
            dst = ([torch.empty(a.shape, dtype=torch.float32).pin_memory().numpy() for a in f]
                   if name == "pinned" else None)
            outs[name] = s.download(out=dst)
    for c in range(6):
        assert np.array_equal(bits(outs["pageable"][c]), bits(outs["pinned"][c])), c


def test_pageable_cell_coeffs(yb):
    """A per-cell Cb array uploaded from pageable memory equals the one the
    device generates from the same seed (yb_set_cell_coeffs vs yb_generate_medium)."""
    nx, ny, nz = 200, 180, 170  # 24 MB of coefficients
    cb = yb.host_medium(nx, ny, nz, 4, -1)[1]
    f = seeded(yb, nx, ny, nz, 9)
    res = []
    for mode in ("host", "device"):
        with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
            if mode == "host":
                s.set_cell_coeffs(yb.CB, np.ascontiguousarray(cb))
            else:
                s.generate_medium(4, -1)
            s.upload(f)
            s.run(6)
            res.append(s.digest())
    assert res[0] == res[1]
