"""Streamed readback (yb_run_to_host): `run(n)` + the FieldSet readout in one
call, the device->host copies of each tile row overlapping the sweeps still
running (skewed item order of the last multi-sweep launch, per-row counters
polled by the copy stream). The result must be bit-identical to run +
download — and to the C oracle — whatever the grid shape (ragged tiles,
rows not a multiple of 8, one tile row), step count (odd, short, long),
medium, sources and initial state, also on repeated calls on one handle
(monotonic counters) and from pageable buffers (streamed through the pinned
staging ring; YB_NO_PAGEABLE_DRAIN=1 takes the phase-by-phase path)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def pinned_like(yb, nx, ny, nz):
    torch = pytest.importorskip("torch")
    return [torch.empty(yb.comp_extents(nx, ny, nz, c)[::-1], dtype=torch.float32).pin_memory().numpy()
            for c in range(6)]


def setup(yb, s, nx, ny, nz, medium, fields_seed, source):
    if medium:
        s.generate_medium(*medium)
    if fields_seed is not None:
        s.fill(fields_seed)
    if source:
        from oracle import pyoracle as O
        s.add_source(yb.EZ, nx // 2, ny // 2, nz // 2, O.gauss_table(400))


CASES = [
    # nx, ny, nz, steps, medium (eps, sigma seeds), fields seed, source
    (130, 37, 41, 12, (2, 2), 3, True),     # ragged x tile, ny not a multiple of 8
    (256, 64, 40, 7, (1, -1), None, True),  # odd step count: one leading one-step launch
    (128, 8, 24, 30, None, 5, False),       # one tile row
    (300, 90, 64, 4, (3, 3), 6, True),      # the shortest streamed run
    (200, 120, 33, 41, (4, -1), 7, True),   # 20 sweeps, odd
]


@pytest.mark.parametrize("case", CASES)
def test_run_to_host_equals_run_download(yb, case):
    nx, ny, nz, steps, medium, fseed, src = case
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        setup(yb, s, nx, ny, nz, medium, fseed, src)
        s.run(steps)
        want = s.download()
    out = pinned_like(yb, nx, ny, nz)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        setup(yb, s, nx, ny, nz, medium, fseed, src)
        got = s.run_to_host(steps, out=out)
        assert s.step_index == steps
        assert s.info()["streamed_readbacks"] == 1
        # the device state is the final one too: continuing matches
        s.run(2)
        cont = s.download()
    for c in range(6):
        assert np.array_equal(bits(got[c]), bits(want[c])), (case, c)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        setup(yb, s, nx, ny, nz, medium, fseed, src)
        s.run(steps + 2)
        want2 = s.download()
    for c in range(6):
        assert np.array_equal(bits(cont[c]), bits(want2[c])), (case, c)


def test_run_to_host_vs_oracle(yb):
    from oracle import pyoracle as O
    nx, ny, nz, steps = 70, 36, 30, 14
    tab = O.gauss_table(steps)
    ca, cb, da, db = O.cell_coeffs(nx, ny, nz, 2, 2)
    want = O.fill_fields(nx, ny, nz, 3)
    O.run(nx, ny, nz, want, O.Coeffs(nx, ny, nz, ca=ca, cb=cb, da=da, db=db), steps,
          sources=[O.Source(2, nx // 2, ny // 2, nz // 2, tab)])
    out = pinned_like(yb, nx, ny, nz)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        s.generate_medium(2, 2)
        s.fill(3)
        s.add_source(yb.EZ, nx // 2, ny // 2, nz // 2, tab)
        got = s.run_to_host(steps, out=out)
        assert s.info()["streamed_readbacks"] == 1
    for c in range(6):
        assert np.array_equal(bits(got[c]), bits(want[c])), c


def test_run_to_host_repeated_calls(yb):
    """Counters are monotonic across calls; the same buffers reused."""
    nx, ny, nz = 160, 48, 36
    out = pinned_like(yb, nx, ny, nz)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as ref:
        setup(yb, ref, nx, ny, nz, (5, 5), 8, True)
        with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
            setup(yb, s, nx, ny, nz, (5, 5), 8, True)
            for n in (10, 6, 9, 4, 16):
                got = s.run_to_host(n, out=out)
                ref.run(n)
                want = ref.download()
                for c in range(6):
                    assert np.array_equal(bits(got[c]), bits(want[c])), (n, c)
            assert s.info()["streamed_readbacks"] == 5


def test_run_to_host_fallbacks(yb):
    """Pageable buffers, the one-step kernel, probes or fewer than 4 steps
    take run + download: same bits, nothing streamed."""
    nx, ny, nz, steps = 96, 40, 20, 9
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        setup(yb, s, nx, ny, nz, (2, -1), 4, True)
        s.run(steps)
        want = s.download()
    for kind in ("fused", "short"):
        variant = yb.VARIANT_FUSED if kind == "fused" else yb.VARIANT_TB2
        with yb.Simulation(nx, ny, nz, variant=variant) as s:
            setup(yb, s, nx, ny, nz, (2, -1), 4, True)
            if kind == "short":
                s.run(steps - 3)
                got = s.run_to_host(3, out=pinned_like(yb, nx, ny, nz))
            else:
                got = s.run_to_host(steps, out=pinned_like(yb, nx, ny, nz))
            assert s.info()["streamed_readbacks"] == 0, kind
        for c in range(6):
            assert np.array_equal(bits(got[c]), bits(want[c])), (kind, c)


@pytest.mark.parametrize("case", CASES)
def test_run_to_host_pageable_streams_through_staging(yb, case, monkeypatch):
    """Pageable destination buffers (std::vector storage of a drop-in caller): the tile rows go
    through the pinned staging ring while the rows above still sweep; same bits as run + download,
    also with the staged path switched off."""
    nx, ny, nz, steps, medium, fseed, src = case
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        setup(yb, s, nx, ny, nz, medium, fseed, src)
        s.run(steps)
        want = s.download()
    for off in (False, True):
        if off:
            monkeypatch.setenv("YB_NO_PAGEABLE_DRAIN", "1")
        with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
            setup(yb, s, nx, ny, nz, medium, fseed, src)
            got = s.run_to_host(steps)  # fresh numpy arrays: pageable
            assert s.info()["streamed_readbacks"] == (0 if off else 1)
            got2 = s.run_to_host(4) if not off else None  # the ring and the counters are reusable
        for c in range(6):
            assert np.array_equal(bits(got[c]), bits(want[c])), (case, off, c)
        if got2 is not None:
            with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
                setup(yb, s, nx, ny, nz, medium, fseed, src)
                s.run(steps + 4)
                want2 = s.download()
            for c in range(6):
                assert np.array_equal(bits(got2[c]), bits(want2[c])), (case, c)
