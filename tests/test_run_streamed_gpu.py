"""Streamed upload + run + readback (yb_run_streamed): run_simulation's host
flow (runner.hpp:349-362) in one call. The per-cell coefficient arrays and the
initial fields go up tile row by tile row while the first sweeps of the one
multi-sweep launch already follow them (mirrored y-skewed order, per-row words
written by the copy stream), and the last sweeps stream out as in
yb_run_to_host. The result must be bit-identical to set_cell_coeffs + upload +
run + download and to the C oracle, whatever the grid shape (ragged tiles, rows
not a multiple of 8), which arrays are given (uniform ones included: they are
stored as given), with or without initial fields / sources, on repeated calls
on one handle, and from pageable buffers or ineligible step counts (the
phase-by-phase path)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def force_streamed_upload(monkeypatch):
    # rows under 4 KB (nx < 1024) upload as whole arrays by default (faster copies); the cut-down
    # grids here force the tile-row upload so that path is what is tested
    monkeypatch.setenv("YB_UP_STREAM", "1")


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def pin(a):
    torch = pytest.importorskip("torch")
    t = torch.empty(a.shape, dtype=torch.float32).pin_memory()
    t.numpy()[...] = a
    return t.numpy()


def pinned_out(yb, nx, ny, nz):
    torch = pytest.importorskip("torch")
    return [torch.empty(yb.comp_extents(nx, ny, nz, c)[::-1], dtype=torch.float32).pin_memory().numpy()
            for c in range(6)]


def inputs(yb, nx, ny, nz, medium, fseed):
    """Host arrays of the pinned inputs: {which: cells}, six fields or None."""
    cells = {}
    if medium:
        eps, sig, want = medium
        med = yb.host_medium_slab(nx, ny, nz, 0, nz, eps, sig, [np.empty((nz, ny, nx), np.float32) for _ in range(4)])
        cells = {q: med[q] for q in want}
    fields = None
    if fseed is not None:
        fields = [np.empty(yb.comp_extents(nx, ny, nz, c)[::-1], np.float32) for c in range(6)]
        yb.host_fields_slab(nx, ny, nz, 0, nz, fseed, out=fields)
    return cells, fields


def add_source(yb, s, nx, ny, nz):
    from oracle import pyoracle as O
    s.add_source(yb.EZ, nx // 2, ny // 2, nz // 2, O.gauss_table(400))


def reference_run(yb, nx, ny, nz, steps, cells, fields, src):
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        if cells:
            s.set_cell_coeffs_many(cells)
        if fields is not None:
            s.upload(fields)
        if src:
            add_source(yb, s, nx, ny, nz)
        s.run(steps)
        return s.download()


CASES = [
    # nx, ny, nz, steps, medium (eps seed, sigma seed, arrays given), fields seed, source
    (130, 37, 41, 12, (2, 2, (0, 1, 2, 3)), 3, True),    # ragged x tile, ny not a multiple of 8, all four arrays
    (256, 64, 40, 16, (1, -1, (1,)), None, True),        # config-2/4 flow: Cb only, zero start
    (300, 90, 64, 8, (3, 3, (0, 1, 2, 3)), 6, False),    # the shortest streamed run (4 sweeps)
    (200, 120, 33, 40, (4, -1, (0, 1, 2, 3)), 7, True),  # uniform Ca / Da / Db given as full arrays
    (128, 256, 24, 100, None, 5, False),                 # fields only, 50 sweeps, both skews 16 deep
    (140, 100, 30, 14, (5, 5, (0, 1, 2, 3)), 8, True),   # an odd number of sweeps (the final state in the other buffer)
    (96, 64, 20, 22, None, 9, True),                     # odd, fields only
]


@pytest.mark.parametrize("case", CASES)
def test_run_streamed_equals_phases(yb, case):
    nx, ny, nz, steps, medium, fseed, src = case
    cells, fields = inputs(yb, nx, ny, nz, medium, fseed)
    want = reference_run(yb, nx, ny, nz, steps, cells, fields, src)
    pc = {q: pin(a) for q, a in cells.items()}
    pf = [pin(a) for a in fields] if fields is not None else None
    out = pinned_out(yb, nx, ny, nz)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        if src:
            add_source(yb, s, nx, ny, nz)
        got = s.run_streamed(steps, pc, pf, out=out)
        info = s.info()
        assert s.step_index == steps
        assert info["streamed_uploads"] == 1 and info["streamed_readbacks"] == 1, info
        assert info["n_cell_arrays"] == len(cells)
        for c in range(6):
            assert np.array_equal(bits(got[c]), bits(want[c])), (case, c)
        # the device state (fields and coefficient arrays, clamped duplicates included) is the
        # phase-by-phase one: continuing with the one-step kernels' sibling launch matches
        s.run(3)
        cont = s.download()
    want2 = reference_run(yb, nx, ny, nz, steps + 3, cells, fields, src)
    for c in range(6):
        assert np.array_equal(bits(cont[c]), bits(want2[c])), (case, c)


def test_run_streamed_vs_oracle(yb):
    from oracle import pyoracle as O
    nx, ny, nz, steps = 70, 36, 30, 14
    tab = O.gauss_table(steps)
    ca, cb, da, db = O.cell_coeffs(nx, ny, nz, 2, 2)
    want = O.fill_fields(nx, ny, nz, 3)
    start = [a.copy() for a in want]
    O.run(nx, ny, nz, want, O.Coeffs(nx, ny, nz, ca=ca, cb=cb, da=da, db=db), steps,
          sources=[O.Source(2, nx // 2, ny // 2, nz // 2, tab)])
    cells = {0: pin(ca.reshape(nz, ny, nx)), 1: pin(cb.reshape(nz, ny, nx)), 2: pin(da.reshape(nz, ny, nx)),
             3: pin(db.reshape(nz, ny, nx))}
    out = pinned_out(yb, nx, ny, nz)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        s.add_source(yb.EZ, nx // 2, ny // 2, nz // 2, tab)
        got = s.run_streamed(steps, cells, [pin(a) for a in start], out=out)
        assert s.info()["streamed_uploads"] == 1
    for c in range(6):
        assert np.array_equal(bits(got[c]), bits(want[c])), c


def test_run_streamed_repeated_and_fallbacks(yb, monkeypatch):
    nx, ny, nz = 160, 72, 28
    cells, fields = inputs(yb, nx, ny, nz, (2, 2, (0, 1, 2, 3)), 3)
    pc = {q: pin(a) for q, a in cells.items()}
    pf = [pin(a) for a in fields]
    out = pinned_out(yb, nx, ny, nz)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        for rep, steps in enumerate((10, 24, 10)):  # monotonic row words / counters across calls
            s.step_index = 0
            got = s.run_streamed(steps, pc, pf, out=out)
            assert s.info()["streamed_uploads"] == rep + 1
            want = reference_run(yb, nx, ny, nz, steps, cells, fields, False)
            for c in range(6):
                assert np.array_equal(bits(got[c]), bits(want[c])), (steps, c)
        # an odd step count and pageable buffers take the phase-by-phase path: same result
        n_up = s.info()["streamed_uploads"]
        s.step_index = 0
        got = s.run_streamed(11, pc, pf, out=out)
        want = reference_run(yb, nx, ny, nz, 11, cells, fields, False)
        for c in range(6):
            assert np.array_equal(bits(got[c]), bits(want[c])), c
        s.step_index = 0
        got = s.run_streamed(10, cells, fields)
        want = reference_run(yb, nx, ny, nz, 10, cells, fields, False)
        for c in range(6):
            assert np.array_equal(bits(got[c]), bits(want[c])), c
        assert s.info()["streamed_uploads"] == n_up
        # a narrow grid without the override: whole-array uploads, then the streamed readback
        monkeypatch.delenv("YB_UP_STREAM")
        s.step_index = 0
        n_rd = s.info()["streamed_readbacks"]
        got = s.run_streamed(10, pc, pf, out=out)
        for c in range(6):
            assert np.array_equal(bits(got[c]), bits(want[c])), c
        assert s.info()["streamed_uploads"] == n_up and s.info()["streamed_readbacks"] == n_rd + 1


def test_run_streamed_argument_errors(yb):
    with yb.Simulation(64, 32, 16) as s:
        out = [np.empty(yb.comp_extents(64, 32, 16, c)[::-1], np.float32) for c in range(6)]
        bad = {7: np.ones((16, 32, 64), np.float32)}
        with pytest.raises(yb.YeeError):
            s.run_streamed(8, bad, None, out=out)
        with pytest.raises(yb.YeeError):
            s.run_streamed(-2, None, None, out=out)
