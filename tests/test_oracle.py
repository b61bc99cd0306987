"""CPU tests: pin the C oracle against the reference (golden fixtures generated
from the compiled reference, the reference's own known-answer tests restated,
and — when oracle/_ref is built — the live reference)."""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def fields(d, prefix):
    return [np.ascontiguousarray(d[f"{prefix}_{c}"]) for c in ("ex", "ey", "ez", "hx", "hy", "hz")]


def bits_equal(a, b):
    return all(np.array_equal(x.view(np.uint32), y.view(np.uint32)) for x, y in zip(a, b))


def test_courant_constant(oracle):
    S = oracle.courant()
    assert S == np.float32(0.99 / math.sqrt(3.0))
    assert np.float32(S).view(np.uint32) == 0x3F1252DB


def test_extents_table(oracle):
    # kernel_test.cpp:43-63 on a 3x4x5 grid
    ext = [oracle.comp_extents(3, 4, 5, c) for c in range(6)]
    assert ext == [(3, 5, 6), (4, 4, 6), (4, 5, 5), (4, 4, 5), (3, 5, 5), (3, 4, 6)]


def test_golden_axis_src(oracle):
    d = load("axis_src")
    nx, ny, nz = (int(v) for v in d["dims"])
    f = fields(d, "in")
    assert bits_equal(f, oracle.fill_fields(nx, ny, nz, int(d["seed"])))  # seeded inputs pinned
    c, i, j, k = (int(v) for v in d["src"])
    src = oracle.Source(c, i, j, k, d["table"])
    assert np.array_equal(d["table"], oracle.gauss_table(len(d["table"])))
    oracle.run(nx, ny, nz, f, oracle.Coeffs(nx, ny, nz), int(d["steps"]), sources=[src])
    assert bits_equal(f, fields(d, "out"))
    assert oracle.digest(nx, ny, nz, f) == int(d["digest"])


def test_golden_stretched(oracle):
    d = load("stretched")
    nx, ny, nz = (int(v) for v in d["dims"])
    f = fields(d, "in")
    co = oracle.Coeffs(nx, ny, nz, cdx=d["cdx"], cdy=d["cdy"], cdz=d["cdz"])
    oracle.run(nx, ny, nz, f, co, int(d["steps"]))
    assert bits_equal(f, fields(d, "out"))
    assert oracle.digest(nx, ny, nz, f) == int(d["digest"])


def test_golden_reference_simulation_source(oracle):
    # yeeblock::Simulation<float> with its own SourceSpec == oracle driven by the
    # per-step increments inject_current adds.
    d = load("sim_refsrc")
    nx, ny, nz = (int(v) for v in d["dims"])
    f = oracle.zeros_state(nx, ny, nz)
    c, i, j, k = (int(v) for v in d["src"])
    oracle.run(nx, ny, nz, f, oracle.Coeffs(nx, ny, nz), int(d["steps"]),
               sources=[oracle.Source(c, i, j, k, d["table"])])
    assert bits_equal(f, fields(d, "out"))
    assert oracle.digest(nx, ny, nz, f) == int(d["digest"])


def test_kat_ampere_hz_face(oracle):
    # kernel_test.cpp:84-106: hz(2,2,2)=1, c*dt/h=0.5 -> four edges +-0.5
    n = 4
    f = oracle.zeros_state(n, n, n)
    f[5][2, 2, 2] = 1.0
    h = np.full(n, 0.5, np.float32)
    oracle.ampere(n, n, n, f, oracle.Coeffs(n, n, n, cdx=h, cdy=h, cdz=h))
    assert f[0][2, 2, 2] == 0.5 and f[0][2, 3, 2] == -0.5
    assert f[1][2, 2, 2] == -0.5 and f[1][2, 2, 3] == 0.5
    assert sum(int((a != 0).sum()) for a in f[:3]) == 4
    assert bits_equal(f, fields(load("kat_hz"), "out"))


def test_kat_faraday_edges(oracle):
    # kernel_test.cpp:108-130
    n = 4
    h = np.full(n, 0.5, np.float32)
    co = oracle.Coeffs(n, n, n, cdx=h, cdy=h, cdz=h)
    f = oracle.zeros_state(n, n, n)
    f[1][2, 1, 1] = 1.0  # ey(1,1,2)
    oracle.faraday(n, n, n, f, co)
    assert f[3][1, 1, 1] == 0.5
    assert bits_equal(f, fields(load("kat_faraday"), "ey"))
    g = oracle.zeros_state(n, n, n)
    g[2][1, 2, 1] = 1.0  # ez(1,2,1)
    oracle.faraday(n, n, n, g, co)
    assert g[3][1, 1, 1] == -0.5
    assert bits_equal(g, fields(load("kat_faraday"), "ez"))


def test_kat_zero_and_uniform_fixed_points(oracle):
    # kernel_test.cpp:65-82
    n = 4
    h = np.full(n, 0.5, np.float32)
    co = oracle.Coeffs(n, n, n, cdx=h, cdy=h, cdz=h)
    f = oracle.zeros_state(n, n, n)
    oracle.ampere(n, n, n, f, co)
    assert all(not a.any() for a in f)
    for c in (3, 4, 5):
        f[c][...] = 3.25
    before = [a.copy() for a in f]
    oracle.ampere(n, n, n, f, co)
    assert bits_equal(f, before)


def test_kat_pec_shell(oracle):
    # kernel_test.cpp:143-165: all-ones E keeps the interior, zeroes the shell
    n = 4
    f = oracle.zeros_state(n, n, n)
    for c in range(3):
        f[c][...] = 1.0
    oracle.pec(n, n, n, f)
    for c in range(3):
        ext = oracle.comp_extents(n, n, n, c)
        kk, jj, ii = np.meshgrid(*[np.arange(e) for e in ext[::-1]], indexing="ij")
        idx = (ii, jj, kk)
        inner = np.ones(f[c].shape, bool)
        for a in range(3):
            if a != c:
                inner &= (idx[a] >= 1) & (idx[a] <= n - 1)
        assert np.array_equal(f[c], inner.astype(np.float32))


def test_kat_digest_bit_sensitivity(oracle):
    # kernel_test.cpp:289-298 (float version)
    a = oracle.zeros_state(4, 4, 4)
    b = oracle.zeros_state(4, 4, 4)
    assert oracle.digest(4, 4, 4, a) == oracle.digest(4, 4, 4, b)
    b[4][3, 2, 1] = np.float32(1e-38)
    assert oracle.digest(4, 4, 4, a) != oracle.digest(4, 4, 4, b)
    b[4][3, 2, 1] = np.float32(-0.0)
    assert oracle.digest(4, 4, 4, a) != oracle.digest(4, 4, 4, b)


def test_material_extension_reduces_to_reference(oracle):
    # Ca = Da = 1, Cb = Db = S per cell is bit-identical to the axis (reference) form
    nx, ny, nz = 13, 11, 9
    f0 = oracle.fill_fields(nx, ny, nz, 5)
    S = oracle.courant()
    ones = np.ones((nz, ny, nx), np.float32)
    sarr = np.full((nz, ny, nx), S, np.float32)
    tab = oracle.gauss_table(12)
    src = [oracle.Source(2, 6, 5, 4, tab)]
    a = [x.copy() for x in f0]
    b = [x.copy() for x in f0]
    oracle.run(nx, ny, nz, a, oracle.Coeffs(nx, ny, nz, ca=ones, cb=sarr, da=ones, db=sarr), 12,
               sources=src)
    oracle.run(nx, ny, nz, b, oracle.Coeffs(nx, ny, nz), 12, sources=src)
    assert bits_equal(a, b)
    # and the pinned vacuum medium produces exactly those coefficients
    ca, cb, da, db = oracle.cell_coeffs(nx, ny, nz, -1, -1)
    assert (ca == 1).all() and (da == 1).all() and (cb == S).all() and (db == S).all()


def test_medium_generator_ranges(oracle):
    ca, cb, da, db = oracle.cell_coeffs(16, 8, 4, 2, 2)
    S = float(oracle.courant())
    assert (ca <= 1).all() and (ca > 0.95).all()
    assert (cb <= S).all() and (cb >= S / 4.0 / 1.1).all()
    assert (da <= 1).all() and (da > 0.97).all() and (db <= S).all()
    # sigma = 0 -> Ca = Da = 1 exactly, Db = S exactly
    ca, cb, da, db = oracle.cell_coeffs(16, 8, 4, 1, -1)
    assert (ca == 1).all() and (da == 1).all() and (db == np.float32(S)).all()
    assert len(np.unique(cb)) > 400
    f = oracle.fill_fields(9, 7, 5, 3)
    assert all((a >= -1).all() and (a < 1).all() for a in f)


def test_oracle_threads_deterministic(oracle):
    nx, ny, nz = 20, 18, 16
    ca, cb, da, db = oracle.cell_coeffs(nx, ny, nz, 2, 2)
    co = oracle.Coeffs(nx, ny, nz, ca=ca, cb=cb, da=da, db=db)
    a = oracle.fill_fields(nx, ny, nz, 3)
    b = [x.copy() for x in a]
    oracle.run(nx, ny, nz, a, co, 6, threads=1)
    oracle.run(nx, ny, nz, b, co, 6, threads=4)
    assert bits_equal(a, b)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLD), "..", "oracle", "_ref",
                                                    "libyeeref.so")),
                    reason="oracle/_ref not built (reference absent)")
def test_live_reference_matches_oracle(oracle):
    nx, ny, nz = 18, 14, 12
    f0 = oracle.fill_fields(nx, ny, nz, 21)
    tab = oracle.gauss_table(10)
    src = oracle.Source(2, 9, 7, 6, tab)
    a = [x.copy() for x in f0]
    b = [x.copy() for x in f0]
    oracle.run(nx, ny, nz, a, oracle.Coeffs(nx, ny, nz), 10, sources=[src])
    oracle.ref_run_kernels(nx, ny, nz, b, 10, source=src)
    assert bits_equal(a, b)
    # the reference's Interleaved multithreaded variant agrees (quiescent skip off)
    c = [x.copy() for x in f0]
    d = [x.copy() for x in f0]
    _, d1 = oracle.ref_simulation(nx, ny, nz, c, 7)
    _, d2 = oracle.ref_simulation(nx, ny, nz, d, 7, variant="interleaved", split=(1, 2, 2), workers=4)
    e = [x.copy() for x in f0]
    oracle.run(nx, ny, nz, e, oracle.Coeffs(nx, ny, nz), 7)
    assert d1 == d2 == oracle.digest(nx, ny, nz, e)


def test_energy_oracle_pinned(oracle):
    """total_energy restatement vs the reference's values (golden/energy.npz,
    fields.hpp:116-146): a stretched-grid value and a 60-step series."""
    d = np.load(os.path.join(GOLD, "energy.npz"))
    nx, ny, nz = (int(v) for v in d["dims"])
    f = oracle.fill_fields(nx, ny, nz, int(d["seeds"][0]))
    prev = oracle.fill_fields(nx, ny, nz, int(d["seeds"][1]))[3:]
    got = oracle.total_energy(nx, ny, nz, f, prev, d["dx"], d["dy"], d["dz"])
    assert abs(got - float(d["static"])) <= 1e-12 * abs(float(d["static"]))
    n, steps = int(d["n"]), int(d["steps"])
    src = oracle.Source(2, n // 2, n // 2, n // 2, d["table"])
    g = oracle.zeros_state(n, n, n)
    co = oracle.Coeffs(n, n, n)
    for t in range(steps):
        h = [a.copy() for a in g[3:]]
        oracle.run(n, n, n, g, co, 1, step0=t, sources=[src])
        want = float(d["series"][t])
        assert abs(oracle.total_energy(n, n, n, g, h) - want) <= 1e-12 * abs(want), t
    assert bits_equal(g, [d[f"out_{c}"] for c in oracle.COMP_NAMES])


def test_energy_kats(oracle):
    """kernel_test.cpp:265-283: E^2 with unit dual volume; H cross term."""
    n = 4
    f = oracle.zeros_state(n, n, n)
    h = [a.copy() for a in f[3:]]
    assert oracle.total_energy(n, n, n, f, h) == 0.0
    f[2][1, 2, 2] = 2.0  # ez(2,2,1)
    assert oracle.total_energy(n, n, n, f, h) == 4.0
    f = oracle.zeros_state(n, n, n)
    f[3][1, 1, 2] = 3.0  # hx(2,1,1)
    prev = [a.copy() for a in f[3:]]
    f[3][1, 1, 2] = 0.5
    assert oracle.total_energy(n, n, n, f, prev) == 1.5
