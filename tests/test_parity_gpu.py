"""GPU parity tests: the CUDA path (through the C-ABI) against the C oracle, the
golden fixtures generated from the compiled reference, and the reference's
known-answer tests. The bar is bit-exact (every component, every bit): the
product path is always built in bit-exact form (explicit _rn arithmetic,
--fmad=false), so the 1e-5 max-relative-error tolerance of north_star is
also checked (trivially) where stated."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL = 1e-5  # north_star: max |d| / max |ref| per component


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


def gfields(d, prefix):
    return [np.ascontiguousarray(d[f"{prefix}_{c}"]) for c in ("ex", "ey", "ez", "hx", "hy", "hz")]


def assert_bits(a, b, what=""):
    for c, (x, y) in enumerate(zip(a, b)):
        assert x.shape == y.shape, (what, c)
        bad = np.nonzero(x.view(np.uint32) != y.view(np.uint32))
        assert bad[0].size == 0, f"{what}: comp {c} differs at {len(bad[0])} DoFs, first (k,j,i)=" \
                                 f"{[int(v[0]) for v in bad]}: {x[tuple(v[0] for v in bad)]} vs " \
                                 f"{y[tuple(v[0] for v in bad)]}"


TB2, NAIVE, FUSED, TB4 = 0, 1, 2, 3  # include/yeeb200.h YB_VARIANT_* (ABI 3)
VARIANTS = [FUSED, NAIVE, TB2]


@pytest.mark.parametrize("variant", VARIANTS)
def test_golden_axis_src(yb, variant):
    d = load("axis_src")
    nx, ny, nz = (int(v) for v in d["dims"])
    c, i, j, k = (int(v) for v in d["src"])
    with yb.Simulation(nx, ny, nz, variant=variant) as sim:
        sim.add_source(c, i, j, k, d["table"])
        sim.upload(gfields(d, "in"))
        sim.run(int(d["steps"]))
        assert_bits(sim.download(), gfields(d, "out"), "axis_src")
        assert sim.digest() == int(d["digest"])
        assert sim.step_index == int(d["steps"])


@pytest.mark.parametrize("variant", VARIANTS)
def test_golden_stretched(yb, variant):
    d = load("stretched")
    nx, ny, nz = (int(v) for v in d["dims"])
    with yb.Simulation(nx, ny, nz, variant=variant, cdx=d["cdx"], cdy=d["cdy"], cdz=d["cdz"]) as sim:
        sim.upload(gfields(d, "in"))
        sim.run(int(d["steps"]))
        assert_bits(sim.download(), gfields(d, "out"), "stretched")
        assert sim.digest() == int(d["digest"])


@pytest.mark.parametrize("variant", VARIANTS)
def test_golden_reference_source(yb, variant):
    d = load("sim_refsrc")
    nx, ny, nz = (int(v) for v in d["dims"])
    c, i, j, k = (int(v) for v in d["src"])
    with yb.Simulation(nx, ny, nz, variant=variant) as sim:
        sim.add_source(c, i, j, k, d["table"])
        sim.run(int(d["steps"]))
        assert_bits(sim.download(), gfields(d, "out"), "sim_refsrc")
        assert sim.digest() == int(d["digest"])


def test_kat_range_ops(yb):
    n = 4
    h = np.full(n, 0.5, np.float32)
    with yb.Simulation(n, n, n, cdx=h, cdy=h, cdz=h) as sim:
        f = [np.zeros(yb.comp_extents(n, n, n, c)[::-1], np.float32) for c in range(6)]
        f[5][2, 2, 2] = 1.0
        sim.upload(f)
        sim.apply_ampere_range()
        assert_bits(sim.download(), gfields(load("kat_hz"), "out"), "kat_hz")
        for name, comp, idx in (("ey", 1, (2, 1, 1)), ("ez", 2, (1, 2, 1))):
            f = [np.zeros(yb.comp_extents(n, n, n, c)[::-1], np.float32) for c in range(6)]
            f[comp][idx] = 1.0
            sim.upload(f)
            sim.apply_faraday_range()
            assert_bits(sim.download(), gfields(load("kat_faraday"), name), "kat_faraday")
        # uniform H has zero curl (kernel_test.cpp:74-82)
        f = [np.zeros(yb.comp_extents(n, n, n, c)[::-1], np.float32) for c in range(6)]
        for c in (3, 4, 5):
            f[c][...] = 3.25
        sim.upload(f)
        sim.apply_ampere_range()
        assert_bits(sim.download(), f, "uniform H")
        # PEC zeroes exactly the shell (kernel_test.cpp:152-165)
        for c in range(3):
            f[c][...] = 1.0
        sim.upload(f)
        sim.apply_pec_boundary()
        g = sim.download()
        for c in range(3):
            ext = yb.comp_extents(n, n, n, c)
            kk, jj, ii = np.meshgrid(*[np.arange(e) for e in ext[::-1]], indexing="ij")
            idx = (ii, jj, kk)
            inner = np.ones(g[c].shape, bool)
            for a in range(3):
                if a != c:
                    inner &= (idx[a] >= 1) & (idx[a] <= n - 1)
            assert np.array_equal(g[c], inner.astype(np.float32))


def test_range_errors(yb):
    with yb.Simulation(4, 4, 4) as sim:
        with pytest.raises(yb.YeeOutOfRange):
            sim.apply_ampere_range((0, 6, 0, 4, 0, 4))  # kernel_test.cpp:136-138
        with pytest.raises(yb.YeeOutOfRange):
            sim.apply_faraday_range((0, 6, 0, 4, 0, 4))
        sim.apply_ampere_range((0, 2, 0, 2, 0, 2))  # sub-box is fine
        with pytest.raises(yb.YeeInvalidArgument):
            sim.add_source(2, 2, 0, 2, np.ones(3, np.float32))  # on the boundary
        with pytest.raises(yb.YeeInvalidArgument):
            sim.add_source(3, 2, 2, 2, np.ones(3, np.float32))  # magnetic
        with pytest.raises(yb.YeeInvalidArgument):
            sim.run(-1)


def oracle_run(oracle, nx, ny, nz, f, steps, medium=None, src=None, cd=None):
    co = oracle.Coeffs(nx, ny, nz)
    if cd is not None:
        co = oracle.Coeffs(nx, ny, nz, cdx=cd[0], cdy=cd[1], cdz=cd[2])
    if medium is not None:
        ca, cb, da, db = oracle.cell_coeffs(nx, ny, nz, *medium)
        co = oracle.Coeffs(nx, ny, nz, ca=ca, cb=cb, da=da, db=db)
    srcs = [oracle.Source(*src)] if src is not None else None
    oracle.run(nx, ny, nz, f, co, steps, sources=srcs)
    return f


CASES = {
    # name: (nx, ny, nz, steps, eps_seed, sigma_seed, field_seed, source?)
    "c1_vacuum_src": (40, 40, 40, 60, -1, -1, None, True),
    "c2_dielectric_src": (48, 40, 36, 60, 1, -1, None, True),
    "c3_lossy_fields": (64, 48, 40, 25, 2, 2, 3, False),
    "c4_slab_src": (136, 72, 40, 20, 4, -1, None, True),
    "c5_lossy_fields": (96, 64, 48, 15, 5, 5, 6, False),
    "odd_sizes": (37, 29, 23, 17, 7, 7, 8, True),
    "thin_x": (1, 9, 11, 9, 9, 9, 10, False),
    "thin_y": (21, 1, 7, 9, 9, 9, 10, False),
    "thin_z": (19, 13, 1, 9, 9, 9, 10, False),
    "two_tiles_partial": (133, 17, 9, 11, 3, 3, 4, True),
}


@pytest.mark.parametrize("variant", VARIANTS + ["tb2_one_sweep_per_launch"])
@pytest.mark.parametrize("name", sorted(CASES))
def test_configs_vs_oracle(yb, oracle, name, variant, monkeypatch):
    if variant == "tb2_one_sweep_per_launch":  # the two-step kernel without multi-sweep launches
        monkeypatch.setenv("YB_TB2_PERSIST", "0")
        variant = yb.VARIANT_TB2
    nx, ny, nz, steps, es, ss, fs, has_src = CASES[name]
    src = None
    if has_src and nx > 2 and ny > 2 and nz > 2:
        src = (2, nx // 2, ny // 2, nz // 2, oracle.gauss_table(steps))
    f = oracle.fill_fields(nx, ny, nz, fs) if fs is not None else oracle.zeros_state(nx, ny, nz)
    with yb.Simulation(nx, ny, nz, variant=variant) as sim:
        sim.generate_medium(es, ss)
        if src is not None:
            sim.add_source(*src[:4], src[4])
        if fs is not None:
            sim.fill(fs)
            assert_bits(sim.download(), f, "device fill")
        sim.run(steps)
        got = sim.download()
    want = oracle_run(oracle, nx, ny, nz, f, steps, medium=(es, ss) if es >= 0 or ss >= 0 else None,
                      src=src)
    assert max(oracle.max_rel_err(got, want)) <= TOL
    assert_bits(got, want, name)


@pytest.mark.parametrize("variant", [FUSED, TB2])
@pytest.mark.parametrize("shape,zchunk", [((40, 24, 30), 1), ((40, 24, 30), 3), ((40, 24, 30), 7),
                                          ((40, 24, 30), 64), ((200, 64, 40), 2), ((130, 40, 33), 1),
                                          ((256, 96, 21), 4)])
def test_zchunks_bit_identical(yb, oracle, shape, zchunk, variant):
    """Persistent CTAs stride over (tile, z-chunk) items; with many items per
    CTA the TMA ring runs across item boundaries (prologue/epilogue planes)."""
    (nx, ny, nz), steps = shape, 9
    f = oracle.fill_fields(nx, ny, nz, 41)
    with yb.Simulation(nx, ny, nz, zchunk=zchunk, variant=variant) as sim:
        sim.generate_medium(42, 43)
        sim.upload(f)
        sim.run(steps)
        got = sim.download()
    assert_bits(got, oracle_run(oracle, nx, ny, nz, f, steps, medium=(42, 43)), f"zchunk={zchunk}")


def test_uploaded_coefficients_match_generated(yb, oracle):
    nx, ny, nz = 33, 20, 18
    ca, cb, da, db = oracle.cell_coeffs(nx, ny, nz, 11, 12)
    f = oracle.fill_fields(nx, ny, nz, 13)
    with yb.Simulation(nx, ny, nz) as sim:
        for w, a in zip((yb.CA, yb.CB, yb.DA, yb.DB), (ca, cb, da, db)):
            sim.set_cell_coeffs(w, a)
        sim.upload(f)
        sim.run(8)
        assert sim.info()["n_cell_arrays"] == 4
        got = sim.download()
    assert_bits(got, oracle_run(oracle, nx, ny, nz, f, 8, medium=(11, 12)), "uploaded coeffs")


def test_uniform_arrays_compressed(yb, oracle):
    nx, ny, nz = 24, 20, 16
    S = yb.S
    f = oracle.fill_fields(nx, ny, nz, 3)
    with yb.Simulation(nx, ny, nz) as sim:
        sim.set_cell_coeffs(yb.CA, np.ones((nz, ny, nx), np.float32))
        sim.set_cell_coeffs(yb.CB, np.full((nz, ny, nx), S, np.float32))
        assert sim.info()["n_cell_arrays"] == 0
        sim.upload(f)
        sim.run(5)
        got = sim.download()
    assert_bits(got, oracle_run(oracle, nx, ny, nz, f, 5), "compressed")


def test_zero_steps_and_resume(yb, oracle):
    nx, ny, nz = 30, 22, 14
    f = oracle.fill_fields(nx, ny, nz, 77)
    tab = oracle.gauss_table(20)
    with yb.Simulation(nx, ny, nz) as sim:
        sim.generate_medium(5, 5)
        sim.upload(f)
        sim.run(0)
        assert_bits(sim.download(), f, "0 steps")  # PEC planes untouched before a step
        sim.add_source(1, 15, 11, 7, tab)
        sim.run(5)
        mid = sim.download()
        sim.run(7)
        got = sim.download()
        assert sim.step_index == 12
    with yb.Simulation(nx, ny, nz) as sim:  # checkpoint / resume: upload mid-state at step 5
        sim.generate_medium(5, 5)
        sim.add_source(1, 15, 11, 7, tab)
        sim.upload(mid)
        sim.step_index = 5
        sim.run(7)
        assert_bits(sim.download(), got, "resume")
    want = oracle_run(oracle, nx, ny, nz, f, 12, medium=(5, 5), src=(1, 15, 11, 7, tab))
    assert_bits(got, want, "resume vs oracle")


def test_full_config1_vs_oracle(yb, oracle):
    """BASELINE config 1 at full size: 128^3 vacuum, zero fields, PEC, Gaussian
    Ez source at the centre, 200 steps. Bit-exact against the oracle (which is
    bit-exact against the reference kernels on this path)."""
    n, steps = 128, 200
    tab = oracle.gauss_table(steps)
    with yb.Simulation(n, n, n) as sim:
        sim.add_source(2, n // 2, n // 2, n // 2, tab)
        sim.run(steps)
        got = sim.download()
        dig = sim.digest()
    want = oracle_run(oracle, n, n, n, oracle.zeros_state(n, n, n), steps,
                      src=(2, n // 2, n // 2, n // 2, tab))
    assert_bits(got, want, "config1")
    assert dig == oracle.digest(n, n, n, want)


@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_full_size_fused_equals_naive(yb, cfg):
    """Full-size configs 3 (512^3 lossy, 100 steps) and 5 (1024x1024x256 at one
    GPU, 100 steps): the fused, two-step and four-step sweeps equal the
    independent per-DoF path bit for bit (size-independent property; the
    oracle covers the cut-downs)."""
    if cfg == "c3":
        nx, ny, nz, es, ss, fs, steps = 512, 512, 512, 2, 2, 3, 100
    else:
        nx, ny, nz, es, ss, fs, steps = 1024, 1024, 256, 5, 5, 6, 100
    digs = []
    for variant in VARIANTS + [yb.VARIANT_TB4]:  # fused, naive, two-step, four-step
        with yb.Simulation(nx, ny, nz, variant=variant) as sim:
            sim.generate_medium(es, ss)
            sim.fill(fs)
            sim.run(steps)
            digs.append(sim.digest())
    assert len(set(digs)) == 1, digs


def test_cpp_shim_known_answers(yb, tmp_path):
    """The reference's Catch2 known-answer tests, restated in C++ against the
    drop-in shim (tests/cpp/shim_kat.cpp), executed on the GPU."""
    import subprocess
    from tests.test_abi import build_shim_kat
    exe = build_shim_kat(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "shim KATs ok" in r.stdout


PROBES = [(2, 20, 16, 14, 1), (3, 5, 6, 7, 3), (5, 10, 10, 29, 2), (0, 0, 0, 0, 5), (4, 39, 0, 28, 4)]


@pytest.mark.parametrize("variant", VARIANTS)
def test_device_probes_vs_oracle(yb, oracle, variant):
    """On-device point probes (probe.hpp:14-51 sample after each completed
    step t with t % stride == 0): same records and bit-identical values as the
    oracle stepped one step at a time. The two-step kernel splits pairs where
    a probe fires in between (stride 1 and 3 here)."""
    nx, ny, nz, steps = 40, 33, 29, 13
    f = oracle.fill_fields(nx, ny, nz, 21)
    tab = oracle.gauss_table(steps)
    src = (2, 20, 16, 14, tab)
    with yb.Simulation(nx, ny, nz, variant=variant) as sim:
        sim.generate_medium(3, 4)
        sim.add_source(*src)
        sim.upload(f)
        sim.set_probes(PROBES)
        sim.run(5)
        st0, pr0, va0 = sim.read_probes(capacity=3)  # partial drain keeps the tail
        sim.run(steps - 5)
        st1, pr1, va1 = sim.read_probes()
        assert sim.read_probes()[0].size == 0
    st, pr, va = (np.concatenate(x) for x in ((st0, st1), (pr0, pr1), (va0, va1)))
    ca, cb, da, db = oracle.cell_coeffs(nx, ny, nz, 3, 4)
    co = oracle.Coeffs(nx, ny, nz, ca=ca, cb=cb, da=da, db=db)
    want = []
    for t in range(steps):
        oracle.run(nx, ny, nz, f, co, 1, step0=t, sources=[oracle.Source(*src)])
        for q, (c, i, j, k, s) in enumerate(PROBES):
            if (t + 1) % s == 0:
                want.append((t + 1, q, f[c][k, j, i]))
    assert list(zip(st.tolist(), pr.tolist())) == [(a, b) for a, b, _ in want]
    assert np.array_equal(va.view(np.uint32), np.array([v for *_, v in want], np.float32).view(np.uint32))


def test_probe_validation(yb):
    with yb.Simulation(8, 8, 8) as sim:
        for bad in [(2, 0, 0, 0, 0), (2, 9, 0, 0, 1), (0, 8, 0, 0, 1), (3, 0, 8, 0, 1), (5, 0, 0, 9, 1), (6, 0, 0, 0, 1)]:
            with pytest.raises(yb.YeeInvalidArgument):
                sim.set_probes([bad])
        with pytest.raises(yb.YeeInvalidArgument):
            sim.set_probes([(2, 1, 1, 1, 1)] * 65)
        sim.set_probes([(5, 7, 7, 8, 1)])  # hz has nz+1 planes
        sim.run(2)
        st, pr, va = sim.read_probes()
        assert st.tolist() == [1, 2] and pr.tolist() == [0, 0]
        sim.set_probes([])
        sim.run(2)
        assert sim.read_probes()[0].size == 0


def test_energy_vs_reference_golden(yb, oracle):
    """Device total_energy (fields.hpp:116-146) against the reference's values
    (golden/energy.npz): stretched spacing, and the per-step leapfrog
    invariant of a sourced 20^3 run (measure_energy_drift pattern). Double
    accumulation in a different order: relative 1e-12."""
    d = load("energy")
    nx, ny, nz = (int(v) for v in d["dims"])
    f = oracle.fill_fields(nx, ny, nz, int(d["seeds"][0]))
    prev = oracle.fill_fields(nx, ny, nz, int(d["seeds"][1]))
    with yb.Simulation(nx, ny, nz) as sim:
        with pytest.raises(yb.YeeInvalidArgument):
            sim.total_energy()
        sim.upload(prev)
        sim.snapshot_h()
        sim.upload(f)
        got = sim.total_energy(d["dx"], d["dy"], d["dz"])
    assert abs(got - float(d["static"])) <= 1e-12 * abs(float(d["static"]))
    n, steps = int(d["n"]), int(d["steps"])
    for variant in VARIANTS:
        with yb.Simulation(n, n, n, variant=variant) as sim:
            sim.add_source(2, n // 2, n // 2, n // 2, d["table"])
            for t in range(steps):
                sim.snapshot_h()
                sim.run(1)
                want = float(d["series"][t])
                assert abs(sim.total_energy() - want) <= 1e-12 * abs(want), (variant, t)
            assert_bits(sim.download(), gfields(d, "out"), "energy run")


def test_energy_drift_single_precision(yb, oracle):
    """SPEC.md:539 / bench.hpp:273-303: 64^3 vacuum cavity, source on for 50
    steps, 1000 steps: single-precision relative drift < 1e-4."""
    n, steps, on = 64, 1000, 50
    tab = oracle.gauss_table(on, t0=25.0, w=8.0)
    with yb.Simulation(n, n, n) as sim:
        sim.add_source(2, n // 2, n // 2, n // 2, tab)
        sim.run(on)
        sim.snapshot_h()
        sim.run(1)
        e0 = sim.total_energy()
        drift = 0.0
        for t in range(on + 1, steps):
            sim.snapshot_h()
            sim.run(1)
            drift = max(drift, abs(sim.total_energy() - e0) / abs(e0))
    assert e0 > 0 and drift < 1e-4, drift


def test_energy_slabs_sum(yb, oracle):
    """On z-slabs each rank sums the planes it owns; the sum over slabs equals
    the single-domain invariant (rel 1e-12)."""
    from paper_1301_4539_b200.slabs import partition
    nx, ny, nzg = 40, 24, 21
    dz = np.linspace(0.8, 1.2, nzg)
    f = oracle.fill_fields(nx, ny, nzg, 5)
    prev = oracle.fill_fields(nx, ny, nzg, 6)
    with yb.Simulation(nx, ny, nzg) as one:
        one.upload(prev)
        one.snapshot_h()
        one.upload(f)
        want = one.total_energy(dz=dz)
    total = 0.0
    for z0, n in partition(nzg, 3):
        with yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg) as s:
            s.fill(6)
            s.snapshot_h()
            s.fill(5)
            total += s.total_energy(dz=dz)
    assert abs(total - want) <= 1e-12 * abs(want)
    assert abs(want - oracle.total_energy(nx, ny, nzg, f, prev[3:], dz=dz)) <= 1e-12 * abs(want)


@pytest.mark.parametrize("variant", [FUSED, TB2])
@pytest.mark.parametrize("shape,zchunk,medium", [((136, 72, 40), 4, (4, -1)), ((200, 40, 33), 0, (-1, -1)),
                                                 ((64, 48, 40), 3, (2, 2)), ((37, 29, 23), 0, (7, 7))])
def test_quiescent_skip_bit_exact(yb, oracle, variant, shape, zchunk, medium):
    """runner.hpp:60-73: skipping all-zero work items changes nothing. A
    point source in a zero field (the configs 1/2/4 situation), skip on vs
    off vs the oracle; the skip must actually fire early on."""
    nx, ny, nz = shape
    steps = 23
    tab = oracle.gauss_table(steps, t0=4.0, w=2.0)
    src = (2, nx // 3, ny // 2, nz // 4, tab)
    outs = []
    for skip in (False, True):
        with yb.Simulation(nx, ny, nz, variant=variant, zchunk=zchunk) as sim:
            sim.generate_medium(*medium)
            sim.add_source(*src)
            sim.set_quiescent_skip(skip)
            sim.run(steps)
            outs.append(sim.download())
            inf = sim.info()
            assert inf["quiescent_skip"] == int(skip)
            if skip and nx * ny * nz > 100000:
                assert inf["skipped_items"] > 0
    assert_bits(outs[1], outs[0], "skip vs no skip")
    want = oracle_run(oracle, nx, ny, nz, oracle.zeros_state(nx, ny, nz), steps,
                      medium=medium if medium != (-1, -1) else None, src=src)
    assert_bits(outs[1], want, "skip vs oracle")


@pytest.mark.parametrize("variant", [FUSED, TB2])
def test_quiescent_skip_stale_buffers(yb, oracle, variant):
    """After a run leaves nonzero state in both buffers, an upload of a mostly
    zero state must rebuild the quiescent map (both buffers are scanned): the
    result equals a fresh simulation's."""
    nx, ny, nz = 140, 40, 30
    tab = oracle.gauss_table(12, t0=3.0, w=2.0)
    f = oracle.zeros_state(nx, ny, nz)
    f[2][5, 20, 70] = 1.0  # one nonzero Ez
    with yb.Simulation(nx, ny, nz, variant=variant) as sim:
        sim.set_quiescent_skip(True)
        sim.fill(9)
        sim.run(7)  # both buffers now hold nonzero data everywhere
        sim.upload(f)
        sim.step_index = 0
        sim.add_source(2, 100, 10, 25, tab)
        sim.run(12)
        got = sim.download()
        assert sim.info()["skipped_items"] > 0
    want = oracle_run(oracle, nx, ny, nz, [a.copy() for a in f], 12, src=(2, 100, 10, 25, tab))
    assert_bits(got, want, "stale buffers")


def test_quiescent_skip_slabs(yb, oracle):
    """z-slabs with skipping on: ghost planes written by the halo exchange are
    scanned into the map; the assembled result equals one domain."""
    from paper_1301_4539_b200.slabs import partition
    nx, ny, nzg, steps = 136, 40, 29, 11
    tab = oracle.gauss_table(steps, t0=3.0, w=2.0)
    src = (2, 60, 20, 13, tab)
    for variant in (FUSED, TB2):
        sims = []
        for z0, n in partition(nzg, 3):
            s = yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, variant=variant)
            s.generate_medium(3, -1)
            s.add_source(*src)
            s.set_quiescent_skip(True)
            sims.append(s)
        import torch
        bufs = [(torch.empty(lo.halo_bytes(1, False), dtype=torch.uint8, device="cuda"),
                 torch.empty(hi.halo_bytes(0, False), dtype=torch.uint8, device="cuda"))
                for lo, hi in zip(sims[:-1], sims[1:])]
        depth = sims[0].info()["halo_depth"]
        done = 0
        while done < steps:
            n = min(depth, steps - done)
            for (lo, hi), (up, down) in zip(zip(sims[:-1], sims[1:]), bufs):
                lo.halo_pack(1, up.data_ptr())
                hi.halo_pack(0, down.data_ptr())
                hi.halo_unpack(0, up.data_ptr())
                lo.halo_unpack(1, down.data_ptr())
            for s in sims:
                s.run(n)
            done += n
        out = oracle.zeros_state(nx, ny, nzg)
        for s in sims:
            d = s.download()
            top = s.z_offset + s.nz == nzg
            for c in range(6):
                k = s.nz + (1 if c in (0, 1, 5) and top else 0)
                out[c][s.z_offset:s.z_offset + k] = d[c][:k]
            s.close()
        want = oracle_run(oracle, nx, ny, nzg, oracle.zeros_state(nx, ny, nzg), steps, medium=(3, -1), src=src)
        assert_bits(out, want, f"slabs skip variant {variant}")


@pytest.mark.parametrize("name", ["c1_vacuum_src", "c3_lossy_fields", "odd_sizes", "two_tiles_partial", "thin_x",
                                  "thin_y", "thin_z", "c4_slab_src", "c2_dielectric_src"])
def test_tb4_vs_oracle(yb, oracle, name):
    """Four steps per sweep (YB_VARIANT_TB4, the depth-8 point of the config-5
    sweep): bit-exact against the oracle; step counts not divisible by four
    finish with two-step / one-step launches."""
    nx, ny, nz, steps, es, ss, fs, has_src = CASES[name]
    src = None
    if has_src and nx > 2 and ny > 2 and nz > 2:
        src = (2, nx // 2, ny // 2, nz // 2, oracle.gauss_table(steps))
    f = oracle.fill_fields(nx, ny, nz, fs) if fs is not None else oracle.zeros_state(nx, ny, nz)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB4) as sim:
        sim.generate_medium(es, ss)
        if src is not None:
            sim.add_source(*src[:4], src[4])
        if fs is not None:
            sim.fill(fs)
        sim.run(steps)
        got = sim.download()
    want = oracle_run(oracle, nx, ny, nz, f, steps, medium=(es, ss) if es >= 0 or ss >= 0 else None, src=src)
    assert_bits(got, want, name)


@pytest.mark.parametrize("zchunk", [1, 3, 9, 0])
def test_tb4_zchunks_and_probes(yb, oracle, zchunk):
    nx, ny, nz, steps = 120, 26, 31, 12
    f = oracle.fill_fields(nx, ny, nz, 41)
    with yb.Simulation(nx, ny, nz, zchunk=zchunk, variant=yb.VARIANT_TB4) as sim:
        sim.generate_medium(42, 43)
        sim.upload(f)
        sim.set_probes([(2, 60, 13, 15, 3), (3, 5, 6, 7, 4)])
        sim.run(steps)
        got = sim.download()
        st, pr, va = sim.read_probes()
    want = oracle_run(oracle, nx, ny, nz, [a.copy() for a in f], steps, medium=(42, 43))
    assert_bits(got, want, f"tb4 zchunk={zchunk}")
    assert st.tolist() == [3, 4, 6, 8, 9, 12, 12] and pr.tolist() == [0, 1, 0, 1, 0, 0, 1]


@pytest.mark.parametrize("name", ["c2_dielectric_src", "c3_lossy_fields", "odd_sizes", "two_tiles_partial",
                                  "thin_z"])
@pytest.mark.parametrize("zchunk", [0, 1, 4])
def test_multi_sweep_launches(yb, oracle, name, zchunk, monkeypatch):
    """Several two-step sweeps per launch (YB_TB2_PERSIST=1): items of sweep s
    start once their neighbourhood finished sweep s-1 (device-side completion
    epochs). Bit-exact, with per-sweep sources."""
    monkeypatch.setenv("YB_TB2_PERSIST", "1")
    nx, ny, nz, steps, es, ss, fs, has_src = CASES[name]
    src = None
    if has_src and nx > 2 and ny > 2 and nz > 2:
        src = (2, nx // 2, ny // 2, nz // 2, oracle.gauss_table(steps))
    f = oracle.fill_fields(nx, ny, nz, fs) if fs is not None else oracle.zeros_state(nx, ny, nz)
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2, zchunk=zchunk) as sim:
        sim.generate_medium(es, ss)
        if src is not None:
            sim.add_source(*src[:4], src[4])
        if fs is not None:
            sim.fill(fs)
        sim.run(steps)
        launches = sim.info()["kernel_launches"]
        got = sim.download()
    assert launches <= 3 + steps % 2  # the pairs ran in one launch
    want = oracle_run(oracle, nx, ny, nz, f, steps, medium=(es, ss) if es >= 0 or ss >= 0 else None, src=src)
    assert_bits(got, want, name)


@pytest.mark.parametrize("variant", [FUSED, TB2, TB4])
def test_uniform_non_unit_ca_da(yb, oracle, variant):
    """A uniform Ca / Da other than 1 (yb_set_cell_coeffs(which, NULL, v)):
    stored as a full array (the sweep kernels treat 'no array' as exactly 1)."""
    nx, ny, nz, steps = 44, 30, 20, 8
    f = oracle.fill_fields(nx, ny, nz, 17)
    with yb.Simulation(nx, ny, nz, variant=variant) as sim:
        sim.set_cell_coeffs(yb.CA, None, 0.75)
        sim.set_cell_coeffs(yb.DA, np.full((nz, ny, nx), 0.5, np.float32))
        assert sim.info()["n_cell_arrays"] == 2
        sim.upload(f)
        sim.run(steps)
        got = sim.download()
    co = oracle.Coeffs(nx, ny, nz, ca_s=0.75, da_s=0.5)
    want = [a.copy() for a in f]
    oracle.run(nx, ny, nz, want, co, steps)
    assert_bits(got, want, "uniform Ca/Da != 1")


def test_cell_coeffs_batched_equals_single(yb, oracle):
    """yb_set_cell_coeffs_n (back-to-back copies, one sync) stores exactly what
    four yb_set_cell_coeffs calls store — including a uniform array (kept as
    the compressed uniform form) and a uniform Da != 1 (a full array)."""
    nx, ny, nz, steps = 44, 30, 20, 6
    ca, cb, da, db = oracle.cell_coeffs(nx, ny, nz, 5, 6)
    cb_u = np.full((nz, ny, nx), cb.flat[0], np.float32)
    da_u = np.full((nz, ny, nx), 0.5, np.float32)
    f = oracle.fill_fields(nx, ny, nz, 9)
    outs = []
    for batched in (False, True):
        with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as sim:
            arrays = {yb.CA: ca, yb.CB: cb_u, yb.DA: da_u, yb.DB: db}
            if batched:
                sim.set_cell_coeffs_many(arrays)
            else:
                for w, a in arrays.items():
                    sim.set_cell_coeffs(w, a)
            info = sim.info()
            sim.upload(f)
            sim.run(steps)
            outs.append((info["n_cell_arrays"], sim.download()))
    assert outs[0][0] == outs[1][0]
    assert_bits(outs[1][1], outs[0][1], "batched coefficients")
    co = oracle.Coeffs(nx, ny, nz, ca=ca, cb=cb_u, da=da_u, db=db)
    want = [a.copy() for a in f]
    oracle.run(nx, ny, nz, want, co, steps)
    assert_bits(outs[1][1], want, "batched vs oracle")
    with yb.Simulation(nx, ny, nz) as sim:
        with pytest.raises(yb.YeeInvalidArgument):
            sim.set_cell_coeffs_many({yb.CA: ca, 7: cb})


@pytest.mark.parametrize("shape", [(700, 40, 24), (1300, 40, 20), (1030, 72, 40)])
@pytest.mark.parametrize("xblock", ["default", "0", "1", "3"])
def test_multisweep_column_block_order(yb, oracle, shape, xblock, monkeypatch):
    """Multi-sweep launches hand a sweep's tiles out in column blocks (FusedArgs::xblock, 4 tiles
    wide by default; the last block may be narrower): any width gives the bits of the one-step
    kernel and of the oracle — grids with 6 / 11 / 9 tile columns, plain runs and both streamed
    calls (whose skewed orders keep the block order in their sweep-major part)."""
    torch = pytest.importorskip("torch")
    nx, ny, nz = shape
    steps = 24
    if xblock != "default":
        monkeypatch.setenv("YB_TB2_XBLOCK", xblock)
    monkeypatch.setenv("YB_UP_STREAM", "1")
    ca, cb, da, db = oracle.cell_coeffs(nx, ny, nz, 2, 2)
    want = oracle.fill_fields(nx, ny, nz, 3)
    start = [a.copy() for a in want]
    oracle.run(nx, ny, nz, want, oracle.Coeffs(nx, ny, nz, ca=ca, cb=cb, da=da, db=db), steps)

    def pin(a):
        t = torch.empty(a.shape, dtype=torch.float32).pin_memory()
        t.numpy()[...] = a
        return t.numpy()

    cells = {q: pin(a.reshape(nz, ny, nx)) for q, a in enumerate((ca, cb, da, db))}
    pf = [pin(a) for a in start]
    out = [torch.empty(a.shape, dtype=torch.float32).pin_memory().numpy() for a in start]
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        s.set_cell_coeffs_many(cells)
        s.upload(start)
        s.run(steps)
        assert s.info()["kernel_launches"] == 1
        got = s.download()
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        got2 = s.run_streamed(steps, cells, pf, out=out)
        assert s.info()["streamed_uploads"] == 1
    for c in range(6):
        assert np.array_equal(got[c].view(np.uint32), want[c].view(np.uint32)), (shape, xblock, c)
        assert np.array_equal(got2[c].view(np.uint32), want[c].view(np.uint32)), (shape, xblock, c)
