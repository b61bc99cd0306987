"""Per-box operations on a caller's host FieldSet (yb_fs_apply /
yb_fs_total_energy, the shim's free functions of kernels.hpp:78-155 and
fields.hpp:116-146) in both precisions: fp32 against the C oracle (pinned to
the reference), fp64 against a numpy restatement with the reference's operand
order (IEEE double per operation, nothing fused) — bit-exact either way."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rand_fields(yb, nx, ny, nz, dt, seed):
    rng = np.random.default_rng(seed)
    return [rng.uniform(-1, 1, yb.comp_extents(nx, ny, nz, c)[::-1]).astype(dt) for c in range(6)]


def np_ampere(f, cd, box):
    """kernels.hpp:18-20 over box ∩ curl_updatable_box, arrays (k, j, i)."""
    ex, ey, ez, hx, hy, hz = f
    cdx, cdy, cdz = cd
    nz, ny, nx = hx.shape[0], hx.shape[1], ey.shape[2] - 1
    x0, x1, y0, y1, z0, z1 = box
    def rng(lo, hi, a, b):
        return max(lo, a), min(hi, b)
    i0, i1 = rng(x0, x1, 0, nx); j0, j1 = rng(y0, y1, 1, ny); k0, k1 = rng(z0, z1, 1, nz)
    if i1 > i0 and j1 > j0 and k1 > k0:
        K, J, I = np.ix_(range(k0, k1), range(j0, j1), range(i0, i1))
        ex[K, J, I] = ex[K, J, I] + (cdy[J] * (hz[K, J, I] - hz[K, J - 1, I]) - cdz[K] * (hy[K, J, I] - hy[K - 1, J, I]))
    i0, i1 = rng(x0, x1, 1, nx); j0, j1 = rng(y0, y1, 0, ny); k0, k1 = rng(z0, z1, 1, nz)
    if i1 > i0 and j1 > j0 and k1 > k0:
        K, J, I = np.ix_(range(k0, k1), range(j0, j1), range(i0, i1))
        ey[K, J, I] = ey[K, J, I] + (cdz[K] * (hx[K, J, I] - hx[K - 1, J, I]) - cdx[I] * (hz[K, J, I] - hz[K, J, I - 1]))
    i0, i1 = rng(x0, x1, 1, nx); j0, j1 = rng(y0, y1, 1, ny); k0, k1 = rng(z0, z1, 0, nz)
    if i1 > i0 and j1 > j0 and k1 > k0:
        K, J, I = np.ix_(range(k0, k1), range(j0, j1), range(i0, i1))
        ez[K, J, I] = ez[K, J, I] + (cdx[I] * (hy[K, J, I] - hy[K, J, I - 1]) - cdy[J] * (hx[K, J, I] - hx[K, J - 1, I]))


def np_faraday(f, cd):
    """kernels.hpp:23-25 over the full H extents."""
    ex, ey, ez, hx, hy, hz = f
    cdx, cdy, cdz = (c.reshape(s) for c, s in zip(cd, ((1, 1, -1), (1, -1, 1), (-1, 1, 1))))
    hx[...] = hx + (cdz * (ey[1:, :, :] - ey[:-1, :, :]) - cdy * (ez[:, 1:, :] - ez[:, :-1, :]))
    hy[...] = hy + (cdx * (ez[:, :, 1:] - ez[:, :, :-1]) - cdz * (ex[1:, :, :] - ex[:-1, :, :]))
    hz[...] = hz + (cdy * (ex[:, 1:, :] - ex[:, :-1, :]) - cdx * (ey[:, :, 1:] - ey[:, :, :-1]))


def bits(a):
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


@pytest.mark.parametrize("dims", [(9, 7, 5), (16, 3, 11), (1, 4, 4)])
def test_fs_ops_fp64_vs_numpy(yb, dims):
    nx, ny, nz = dims
    rng = np.random.default_rng(1)
    cd = [rng.uniform(0.2, 0.6, n) for n in dims]
    f = rand_fields(yb, nx, ny, nz, np.float64, 2)
    want = [a.copy() for a in f]
    for box in ((0, nx + 1, 0, ny + 1, 0, nz + 1), (1, max(2, nx - 1), 0, 3, 2, nz + 1)):
        yb.fs_apply(f, cd, yb.OP_AMPERE, box=box)
        np_ampere(want, cd, box)
        for c in range(6):
            assert np.array_equal(bits(f[c]), bits(want[c])), (box, c)
    yb.fs_apply(f, cd, yb.OP_FARADAY, box=(0, nx + 1, 0, ny + 1, 0, nz + 1))
    np_faraday(want, [np.asarray(c) for c in cd])
    for c in range(6):
        assert np.array_equal(bits(f[c]), bits(want[c])), c


def test_fs_ops_fp32_vs_oracle(yb, oracle):
    nx, ny, nz = 21, 13, 9
    f = rand_fields(yb, nx, ny, nz, np.float32, 3)
    want = [a.copy() for a in f]
    co = oracle.Coeffs(nx, ny, nz)
    cd = [co.cdx, co.cdy, co.cdz]
    yb.fs_apply(f, cd, yb.OP_AMPERE, box=(0, nx + 1, 0, ny + 1, 0, nz + 1))
    yb.fs_apply(f, None, yb.OP_PEC)
    yb.fs_apply(f, cd, yb.OP_FARADAY, box=(0, nx + 1, 0, ny + 1, 0, nz + 1))
    oracle.ampere(nx, ny, nz, want, co)
    oracle.pec(nx, ny, nz, want)
    oracle.faraday(nx, ny, nz, want, co)
    for c in range(6):
        assert np.array_equal(bits(f[c]), bits(want[c])), c


def test_fs_ops_boxes_and_errors(yb):
    nx, ny, nz = 6, 5, 4
    f = rand_fields(yb, nx, ny, nz, np.float64, 4)
    cd = [np.full(n, 0.5) for n in (nx, ny, nz)]
    g = [a.copy() for a in f]
    yb.fs_apply(g, None, yb.OP_ZERO, comp=4, box=(1, 3, 0, 2, 1, 2))  # zero_box
    assert np.all(g[4][1:2, 0:2, 1:3] == 0) and np.array_equal(g[4][0], f[4][0])
    with pytest.raises(yb.YeeOutOfRange):
        yb.fs_apply(g, cd, yb.OP_AMPERE, box=(0, nx + 2, 0, ny, 0, nz))
    with pytest.raises(yb.YeeOutOfRange):  # update_e_box on a PEC plane (kernel_test.cpp:140-141)
        yb.fs_apply(g, cd, yb.OP_UPDATE_E, comp=0, box=(0, nx, 0, ny + 1, 0, nz + 1))
    with pytest.raises(yb.YeeOutOfRange):
        yb.fs_apply(g, cd, yb.OP_UPDATE_H, comp=3, box=(0, nx + 2, 0, ny, 0, nz))
    with pytest.raises(yb.YeeInvalidArgument):
        yb.fs_apply(g, cd, yb.OP_UPDATE_E, comp=3, box=(1, 2, 1, 2, 1, 2))
    h = [a.copy() for a in g]
    yb.fs_apply(h, cd, yb.OP_UPDATE_E, comp=1, box=(2, 2, 1, 3, 1, 3))  # empty box: no-op
    for c in range(6):
        assert np.array_equal(bits(h[c]), bits(g[c]))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_fs_total_energy(yb, oracle, dt):
    nx, ny, nz = 8, 6, 5
    f = rand_fields(yb, nx, ny, nz, dt, 5)
    prev = [a.copy() for a in f[3:]]
    dx = np.linspace(0.5, 1.5, nx)
    e = yb.fs_total_energy(f, prev, dx=dx)
    want = oracle.total_energy(nx, ny, nz, [a.astype(np.float64) for a in f], [a.astype(np.float64) for a in prev],
                               dx=dx)
    assert abs(e - want) <= 1e-12 * abs(want)
