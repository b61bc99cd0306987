"""ctypes front end for the CPU ORACLE (test infrastructure only).

Loads oracle/liboracle.so (the C restatement, yee_oracle.c) and, when built,
oracle/_ref/libyeeref.so (the unmodified reference headers compiled by
oracle/Makefile). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs import this module; the product package
(paper_1301_4539_b200) never does.

Field states are lists of six numpy float32 arrays in the reference's dense
Array3 layout: shape (ez, ey, ex) of each component's extents
(staggering.hpp:34-39), x fastest (array3.hpp:104-107).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libyeeref.so")

COMP_NAMES = ("ex", "ey", "ez", "hx", "hy", "hz")
_f32p = C.POINTER(C.c_float)


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def comp_extents(nx, ny, nz, comp):
    """(ex, ey, ez) extents of a component (staggering.hpp:34-39)."""
    n = (nx, ny, nz)
    axis = comp % 3
    electric = comp < 3
    return tuple(n[a] + (1 if (electric and a != axis) or (not electric and a == axis) else 0)
                 for a in range(3))


def zeros_state(nx, ny, nz):
    return [np.zeros(comp_extents(nx, ny, nz, c)[::-1], dtype=np.float32) for c in range(6)]


class _YoState(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("f", _f32p * 6)]


class _YoCoeffs(C.Structure):
    _fields_ = [("ca", _f32p), ("cb", _f32p), ("da", _f32p), ("db", _f32p),
                ("ca_s", C.c_float), ("da_s", C.c_float),
                ("cdx", _f32p), ("cdy", _f32p), ("cdz", _f32p)]


class _YoSource(C.Structure):
    _fields_ = [("comp", C.c_int), ("i", C.c_int), ("j", C.c_int), ("k", C.c_int),
                ("table", _f32p), ("n", C.c_int64)]


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_f32p)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.yo_step.argtypes = [C.POINTER(_YoState), C.POINTER(_YoCoeffs), C.POINTER(_YoSource),
                              C.c_int, C.c_int64, C.c_int]
        L.yo_run.argtypes = [C.POINTER(_YoState), C.POINTER(_YoCoeffs), C.POINTER(_YoSource),
                             C.c_int, C.c_int64, C.c_int64, C.c_int]
        L.yo_ampere.argtypes = [C.POINTER(_YoState), C.POINTER(_YoCoeffs), C.c_int]
        L.yo_faraday.argtypes = [C.POINTER(_YoState), C.POINTER(_YoCoeffs), C.c_int]
        L.yo_pec.argtypes = [C.POINTER(_YoState)]
        L.yo_digest.argtypes = [C.POINTER(_YoState)]
        L.yo_digest.restype = C.c_uint64
        L.yo_fill_fields.argtypes = [C.POINTER(_YoState), C.c_uint64, C.c_int]
        L.yo_make_cell_coeffs.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                          _f32p, _f32p, _f32p, _f32p, C.c_int]
        L.yo_courant.restype = C.c_float
        L.yo_gauss_table.argtypes = [_f32p, C.c_int64, C.c_double, C.c_double]
        _lib = L
    return _lib


def have_ref():
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        R = C.CDLL(REF_PATH)
        R.yr_last_error.restype = C.c_char_p
        R.yr_uniform_dt.argtypes = [C.c_int, C.c_float, C.c_float, C.c_double]
        R.yr_uniform_dt.restype = C.c_float
        R.yr_stable_dt.argtypes = [C.c_int] * 3 + [_f32p] * 3 + [C.c_float, C.c_double]
        R.yr_stable_dt.restype = C.c_double
        R.yr_build_coefficients.argtypes = [C.c_int] * 3 + [_f32p] * 3 + [C.c_float, C.c_float] + [_f32p] * 3
        R.yr_run_kernels.argtypes = ([C.c_int] * 3 + [_f32p] * 3 + [C.c_float, C.c_float, _f32p * 6,
                                     C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                     _f32p, C.c_int64, C.c_int])
        R.yr_simulation.argtypes = ([C.c_int] * 3 + [C.c_float, C.c_float, C.c_double]
                                    + [C.c_int] * 11 + [C.c_double] * 3
                                    + [C.c_int64, _f32p * 6, C.c_int64, C.c_int64,
                                       C.POINTER(C.c_double), C.POINTER(C.c_uint64)])
        R.yr_source_table.argtypes = ([C.c_int] * 7 + [C.c_double] * 3
                                      + [C.c_int64, C.c_double, C.c_int64, _f32p])
        R.yr_source_table.restype = C.c_int64
        R.yr_digest.argtypes = [C.c_int] * 3 + [_f32p * 6]
        R.yr_digest.restype = C.c_uint64
        R.yr_total_energy.argtypes = [C.c_int] * 3 + [_f32p] * 3 + [_f32p * 6, _f32p * 3]
        R.yr_total_energy.restype = C.c_double
        R.yr_run_case.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int, C.c_int,
                                  C.c_char_p, C.c_char_p, C.c_int64]
        R.yr_run_case.restype = C.c_int64
        _ref = R
    return _ref


def courant():
    return np.float32(lib().yo_courant())


def _state(nx, ny, nz, fields):
    st = _YoState(nx, ny, nz)
    for c in range(6):
        assert fields[c].shape == comp_extents(nx, ny, nz, c)[::-1], (c, fields[c].shape)
        st.f[c] = _p(fields[c])
    return st


class Coeffs:
    """Coefficient set (yo_coeffs). Keeps numpy arrays alive."""

    def __init__(self, nx, ny, nz, ca=None, cb=None, da=None, db=None,
                 ca_s=1.0, da_s=1.0, cdx=None, cdy=None, cdz=None):
        S = courant()
        self.cdx = np.full(nx, S, np.float32) if cdx is None else np.ascontiguousarray(cdx, np.float32)
        self.cdy = np.full(ny, S, np.float32) if cdy is None else np.ascontiguousarray(cdy, np.float32)
        self.cdz = np.full(nz, S, np.float32) if cdz is None else np.ascontiguousarray(cdz, np.float32)
        self.ca, self.cb, self.da, self.db = ca, cb, da, db
        self.ca_s, self.da_s = ca_s, da_s

    def struct(self):
        return _YoCoeffs(_p(self.ca), _p(self.cb), _p(self.da), _p(self.db),
                         self.ca_s, self.da_s, _p(self.cdx), _p(self.cdy), _p(self.cdz))


def cell_coeffs(nx, ny, nz, eps_seed, sigma_seed, threads=0):
    """Per-cell (ca, cb, da, db) arrays, shape (nz, ny, nx) (yeeb200_inputs.h)."""
    arrs = [np.empty((nz, ny, nx), np.float32) for _ in range(4)]
    lib().yo_make_cell_coeffs(nx, ny, nz, eps_seed, sigma_seed, *[_p(a) for a in arrs],
                              threads or os.cpu_count())
    return arrs


def fill_fields(nx, ny, nz, seed, threads=0):
    f = zeros_state(nx, ny, nz)
    st = _state(nx, ny, nz, f)
    lib().yo_fill_fields(C.byref(st), seed, threads or os.cpu_count())
    return f


def gauss_table(n, t0=40.0, w=12.0):
    t = np.empty(n, np.float32)
    lib().yo_gauss_table(_p(t), n, t0, w)
    return t


class Source:
    def __init__(self, comp, i, j, k, table):
        self.comp, self.i, self.j, self.k = comp, i, j, k
        self.table = np.ascontiguousarray(table, np.float32)

    def struct(self):
        return _YoSource(self.comp, self.i, self.j, self.k, _p(self.table), len(self.table))


def _sources(srcs):
    srcs = srcs or []
    arr = (_YoSource * max(1, len(srcs)))()
    for q, s in enumerate(srcs):
        arr[q] = s.struct()
    return arr, len(srcs)


def run(nx, ny, nz, fields, coeffs, nsteps, step0=0, sources=None, threads=0):
    """Advances `fields` (in place) by nsteps Standard steps."""
    st = _state(nx, ny, nz, fields)
    co = coeffs.struct()
    arr, n = _sources(sources)
    lib().yo_run(C.byref(st), C.byref(co), arr, n, step0, nsteps, threads or os.cpu_count())
    return fields


def ampere(nx, ny, nz, fields, coeffs, threads=1):
    st = _state(nx, ny, nz, fields)
    co = coeffs.struct()
    lib().yo_ampere(C.byref(st), C.byref(co), threads)


def faraday(nx, ny, nz, fields, coeffs, threads=1):
    st = _state(nx, ny, nz, fields)
    co = coeffs.struct()
    lib().yo_faraday(C.byref(st), C.byref(co), threads)


def pec(nx, ny, nz, fields):
    st = _state(nx, ny, nz, fields)
    lib().yo_pec(C.byref(st))


def digest(nx, ny, nz, fields):
    st = _state(nx, ny, nz, fields)
    return int(lib().yo_digest(C.byref(st)))


# ---------------------------------------------------------------- reference
def _fptrs(fields):
    arr = (_f32p * 6)()
    for c in range(6):
        arr[c] = _p(fields[c])
    return arr


def ref_run_kernels(nx, ny, nz, fields, nsteps, step0=0, dx=None, dy=None, dz=None,
                    dt=None, c=1.0, source=None, phases=7):
    """Reference range kernels in the Standard order (see ref_driver.cpp)."""
    dx = np.ones(nx, np.float32) if dx is None else np.ascontiguousarray(dx, np.float32)
    dy = np.ones(ny, np.float32) if dy is None else np.ascontiguousarray(dy, np.float32)
    dz = np.ones(nz, np.float32) if dz is None else np.ascontiguousarray(dz, np.float32)
    if dt is None:
        dt = ref_stable_dt(nx, ny, nz, dx, dy, dz, c, 0.99)
    if source is None:
        sc, si, sj, sk, tab, n = 2, 0, 0, 0, None, 0
    else:
        sc, si, sj, sk, tab, n = source.comp, source.i, source.j, source.k, _p(source.table), len(source.table)
    rc = ref().yr_run_kernels(nx, ny, nz, _p(dx), _p(dy), _p(dz), np.float32(dt), c,
                              _fptrs(fields), step0, nsteps, sc, si, sj, sk, tab, n, phases)
    if rc:
        raise RuntimeError(ref().yr_last_error().decode())
    return fields


def ref_stable_dt(nx, ny, nz, dx, dy, dz, c, safety):
    d = ref().yr_stable_dt(nx, ny, nz, _p(dx), _p(dy), _p(dz), c, safety)
    if d < 0:
        raise ValueError(ref().yr_last_error().decode())
    return np.float32(d)


def ref_coefficients(nx, ny, nz, dx, dy, dz, dt, c=1.0):
    out = [np.empty(n, np.float32) for n in (nx, ny, nz)]
    dx, dy, dz = (np.ascontiguousarray(a, np.float32) for a in (dx, dy, dz))
    if ref().yr_build_coefficients(nx, ny, nz, _p(dx), _p(dy), _p(dz), np.float32(dt), c,
                                   *[_p(a) for a in out]):
        raise ValueError(ref().yr_last_error().decode())
    return out


VARIANTS = {"standard": 0, "tiled": 1, "interleaved": 2, "planewise": 3, "twostep": 4}


def ref_simulation(nx, ny, nz, fields, nsteps, variant="standard", split=(1, 1, 1), workers=1,
                   quiescent_skip=False, source=None, step0=0, h=1.0, c=1.0, safety=0.99):
    """yeeblock::Simulation<float>::run. source = (comp, i, j, k, amp, sigma, t0, active_steps).
    Returns (seconds, digest); fields updated in place."""
    secs = C.c_double(0)
    dig = C.c_uint64(0)
    if source is None:
        hs, s = 0, (2, 0, 0, 0, 0.0, 1.0, 4.0, 0)
    else:
        hs, s = 1, source
    rc = ref().yr_simulation(nx, ny, nz, h, c, safety, VARIANTS[variant], *split, workers,
                             int(quiescent_skip), hs, s[0], s[1], s[2], s[3], s[4], s[5], s[6],
                             s[7], _fptrs(fields), step0, nsteps, C.byref(secs), C.byref(dig))
    if rc:
        raise RuntimeError(ref().yr_last_error().decode())
    return secs.value, int(dig.value)


def ref_source_table(nx, ny, nz, comp, i, j, k, amp, sigma, t0, active_steps, dt, n):
    out = np.zeros(n, np.float32)
    m = ref().yr_source_table(nx, ny, nz, comp, i, j, k, amp, sigma, t0, active_steps, dt, n, _p(out))
    if m < 0:
        raise ValueError(ref().yr_last_error().decode())
    return out[:m]


def ref_digest(nx, ny, nz, fields):
    return int(ref().yr_digest(nx, ny, nz, _fptrs(fields)))


def max_rel_err(a, b):
    """Per-component max |a-b| / max|b| (north_star tolerance metric)."""
    out = []
    for x, y in zip(a, b):
        m = float(np.max(np.abs(y))) if y.size else 0.0
        d = float(np.max(np.abs(x.astype(np.float64) - y.astype(np.float64)))) if y.size else 0.0
        out.append(d / m if m > 0 else d)
    return out


def total_energy(nx, ny, nz, fields, prev_h, dx=None, dy=None, dz=None):
    """Leapfrog invariant (fields.hpp:116-146, dual_spacing :86-93, dof_volume
    :96-105) in float64: sum_E V*E^2 + sum_H V*Hprev*Hnow. numpy summation
    order (the reference's is a serial loop): compare with a relative tolerance."""
    def weights(d, n):
        d = np.ones(n) if d is None else np.asarray(d, np.float64)
        node = np.empty(n + 1)
        node[0], node[n] = 0.5 * d[0], 0.5 * d[n - 1]
        node[1:n] = 0.5 * (d[:-1] + d[1:])
        return node, d
    W = [weights(dx, nx), weights(dy, ny), weights(dz, nz)]
    total = 0.0
    for c in range(6):
        axis = c % 3
        node = [(a != axis) if c < 3 else (a == axis) for a in range(3)]
        wx, wy, wz = (W[a][0 if node[a] else 1] for a in range(3))
        v = wz[:, None, None] * wy[None, :, None] * wx[None, None, :]
        now = fields[c].astype(np.float64)
        other = now if c < 3 else prev_h[c - 3].astype(np.float64)
        total += float(np.sum(v * other * now))
    return total


def ref_total_energy(nx, ny, nz, fields, prev_h, dx=None, dy=None, dz=None):
    ax = [np.ascontiguousarray(np.ones(n) if d is None else d, np.float32)
          for d, n in ((dx, nx), (dy, ny), (dz, nz))]
    ph = (_f32p * 3)(*[_p(a) for a in prev_h])
    return float(ref().yr_total_energy(nx, ny, nz, *[_p(a) for a in ax], _fptrs(fields), ph))


def ref_run_case(size, steps, source_steps=50, sigma_dt=8.0, amplitude=1.0, probe_stride=20,
                 quiescent_skip=True):
    """The reference bench harness's run_case (bench.hpp:105-127): (checksum hex, probe text)."""
    chk = C.create_string_buffer(17)
    buf = C.create_string_buffer(1 << 20)
    n = ref().yr_run_case(size, steps, source_steps, sigma_dt, amplitude, probe_stride, int(quiescent_skip),
                          chk, buf, len(buf))
    if n < 0:
        raise RuntimeError(ref().yr_last_error().decode())
    return chk.value.decode(), buf.value.decode()
