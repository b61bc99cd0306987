"""paper_1301_4539_b200 — B200-native Yee FDTD leapfrog step (arXiv 1301.4539 hot path).

Python front end over the C-ABI library ``libyeeb200.so`` (include/yeeb200.h),
used by the tests and bench.py. The reference-facing drop-in for C++ callers is
``include/yeeb200/yeeblock.hpp``; this module mirrors the same surface:
``Simulation(nx, ny, nz)`` owns device-resident padded SoA state,
``run(n)`` advances ``step_index`` (runner.hpp:243-266), fields cross the
boundary in the reference's dense Array3 layout (array3.hpp:104-107).

There is no CPU fallback: if the CUDA library is missing or no GPU is present
every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# YB_LIB: an alternative build of the same library (A/B of kernel variants)
LIB_PATH = os.environ.get("YB_LIB") or os.path.join(HERE, "libyeeb200.so")
CSRC = os.path.join(HERE, "csrc")

EX, EY, EZ, HX, HY, HZ = range(6)
COMP_NAMES = ("ex", "ey", "ez", "hx", "hy", "hz")
CA, CB, DA, DB = range(4)
ABI_VERSION = 5  # YB_ABI_VERSION of include/yeeb200.h
VARIANT_TB2, VARIANT_NAIVE, VARIANT_FUSED, VARIANT_TB4 = 0, 1, 2, 3  # YB_VARIANT_* (TB2 = 0: the default)
S_BITS = 0x3F1252DB
S = np.array([S_BITS], dtype=np.uint32).view(np.float32)[0]  # (float)(0.99/sqrt(3))

# C-ABI exported symbols (include/yeeb200.h) — checked by tests.
ABI_SYMBOLS = (
    "yb_last_error", "yb_abi_version", "yb_create", "yb_destroy", "yb_set_axis_coeffs",
    "yb_set_cell_coeffs", "yb_set_cell_coeffs_n", "yb_generate_medium", "yb_upload_field", "yb_download_field",
    "yb_upload_fields", "yb_download_fields", "yb_zero_fields", "yb_fill_fields", "yb_set_step_index", "yb_get_step_index",
    "yb_add_source", "yb_clear_sources", "yb_advance", "yb_synchronize", "yb_advance_timed",
    "yb_apply_ampere_range", "yb_apply_faraday_range", "yb_apply_pec_boundary",
    "yb_field_digest", "yb_set_stream", "yb_set_kernel_timing", "yb_get_info",
    "yb_host_medium", "yb_host_field", "yb_halo_bytes", "yb_halo_pack", "yb_halo_unpack",
    "yb_host_field_slab", "yb_host_medium_slab", "yb_set_probes", "yb_read_probes",
    "yb_snapshot_h", "yb_total_energy", "yb_set_quiescent_skip", "yb_advance_begin", "yb_advance_end",
    "yb_peer_handle_bytes", "yb_peer_export", "yb_peer_open", "yb_peer_link", "yb_peer_push", "yb_peer_wait", "yb_peer_step",
    "yb_peer_run", "yb_run_to_host", "yb_run_streamed",
    "yb_fs_apply", "yb_fs_total_energy",
)


class YeeError(RuntimeError):
    pass


class YeeInvalidArgument(YeeError, ValueError):
    pass


class YeeOutOfRange(YeeError, IndexError):
    pass


class _Desc(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("device", C.c_int),
                ("variant", C.c_int), ("zchunk", C.c_int), ("z_offset", C.c_int),
                ("nz_global", C.c_int), ("reserved", C.c_int * 4)]


class Info(C.Structure):
    _fields_ = [("step_index", C.c_int64), ("steps", C.c_int64), ("kernel_launches", C.c_int64),
                ("main_kernel_ms", C.c_double), ("main_kernel_timed", C.c_int64),
                ("n_cell_arrays", C.c_int), ("variant", C.c_int), ("stages", C.c_int),
                ("grid_x", C.c_int), ("grid_y", C.c_int), ("grid_z", C.c_int), ("zchunk", C.c_int),
                ("bytes_per_cell_update", C.c_double), ("device_bytes", C.c_size_t),
                ("halo_depth", C.c_int), ("quiescent_skip", C.c_int), ("skipped_items", C.c_int64),
                ("streamed_readbacks", C.c_int64), ("streamed_uploads", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_f32p = C.POINTER(C.c_float)
_lib = None


def build(verbose=False):
    """Compile libyeeb200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    r = subprocess.run(["make", "-C", CSRC, "-j3"], capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise YeeError("libyeeb200 build failed:\n" + (r.stdout or "") + (r.stderr or ""))


def lib():
    """Load libyeeb200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise YeeError(f"{LIB_PATH} missing: run paper_1301_4539_b200.build()")
        L = C.CDLL(LIB_PATH)
        L.yb_last_error.restype = C.c_char_p
        vp = C.c_void_p
        L.yb_create.argtypes = [C.POINTER(_Desc), C.POINTER(vp)]
        L.yb_destroy.argtypes = [vp]
        L.yb_set_axis_coeffs.argtypes = [vp, _f32p, _f32p, _f32p]
        L.yb_set_cell_coeffs.argtypes = [vp, C.c_int, _f32p, C.c_float]
        L.yb_set_cell_coeffs_n.argtypes = [vp, C.c_int, C.POINTER(C.c_int), C.POINTER(vp)]
        L.yb_generate_medium.argtypes = [vp, C.c_int64, C.c_int64]
        L.yb_upload_field.argtypes = [vp, C.c_int, _f32p]
        L.yb_upload_fields.argtypes = [vp, C.POINTER(vp)]
        L.yb_download_fields.argtypes = [vp, C.POINTER(vp)]
        L.yb_download_field.argtypes = [vp, C.c_int, _f32p]
        L.yb_run_to_host.argtypes = [vp, C.c_int64, C.POINTER(vp)]
        L.yb_run_streamed.argtypes = [vp, C.c_int64, C.c_int, C.POINTER(C.c_int), C.POINTER(vp), C.POINTER(vp),
                                      C.POINTER(vp)]
        L.yb_zero_fields.argtypes = [vp]
        L.yb_fill_fields.argtypes = [vp, C.c_uint64]
        L.yb_set_step_index.argtypes = [vp, C.c_int64]
        L.yb_get_step_index.argtypes = [vp, C.POINTER(C.c_int64)]
        L.yb_add_source.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, _f32p, C.c_int64]
        L.yb_clear_sources.argtypes = [vp]
        L.yb_advance.argtypes = [vp, C.c_int64]
        L.yb_synchronize.argtypes = [vp]
        L.yb_advance_timed.argtypes = [vp, C.c_int64, C.POINTER(C.c_float)]
        L.yb_apply_ampere_range.argtypes = [vp, C.POINTER(C.c_int)]
        L.yb_apply_faraday_range.argtypes = [vp, C.POINTER(C.c_int)]
        L.yb_apply_pec_boundary.argtypes = [vp]
        L.yb_field_digest.argtypes = [vp, C.POINTER(C.c_uint64)]
        L.yb_set_stream.argtypes = [vp, vp]
        L.yb_set_kernel_timing.argtypes = [vp, C.c_int]
        L.yb_get_info.argtypes = [vp, C.POINTER(Info)]
        L.yb_host_medium.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                     _f32p, _f32p, _f32p, _f32p]
        L.yb_host_field.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, _f32p]
        L.yb_host_field_slab.argtypes = [C.c_int] * 5 + [C.c_uint64, C.c_int, _f32p]
        L.yb_host_medium_slab.argtypes = [C.c_int] * 5 + [C.c_int64, C.c_int64] + [_f32p] * 4
        L.yb_set_probes.argtypes = [vp, C.c_int] + [C.POINTER(C.c_int)] * 5
        L.yb_read_probes.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int), _f32p, C.c_int64,
                                     C.POINTER(C.c_int64)]
        L.yb_snapshot_h.argtypes = [vp]
        L.yb_set_quiescent_skip.argtypes = [vp, C.c_int]
        L.yb_advance_begin.argtypes = [vp, C.c_int64]
        L.yb_advance_end.argtypes = [vp]
        L.yb_peer_handle_bytes.restype = C.c_size_t
        L.yb_peer_export.argtypes = [vp, vp]
        L.yb_peer_open.argtypes = [vp, C.c_int, vp, C.c_int]
        L.yb_peer_link.argtypes = [vp, C.c_int, vp]
        L.yb_peer_push.argtypes = [vp, C.c_int]
        L.yb_peer_wait.argtypes = [vp]
        L.yb_peer_step.argtypes = [vp, C.c_int64]
        L.yb_peer_run.argtypes = [C.POINTER(vp), C.c_int, C.c_int64]
        L.yb_total_energy.argtypes = [vp] + [C.POINTER(C.c_double)] * 4
        L.yb_halo_bytes.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_size_t)]
        L.yb_halo_pack.argtypes = [vp, C.c_int, vp]
        L.yb_halo_unpack.argtypes = [vp, C.c_int, vp]
        L.yb_fs_apply.argtypes = [C.c_int] * 5 + [C.POINTER(vp), C.POINTER(vp), C.c_int, C.c_int,
                                                   C.POINTER(C.c_int)]
        L.yb_fs_total_energy.argtypes = [C.c_int] * 5 + [C.POINTER(vp)] * 2 + [C.POINTER(C.c_double)] * 4
        if L.yb_abi_version() != ABI_VERSION:
            raise YeeError(f"{LIB_PATH}: ABI {L.yb_abi_version()}, this module needs {ABI_VERSION} (rebuild)")
        _lib = L
    return _lib


def _check(rc):
    if rc == 0:
        return
    msg = lib().yb_last_error().decode()
    if rc == 1:
        raise YeeInvalidArgument(msg)
    if rc == 2:
        raise YeeOutOfRange(msg)
    raise YeeError(f"status {rc}: {msg}")


def comp_extents(nx, ny, nz, comp):
    """(ex, ey, ez) extents of one component (staggering.hpp:34-39)."""
    n = (nx, ny, nz)
    axis = comp % 3
    electric = comp < 3
    return tuple(n[a] + (1 if (electric and a != axis) or (not electric and a == axis) else 0)
                 for a in range(3))


def _fp(a):
    return a.ctypes.data_as(_f32p)


def _f32c(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Simulation:
    """Device-resident Yee state + Standard-step driver (runner.hpp:205-266 mirror).

    Coefficients default to the reference unit grid: cdx = cdy = cdz = S
    (make_uniform_grid<float>(n, 1, 1, 0.99) + build_coefficients).
    """

    def __init__(self, nx, ny, nz, device=0, variant=VARIANT_TB2, zchunk=0, cdx=None, cdy=None,
                 cdz=None, z_offset=0, nz_global=0):
        """nz_global > 0: this handle is the z-slab [z_offset, z_offset+nz) of a grid with
        nz_global cell planes (halo exchange: halo_pack / halo_unpack, see slabs.py)."""
        self.nx, self.ny, self.nz = nx, ny, nz
        self.z_offset, self.nz_global = z_offset, (nz_global or nz)
        h = C.c_void_p()
        d = _Desc(nx, ny, nz, device, variant, zchunk, z_offset, nz_global)
        _check(lib().yb_create(C.byref(d), C.byref(h)))
        self._h = h
        self.stream_ptr = 0
        self.set_axis_coeffs(np.full(nx, S, np.float32) if cdx is None else cdx,
                             np.full(ny, S, np.float32) if cdy is None else cdy,
                             np.full(self.nz_global, S, np.float32) if cdz is None else cdz)

    def close(self):
        if getattr(self, "_h", None):
            lib().yb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # coefficients ---------------------------------------------------------
    def set_axis_coeffs(self, cdx, cdy, cdz):
        cdx, cdy, cdz = _f32c(cdx), _f32c(cdy), _f32c(cdz)
        assert cdx.size == self.nx and cdy.size == self.ny and cdz.size == self.nz_global
        _check(lib().yb_set_axis_coeffs(self._h, _fp(cdx), _fp(cdy), _fp(cdz)))

    def set_cell_coeffs(self, which, cells=None, uniform=1.0):
        if cells is None:
            _check(lib().yb_set_cell_coeffs(self._h, which, None, uniform))
        else:
            cells = _f32c(cells)
            slab = self.nz_global != self.nz  # z-slab: nz + 4 cell planes from z_offset - 2
            assert cells.size == self.nx * self.ny * (self.nz + (4 if slab else 0))
            _check(lib().yb_set_cell_coeffs(self._h, which, _fp(cells), uniform))

    def set_cell_coeffs_many(self, arrays):
        """{which: cells} for several coefficient arrays in one call
        (yb_set_cell_coeffs_n: the copies run back to back)."""
        slab = self.nz_global != self.nz
        items = [(w, _f32c(a)) for w, a in arrays.items()]
        for _, a in items:
            assert a.size == self.nx * self.ny * (self.nz + (4 if slab else 0))
        which = (C.c_int * len(items))(*[w for w, _ in items])
        ptrs = (C.c_void_p * len(items))(*[a.ctypes.data for _, a in items])
        _check(lib().yb_set_cell_coeffs_n(self._h, len(items), which, ptrs))

    def generate_medium(self, eps_seed=-1, sigma_seed=-1):
        _check(lib().yb_generate_medium(self._h, eps_seed, sigma_seed))

    # fields -----------------------------------------------------------------
    def upload(self, fields):
        arrs = []
        for c in range(6):
            a = _f32c(fields[c])
            assert a.shape == comp_extents(self.nx, self.ny, self.nz, c)[::-1], (c, a.shape)
            arrs.append(a)
        ptrs = (C.c_void_p * 6)(*[a.ctypes.data for a in arrs])  # arrs keeps the buffers alive
        _check(lib().yb_upload_fields(self._h, ptrs))

    def download(self, out=None):
        """Dense host copies of the six components (into `out` if given, e.g.
        pinned buffers; fresh arrays otherwise)."""
        res = []
        for c in range(6):
            shape = comp_extents(self.nx, self.ny, self.nz, c)[::-1]
            a = np.empty(shape, np.float32) if out is None else out[c]
            assert a.shape == shape and a.dtype == np.float32 and a.flags.c_contiguous
            res.append(a)
        ptrs = (C.c_void_p * 6)(*[a.ctypes.data for a in res])
        _check(lib().yb_download_fields(self._h, ptrs))
        return res

    def run_to_host(self, nsteps, out=None):
        """run(nsteps) then download(out) in one call (yb_run_to_host): with
        page-locked `out` buffers the device->host copies of each tile row
        start as soon as it finished its last sweep, overlapping the rest of
        the run. Returns the six dense arrays."""
        res = []
        for c in range(6):
            shape = comp_extents(self.nx, self.ny, self.nz, c)[::-1]
            a = np.empty(shape, np.float32) if out is None else out[c]
            assert a.shape == shape and a.dtype == np.float32 and a.flags.c_contiguous
            res.append(a)
        ptrs = (C.c_void_p * 6)(*[a.ctypes.data for a in res])
        _check(lib().yb_run_to_host(self._h, nsteps, ptrs))
        return res

    def run_streamed(self, nsteps, cell_arrays=None, fields=None, out=None):
        """run_simulation's host flow in one call (yb_run_streamed): upload the
        per-cell coefficient arrays {which: cells} and (if given) the six
        initial fields, advance nsteps, read all six components back. With
        page-locked buffers both transfers overlap the run (tile row by tile
        row); otherwise the phases run one after the other. Returns the six
        dense arrays."""
        items = [(w, _f32c(a)) for w, a in (cell_arrays or {}).items()]
        for _, a in items:
            assert a.size == self.nx * self.ny * self.nz
        which = (C.c_int * max(1, len(items)))(*[w for w, _ in items])
        cptr = (C.c_void_p * max(1, len(items)))(*[a.ctypes.data for _, a in items])
        fin = None
        if fields is not None:
            arrs = []
            for c in range(6):
                a = _f32c(fields[c])
                assert a.shape == comp_extents(self.nx, self.ny, self.nz, c)[::-1], (c, a.shape)
                arrs.append(a)
            fin = (C.c_void_p * 6)(*[a.ctypes.data for a in arrs])
        res = []
        for c in range(6):
            shape = comp_extents(self.nx, self.ny, self.nz, c)[::-1]
            a = np.empty(shape, np.float32) if out is None else out[c]
            assert a.shape == shape and a.dtype == np.float32 and a.flags.c_contiguous
            res.append(a)
        optr = (C.c_void_p * 6)(*[a.ctypes.data for a in res])
        _check(lib().yb_run_streamed(self._h, nsteps, len(items), which, cptr, fin, optr))
        return res

    def zero(self):
        _check(lib().yb_zero_fields(self._h))

    def fill(self, seed):
        _check(lib().yb_fill_fields(self._h, seed))

    @property
    def step_index(self):
        v = C.c_int64()
        _check(lib().yb_get_step_index(self._h, C.byref(v)))
        return v.value

    @step_index.setter
    def step_index(self, v):
        _check(lib().yb_set_step_index(self._h, v))

    # sources / stepping ----------------------------------------------------
    def add_source(self, comp, i, j, k, table):
        t = _f32c(table)
        _check(lib().yb_add_source(self._h, comp, i, j, k, _fp(t) if t.size else None, t.size))

    def clear_sources(self):
        _check(lib().yb_clear_sources(self._h))

    def run(self, nsteps, sync=True):
        _check(lib().yb_advance(self._h, nsteps))
        if sync:
            self.synchronize()

    def advance_begin(self, nsteps):
        """Split sweep, part 1: the slab's boundary planes (halo_pack then
        reads the new planes); enqueued only."""
        _check(lib().yb_advance_begin(self._h, nsteps))

    def advance_end(self):
        """Split sweep, part 2: the interior planes; completes the steps."""
        _check(lib().yb_advance_end(self._h))

    # direct halo push over peer memory (see yb_peer_* in include/yeeb200.h)
    def peer_export(self):
        buf = C.create_string_buffer(lib().yb_peer_handle_bytes())
        _check(lib().yb_peer_export(self._h, buf))
        return buf.raw

    def peer_open(self, side, handles, peer_nz):
        buf = C.create_string_buffer(bytes(handles), len(handles))
        _check(lib().yb_peer_open(self._h, side, buf, peer_nz))

    def peer_link(self, side, other):
        _check(lib().yb_peer_link(self._h, side, other._h))

    def peer_push(self, overlap=False):
        _check(lib().yb_peer_push(self._h, 1 if overlap else 0))

    def peer_wait(self):
        _check(lib().yb_peer_wait(self._h))

    def peer_step(self, nsteps):
        """One exchange period over peer memory (the two-step sweep stores its
        boundary planes straight into the neighbours' ghost planes)."""
        _check(lib().yb_peer_step(self._h, nsteps))

    def peer_run(self, nsteps):
        """nsteps (even) / 2 exchange periods of this slab in ONE persistent launch
        (chained periods; the neighbours make the same call on their GPUs)."""
        peer_run([self], nsteps)

    def run_timed(self, nsteps):
        ms = C.c_float()
        _check(lib().yb_advance_timed(self._h, nsteps, C.byref(ms)))
        return ms.value

    def synchronize(self):
        _check(lib().yb_synchronize(self._h))

    def apply_ampere_range(self, box=None):
        b = None if box is None else (C.c_int * 6)(*box)
        _check(lib().yb_apply_ampere_range(self._h, b))

    def apply_faraday_range(self, box=None):
        b = None if box is None else (C.c_int * 6)(*box)
        _check(lib().yb_apply_faraday_range(self._h, b))

    def apply_pec_boundary(self):
        _check(lib().yb_apply_pec_boundary(self._h))

    def digest(self):
        v = C.c_uint64()
        _check(lib().yb_field_digest(self._h, C.byref(v)))
        return v.value

    def set_stream(self, stream_ptr):
        """Work on a caller stream (e.g. torch.cuda.current_stream().cuda_stream);
        0 / None restores the handle's own stream."""
        _check(lib().yb_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))
        self.stream_ptr = stream_ptr or 0

    # z-slab halo planes (device pointers, e.g. torch CUDA tensor .data_ptr())
    def halo_bytes(self, side, receive):
        v = C.c_size_t()
        _check(lib().yb_halo_bytes(self._h, side, 1 if receive else 0, C.byref(v)))
        return v.value

    def halo_pack(self, side, dst_ptr):
        _check(lib().yb_halo_pack(self._h, side, C.c_void_p(dst_ptr)))

    def halo_unpack(self, side, src_ptr):
        _check(lib().yb_halo_unpack(self._h, side, C.c_void_p(src_ptr)))

    def set_probes(self, probes):
        """probes: [(comp, i, j, k, stride)] sampled on the device after every
        completed step t with t % stride == 0 (probe.hpp:14-51)."""
        n = len(probes)
        cols = [np.ascontiguousarray([p[q] for p in probes], dtype=np.int32) for q in range(5)]
        ptr = [c.ctypes.data_as(C.POINTER(C.c_int)) for c in cols]
        _check(lib().yb_set_probes(self._h, n, *ptr))

    def read_probes(self, capacity=1 << 20):
        """Drains recorded samples: (steps int64, probe int32, values float32)."""
        st = np.empty(capacity, np.int64)
        pr = np.empty(capacity, np.int32)
        va = np.empty(capacity, np.float32)
        n = C.c_int64()
        _check(lib().yb_read_probes(self._h, st.ctypes.data_as(C.POINTER(C.c_int64)),
                                    pr.ctypes.data_as(C.POINTER(C.c_int)), _fp(va), capacity, C.byref(n)))
        k = n.value
        return st[:k].copy(), pr[:k].copy(), va[:k].copy()

    def set_quiescent_skip(self, on=True):
        """Skip work items whose input box is all +0 (runner.hpp:60-73);
        results are unchanged. info()['skipped_items'] counts them."""
        _check(lib().yb_set_quiescent_skip(self._h, 1 if on else 0))

    def snapshot_h(self):
        """HSnapshot of the current H on the device (fields.hpp:71-82)."""
        _check(lib().yb_snapshot_h(self._h))

    def total_energy(self, dx=None, dy=None, dz=None):
        """Leapfrog invariant against the last snapshot (fields.hpp:116-146);
        spacings default to 1 (dz has nz_global entries)."""
        arrs = [None if d is None else np.ascontiguousarray(d, np.float64) for d in (dx, dy, dz)]
        ptr = [None if a is None else a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs]
        out = C.c_double()
        _check(lib().yb_total_energy(self._h, *ptr, C.byref(out)))
        return out.value

    def set_kernel_timing(self, on):
        _check(lib().yb_set_kernel_timing(self._h, 1 if on else 0))

    def info(self):
        i = Info()
        _check(lib().yb_get_info(self._h, C.byref(i)))
        return i.as_dict()


OP_UPDATE_E, OP_UPDATE_H, OP_ZERO, OP_AMPERE, OP_FARADAY, OP_PEC = range(6)


def peer_run(sims, nsteps):
    """yb_peer_run: chained exchange periods of 1..8 linked slabs. Several slabs of one
    device (yb_peer_link) run in ONE launch — the one-GPU emulation of that many ranks."""
    hs = (C.c_void_p * len(sims))(*[s._h for s in sims])
    _check(lib().yb_peer_run(hs, len(sims), nsteps))


def fs_apply(fields, cd, op, comp=0, box=None, device=0):
    """A per-box operation on a host FieldSet (six dense float32 or float64
    arrays, updated in place): the reference's free functions
    update_e_box / update_h_box / zero_box / apply_ampere_range /
    apply_faraday_range / apply_pec_boundary (kernels.hpp:78-155) run on the
    device. cd = (cdx, cdy, cdz) in the same dtype."""
    dt = fields[0].dtype
    assert dt in (np.float32, np.float64) and all(a.dtype == dt and a.flags.c_contiguous for a in fields)
    nz, ny, nx = fields[0].shape[0] - 1, fields[0].shape[1] - 1, fields[0].shape[2]  # ex: nx x (ny+1) x (nz+1)
    cds = [np.ascontiguousarray(a, dt) for a in cd] if cd is not None else None
    f6 = (C.c_void_p * 6)(*[a.ctypes.data for a in fields])
    c3 = (C.c_void_p * 3)(*[a.ctypes.data for a in cds]) if cds is not None else None
    b = (C.c_int * 6)(*box) if box is not None else None
    _check(lib().yb_fs_apply(device, 0 if dt == np.float32 else 1, nx, ny, nz, f6, c3, op, comp, b))
    return fields


def fs_total_energy(fields, prev_h, dx=None, dy=None, dz=None, device=0):
    """total_energy (fields.hpp:116-146) of a host FieldSet and an H snapshot, on the device."""
    dt = fields[0].dtype
    nz, ny, nx = fields[0].shape[0] - 1, fields[0].shape[1] - 1, fields[0].shape[2]
    f6 = (C.c_void_p * 6)(*[a.ctypes.data for a in fields])
    p3 = (C.c_void_p * 3)(*[a.ctypes.data for a in prev_h])
    ds = [None if d is None else np.ascontiguousarray(d, np.float64) for d in (dx, dy, dz)]
    ptr = [None if d is None else d.ctypes.data_as(C.POINTER(C.c_double)) for d in ds]
    out = C.c_double()
    _check(lib().yb_fs_total_energy(device, 0 if dt == np.float32 else 1, nx, ny, nz, f6, p3, *ptr,
                                    C.byref(out)))
    return out.value


def host_medium(nx, ny, nz, eps_seed, sigma_seed, out=None):
    """Pinned seeded medium on the host: (ca, cb, da, db) dense (nz, ny, nx) arrays."""
    out = out or [np.empty((nz, ny, nx), np.float32) for _ in range(4)]
    _check(lib().yb_host_medium(nx, ny, nz, eps_seed, sigma_seed,
                                *[None if a is None else _fp(a) for a in out]))
    return out


def host_fields(nx, ny, nz, seed, out=None):
    """Pinned seeded fields on the host (dense reference layout)."""
    out = out or [np.empty(comp_extents(nx, ny, nz, c)[::-1], np.float32) for c in range(6)]
    for c in range(6):
        _check(lib().yb_host_field(nx, ny, nz, seed, c, _fp(out[c])))
    return out


def host_fields_slab(nx, ny, nz_global, z_offset, nz_local, seed, out=None):
    """Seeded fields of one z-slab (dense local layout: node-z components carry
    nz_local+1 planes, the same planes a slab Simulation uploads)."""
    res = []
    for c in range(6):
        e = comp_extents(nx, ny, nz_local, c)
        a = np.empty(e[::-1], np.float32) if out is None else out[c]
        _check(lib().yb_host_field_slab(nx, ny, nz_global, z_offset, e[2], seed, c, _fp(a)))
        res.append(a)
    return res


def host_medium_slab(nx, ny, nz_global, z_offset, nplanes, eps_seed, sigma_seed, out):
    """Seeded medium for cell planes [z_offset, z_offset+nplanes) into out=(ca, cb, da, db)
    (None entries skipped)."""
    _check(lib().yb_host_medium_slab(nx, ny, nz_global, z_offset, nplanes, eps_seed, sigma_seed,
                                     *[None if a is None else _fp(a) for a in out]))
    return out


def run_simulation(nx, ny, nz, fields, nsteps, step0=0, sources=(), medium=None, cells=None,
                   variant=VARIANT_TB2, device=0):
    """run_simulation (runner.hpp:349-362) mirror: copy the host state in, advance, copy out.

    medium=(eps_seed, sigma_seed) generates the pinned medium on the device;
    cells={CA: arr, ...} uploads per-cell coefficient arrays instead.
    Returns the new host state (list of six dense arrays)."""
    with Simulation(nx, ny, nz, device=device, variant=variant) as sim:
        if medium is not None:
            sim.generate_medium(*medium)
        for w, a in (cells or {}).items():
            sim.set_cell_coeffs(w, a)
        for s in sources:
            sim.add_source(*s)
        sim.upload(fields)
        sim.step_index = step0
        sim.run(nsteps)
        return sim.download()
