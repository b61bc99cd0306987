"""CPU ORACLE for the z-slab decomposition (test infrastructure only).

A numpy restatement of one Standard step (kernels.hpp:27-63 operand order,
PEC staggering.hpp:70-86, sources source.hpp:61-68, order schedule.hpp:171-210)
on ONE z-slab with ghost planes, exposing the same halo interface as the CUDA
Simulation (halo_bytes / halo_pack / halo_unpack / run). It lets the gloo
tests run the real HaloExchange protocol across processes and compare the
assembled result with the single-domain C oracle bit for bit.

Local arrays: every component on the node box with one ghost plane below and
one pad cell around x/y: shape (nz+2, ny+3, nx+3), index [k+1, j+1, i+1].
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from oracle import pyoracle as O

HALO_DOWN = (0, 1, 3, 4, 5)  # ex, ey, hx, hy, hz of plane 0 -> slab below's ghost plane nz
HALO_UP = (3, 4)             # hx, hy of plane nz-1 -> slab above's ghost plane -1


class OracleSlab:
    def __init__(self, nx, ny, nz_global, z_offset, nz, medium=None, sources=()):
        self.nx, self.ny, self.nzg, self.zoff, self.nz = nx, ny, nz_global, z_offset, nz
        self.at_bot, self.at_top = z_offset == 0, z_offset + nz == nz_global
        self.f = [np.zeros((nz + 2, ny + 3, nx + 3), np.float32) for _ in range(6)]
        S = O.courant()
        cells = None
        if medium is not None:
            cells = O.cell_coeffs(nx, ny, nz_global, *medium)
        # per-position coefficients on the local node box (cell clamped, global z)
        k = np.clip(np.arange(-1, nz + 1) + z_offset, 0, nz_global - 1)
        j = np.clip(np.arange(-1, ny + 2), 0, ny - 1)
        i = np.clip(np.arange(-1, nx + 2), 0, nx - 1)
        if cells is None:
            self.ca = self.da = np.float32(1.0)
            self.cb = self.db = None
        else:
            pick = np.ix_(k, j, i)
            self.ca, self.cb, self.da, self.db = (a[pick] for a in cells)
        self.S = S
        self.sources = list(sources)  # (comp, i, j, k_global, table)
        self.step_index = 0

    # -------- state in/out (global dense arrays, planes of this slab)
    def load_global(self, fields):
        for c in range(6):
            e0, e1, e2 = O.comp_extents(self.nx, self.ny, self.nzg, c)
            k0, k1 = self.zoff, min(self.zoff + self.nz + 1, e2)
            self.f[c][1 + (k0 - self.zoff):1 + (k1 - self.zoff), 1:1 + e1, 1:1 + e0] = fields[c][k0:k1]

    def owned(self, c):
        """(global k range, local array) this slab owns for component c."""
        e0, e1, e2 = O.comp_extents(self.nx, self.ny, self.nzg, c)
        node_z = c in (0, 1, 5)
        n = self.nz + (1 if node_z and self.at_top else 0)
        return (self.zoff, self.zoff + n), self.f[c][1:1 + n, 1:1 + e1, 1:1 + e0]

    # -------- halo interface (same semantics as yb_halo_*)
    def _plane_bytes(self):
        return (self.ny + 3) * (self.nx + 3) * 4

    def halo_bytes(self, side, receive):
        n = len(HALO_DOWN) if (side == 0) != bool(receive) else len(HALO_UP)
        return n * self._plane_bytes()

    def halo_pack(self, side, ptr):
        planes = [self.f[c][1] for c in HALO_DOWN] if side == 0 else \
                 [self.f[c][self.nz] for c in HALO_UP]
        buf = np.ascontiguousarray(np.stack(planes))
        C.memmove(ptr, buf.ctypes.data, buf.nbytes)

    def halo_unpack(self, side, ptr):
        comps, plane = (HALO_UP, 0) if side == 0 else (HALO_DOWN, self.nz + 1)
        n = len(comps)
        buf = np.empty((n, self.ny + 3, self.nx + 3), np.float32)
        C.memmove(buf.ctypes.data, ptr, buf.nbytes)
        for q, c in enumerate(comps):
            self.f[c][plane] = buf[q]

    # -------- one Standard step on the slab
    def run(self, nsteps, sync=True):
        for _ in range(nsteps):
            self._step()

    def _step(self):
        nx, ny, nz, S = self.nx, self.ny, self.nz, self.S
        ex, ey, ez, hx, hy, hz = self.f
        K = np.arange(0, nz + 1)[:, None, None] + self.zoff  # global plane of local 0..nz
        J = np.arange(0, ny + 1)[None, :, None]
        I = np.arange(0, nx + 1)[None, None, :]

        def v(a, dk=0, dj=0, di=0, k_hi=nz + 1):  # local k in [0, k_hi), j in [0,ny], i in [0,nx]
            return a[1 + dk:1 + k_hi + dk, 1 + dj:ny + 2 + dj, 1 + di:nx + 2 + di]

        def coef(a, k_hi=nz + 1):
            return a if np.isscalar(a) or a.ndim == 0 else a[1:1 + k_hi, 1:ny + 2, 1:nx + 2]

        ca = coef(self.ca)
        cb1 = coef(self.cb) if self.cb is not None else np.float32(S)
        kin = (K >= 1) & (K < self.nzg)
        # Ampere + PEC on planes 0..nz (plane nz below the global top = the recompute)
        e_new = [None] * 3
        m = (I < nx) & (J >= 1) & (J < ny) & kin
        e_new[0] = np.where(m, ca * v(ex) + (cb1 * (v(hz) - v(hz, dj=-1)) - cb1 * (v(hy) - v(hy, dk=-1))), 0)
        m = (I >= 1) & (I < nx) & (J < ny) & kin
        e_new[1] = np.where(m, ca * v(ey) + (cb1 * (v(hx) - v(hx, dk=-1)) - cb1 * (v(hz) - v(hz, di=-1))), 0)
        m = (I >= 1) & (I < nx) & (J >= 1) & (J < ny) & (K < self.nzg)
        e_new[2] = np.where(m, ca * v(ez) + (cb1 * (v(hy) - v(hy, di=-1)) - cb1 * (v(hx) - v(hx, dj=-1))), 0)
        for c in range(3):
            e_new[c] = e_new[c].astype(np.float32)
            v(self.f[c])[...] = e_new[c]
        for (sc, si, sj, sk, tab) in self.sources:
            kl = sk - self.zoff
            if 0 <= kl <= nz and self.step_index < len(tab):
                self.f[sc][1 + kl, 1 + sj, 1 + si] += np.float32(tab[self.step_index])
        # Faraday on planes 0..nz-1 (hz also on plane nz at the global top)
        da = coef(self.da, nz)
        db1 = coef(self.db, nz) if self.db is not None else np.float32(S)
        Kh = K[:nz]
        m = (J < ny) & (Kh < self.nzg)
        hx_n = np.where(m, da * v(hx, k_hi=nz) + (db1 * (v(ey, dk=1, k_hi=nz) - v(ey, k_hi=nz))
                                                   - db1 * (v(ez, dj=1, k_hi=nz) - v(ez, k_hi=nz))), 0)
        m = (I < nx) & (Kh < self.nzg)
        hy_n = np.where(m, da * v(hy, k_hi=nz) + (db1 * (v(ez, di=1, k_hi=nz) - v(ez, k_hi=nz))
                                                   - db1 * (v(ex, dk=1, k_hi=nz) - v(ex, k_hi=nz))), 0)
        nzh = nz + 1 if self.at_top else nz
        da2 = coef(self.da, nzh)
        db2 = coef(self.db, nzh) if self.db is not None else np.float32(S)
        m = (I < nx) & (J < ny)
        hz_n = np.where(m, da2 * v(hz, k_hi=nzh) + (db2 * (v(ex, dj=1, k_hi=nzh) - v(ex, k_hi=nzh))
                                                     - db2 * (v(ey, di=1, k_hi=nzh) - v(ey, k_hi=nzh))), 0)
        v(hx, k_hi=nz)[...] = hx_n.astype(np.float32)
        v(hy, k_hi=nz)[...] = hy_n.astype(np.float32)
        v(hz, k_hi=nzh)[...] = hz_n.astype(np.float32)
        self.step_index += 1
