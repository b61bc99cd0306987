"""CPU ORACLE for the z-slab decomposition (test infrastructure only).

A numpy restatement of the Standard step (kernels.hpp:27-63 operand order,
PEC staggering.hpp:70-86, sources source.hpp:61-68, order schedule.hpp:171-210)
on ONE z-slab with `depth` ghost planes on each side, exposing the same halo
protocol as the CUDA Simulation (halo_bytes / halo_pack / halo_unpack / run;
include/yeeb200.h): after an exchange it may advance up to `depth` steps, each
step updating a plane range that shrinks by one ghost plane per step (the
ghost-zone scheme the two-step kernel uses). The gloo tests run the real
HaloExchange across processes and compare the assembled result with the
single-domain C oracle bit for bit.

Local arrays: every component on the node box with `depth` ghost planes below
and above and one pad cell around x/y: shape (nz + 2*depth + 1, ny+3, nx+3),
index [k + depth, j+1, i+1].
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from oracle import pyoracle as O


class OracleSlab:
    def __init__(self, nx, ny, nz_global, z_offset, nz, medium=None, sources=(), depth=1):
        self.nx, self.ny, self.nzg, self.zoff, self.nz, self.d = nx, ny, nz_global, z_offset, nz, depth
        self.at_bot, self.at_top = z_offset == 0, z_offset + nz == nz_global
        P = nz + 2 * depth + 1
        self.f = [np.zeros((P, ny + 3, nx + 3), np.float32) for _ in range(6)]
        S = O.courant()
        k = np.clip(np.arange(-depth, nz + depth + 1) + z_offset, 0, nz_global - 1)
        j = np.clip(np.arange(-1, ny + 2), 0, ny - 1)
        i = np.clip(np.arange(-1, nx + 2), 0, nx - 1)
        if medium is None:
            self.ca = self.da = np.float32(1.0)
            self.cb = self.db = np.float32(S)
        else:
            cells = O.cell_coeffs(nx, ny, nz_global, *medium)
            pick = np.ix_(k, j, i)
            self.ca, self.cb, self.da, self.db = (a[pick] for a in cells)
        self.sources = list(sources)  # (comp, i, j, k_global, table)
        self.step_index = 0
        self.since_exchange = 0

    # -------- state in/out (global dense arrays, planes of this slab)
    def load_global(self, fields):
        d = self.d
        for c in range(6):
            e0, e1, e2 = O.comp_extents(self.nx, self.ny, self.nzg, c)
            k0, k1 = self.zoff, min(self.zoff + self.nz + 1, e2)
            self.f[c][d + k0 - self.zoff:d + k1 - self.zoff, 1:1 + e1, 1:1 + e0] = fields[c][k0:k1]

    def owned(self, c):
        """(global k range, local array) this slab owns for component c."""
        e0, e1, e2 = O.comp_extents(self.nx, self.ny, self.nzg, c)
        n = self.nz + (1 if c in (0, 1, 5) and self.at_top else 0)
        return (self.zoff, self.zoff + n), self.f[c][self.d:self.d + n, 1:1 + e1, 1:1 + e0]

    # -------- halo protocol (same plane lists as yb_halo_*, own buffer layout)
    def _planes(self, side, pack):
        d, nz = self.d, self.nz
        if (side == 0) == pack:  # down-data: planes 0..d-1 (sender) / nz..nz+d-1 (receiver)
            base = 0 if pack else nz
            return [(c, base + q) for q in range(d) for c in range(6)]
        base = nz - d if pack else -d  # up-data: plane base hx, hy; base+1..base+d-1 all
        return [(3, base), (4, base)] + [(c, base + q) for q in range(1, d) for c in range(6)]

    def halo_bytes(self, side, receive):
        return len(self._planes(side, not receive)) * (self.ny + 3) * (self.nx + 3) * 4

    def halo_pack(self, side, ptr):
        f = getattr(self, "_pack_from", None) or self.f
        buf = np.ascontiguousarray(np.stack([f[c][self.d + k] for c, k in self._planes(side, True)]))
        C.memmove(ptr, buf.ctypes.data, buf.nbytes)

    def halo_unpack(self, side, ptr):
        pl = self._planes(side, False)
        buf = np.empty((len(pl), self.ny + 3, self.nx + 3), np.float32)
        C.memmove(buf.ctypes.data, ptr, buf.nbytes)
        for q, (c, k) in enumerate(pl):
            self.f[c][self.d + k] = buf[q]
        self.since_exchange = 0

    # -------- split sweeps (yb_advance_begin / yb_advance_end semantics):
    # begin computes the n steps into a pending copy that halo_pack reads;
    # end commits it.
    def advance_begin(self, nsteps):
        saved = [a.copy() for a in self.f]
        step0, since = self.step_index, self.since_exchange
        self.run(nsteps)
        self.pending = [a.copy() for a in self.f]
        self.pending_state = (self.step_index, self.since_exchange)
        self.f = saved
        self.step_index, self.since_exchange = step0, since
        self._pack_from = self.pending

    def advance_end(self):
        self.f = self.pending
        self.step_index, self.since_exchange = self.pending_state
        self.pending = self._pack_from = None

    # -------- steps
    def run(self, nsteps, sync=True):
        for _ in range(nsteps):
            self.since_exchange += 1
            alone = self.at_bot and self.at_top
            assert alone or self.since_exchange <= self.d, "ghost planes exhausted: exchange first"
            g = max(self.d - self.since_exchange, 0)  # ghost planes still valid after this step
            lo = 0 if self.at_bot else -g
            self._step(lo, self.nz + (0 if self.at_top else g))

    def _step(self, lo, hi):
        """E on local planes [lo, hi], H on [lo, hi-1] (+ hz on plane nz at the global top)."""
        nx, ny, d = self.nx, self.ny, self.d
        ex, ey, ez, hx, hy, hz = self.f

        def v(a, k0, k1, dk=0, dj=0, di=0):  # local planes k0..k1-1, j 0..ny, i 0..nx
            return a[d + k0 + dk:d + k1 + dk, 1 + dj:ny + 2 + dj, 1 + di:nx + 2 + di]

        def cf(a, k0, k1):
            return a if np.ndim(a) == 0 else a[d + k0:d + k1, 1:ny + 2, 1:nx + 2]

        def grid(k0, k1):
            K = np.arange(k0, k1)[:, None, None] + self.zoff
            J = np.arange(0, ny + 1)[None, :, None]
            I = np.arange(0, nx + 1)[None, None, :]
            return K, J, I

        k0, k1 = lo, hi + 1
        K, J, I = grid(k0, k1)
        kin = (K >= 1) & (K < self.nzg)
        ca, cb = cf(self.ca, k0, k1), cf(self.cb, k0, k1)
        new = [
            np.where((I < nx) & (J >= 1) & (J < ny) & kin,
                     ca * v(ex, k0, k1) + (cb * (v(hz, k0, k1) - v(hz, k0, k1, dj=-1))
                                           - cb * (v(hy, k0, k1) - v(hy, k0, k1, dk=-1))), 0),
            np.where((I >= 1) & (I < nx) & (J < ny) & kin,
                     ca * v(ey, k0, k1) + (cb * (v(hx, k0, k1) - v(hx, k0, k1, dk=-1))
                                           - cb * (v(hz, k0, k1) - v(hz, k0, k1, di=-1))), 0),
            np.where((I >= 1) & (I < nx) & (J >= 1) & (J < ny) & (K >= 0) & (K < self.nzg),
                     ca * v(ez, k0, k1) + (cb * (v(hy, k0, k1) - v(hy, k0, k1, di=-1))
                                           - cb * (v(hx, k0, k1) - v(hx, k0, k1, dj=-1))), 0),
        ]
        for c in range(3):
            v(self.f[c], k0, k1)[...] = new[c].astype(np.float32)
        for (sc, si, sj, sk, tab) in self.sources:
            kl = sk - self.zoff
            if k0 <= kl < k1 and self.step_index < len(tab):
                self.f[sc][d + kl, 1 + sj, 1 + si] += np.float32(tab[self.step_index])
        # Faraday: hx, hy on [lo, hi-1]; hz on [lo, hi-1] (+ plane nz at the global top)
        K, J, I = grid(k0, hi)
        da, db = cf(self.da, k0, hi), cf(self.db, k0, hi)
        kzl = K < self.nzg
        hxn = np.where((J < ny) & kzl, da * v(hx, k0, hi) + (db * (v(ey, k0, hi, dk=1) - v(ey, k0, hi))
                                                             - db * (v(ez, k0, hi, dj=1) - v(ez, k0, hi))), 0)
        hyn = np.where((I < nx) & kzl, da * v(hy, k0, hi) + (db * (v(ez, k0, hi, di=1) - v(ez, k0, hi))
                                                             - db * (v(ex, k0, hi, dk=1) - v(ex, k0, hi))), 0)
        hz_hi = hi + 1 if self.at_top else hi
        K2, J2, I2 = grid(k0, hz_hi)
        da2, db2 = cf(self.da, k0, hz_hi), cf(self.db, k0, hz_hi)
        hzn = np.where((I2 < nx) & (J2 < ny), da2 * v(hz, k0, hz_hi)
                       + (db2 * (v(ex, k0, hz_hi, dj=1) - v(ex, k0, hz_hi))
                          - db2 * (v(ey, k0, hz_hi, di=1) - v(ey, k0, hz_hi))), 0)
        v(hx, k0, hi)[...] = hxn.astype(np.float32)
        v(hy, k0, hi)[...] = hyn.astype(np.float32)
        v(hz, k0, hz_hi)[...] = hzn.astype(np.float32)
        self.step_index += 1
