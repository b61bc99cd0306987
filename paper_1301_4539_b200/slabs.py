"""z-slab domain decomposition across ranks (one GPU per rank, §8(e)).

The grid is split along z into contiguous cell slabs [K_r, K_{r+1})
(partition). Each step needs, per interface, one plane of H going up
(hx, hy of the slab's last plane -> the slab above's ghost plane -1, read by
its first E update, kernels.hpp:18-19 `k-1`) and one plane of state going
down (ex, ey, hx, hy, hz of the slab's first plane -> the slab below's ghost
plane nz, from which it recomputes E^{n+1} on that plane for its last H
update, kernels.hpp:23-24 `k+1`). This is the paper's "2 fields per face"
exchange plus the three fields the recompute reads.
Decomposition changes no arithmetic: results are bit-identical to one domain.

HaloExchange is transport-agnostic: it moves the planes with
torch.distributed point-to-point ops (NCCL between GPUs, gloo on CPU in the
tests). `sim` is anything with halo_bytes/halo_pack/halo_unpack (the CUDA
Simulation, or the CPU slab oracle in tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def partition(nz_global: int, world: int):
    """[(z_offset, nz_local)] per rank: contiguous, near-equal cell slabs."""
    if world < 1 or nz_global < world:
        raise ValueError(f"cannot split {nz_global} planes over {world} ranks")
    bounds = [r * nz_global // world for r in range(world + 1)]
    return [(bounds[r], bounds[r + 1] - bounds[r]) for r in range(world)]


class HaloExchange:
    """Per-step ghost-plane refresh between neighbouring slabs."""

    def __init__(self, sim, rank: int, world: int, device, group=None):
        self.sim, self.group = sim, group
        self.below = rank - 1 if rank > 0 else None
        self.above = rank + 1 if rank < world - 1 else None
        self.device = torch.device(device)
        self.buf = {}
        for side, peer in ((0, self.below), (1, self.above)):
            if peer is None:
                continue
            self.buf[side] = (
                torch.empty(sim.halo_bytes(side, False), dtype=torch.uint8, device=self.device),
                torch.empty(sim.halo_bytes(side, True), dtype=torch.uint8, device=self.device))
        self.bytes_per_exchange = sum(s.numel() for s, _ in self.buf.values())
        self._works = []

    def exchange(self):
        self.start()
        self.finish()

    def start(self):
        """Pack this slab's boundary planes and post the sends / receives."""
        for side, (send, _) in self.buf.items():
            self.sim.halo_pack(side, send.data_ptr())
        ops = []
        for side, (send, recv) in self.buf.items():
            peer = self.below if side == 0 else self.above
            ops.append(dist.P2POp(dist.isend, send, peer, self.group))
            ops.append(dist.P2POp(dist.irecv, recv, peer, self.group))
        self._works = dist.batch_isend_irecv(ops) if ops else []

    def finish(self):
        """Complete the transfers and write the received ghost planes."""
        if self._works:
            # NCCL: wait() makes the current torch stream wait for the
            # transfer. When the sim works on that stream (set_stream), pack ->
            # send/recv -> unpack -> the next sweep are all stream-ordered and
            # the host never blocks; otherwise synchronise before unpacking.
            for w in self._works:
                w.wait()
            if self.device.type == "cuda" and not self._stream_ordered():
                torch.cuda.synchronize(self.device)
        self._works = []
        for side, (_, recv) in self.buf.items():
            self.sim.halo_unpack(side, recv.data_ptr())

    def _stream_ordered(self):
        ptr = getattr(self.sim, "stream_ptr", 0)
        return bool(ptr) and ptr == torch.cuda.current_stream(self.device).cuda_stream


def run_steps(sim, exchanger: HaloExchange, nsteps: int, depth: int = 1, overlap: bool = False):
    """Advance nsteps, refreshing the ghost planes every `depth` steps (the
    sim's halo depth: 1 for one-step sweeps, 2 for two-step sweeps).

    overlap: split each sweep (advance_begin / advance_end): the boundary
    planes are computed first, their exchange is posted, and it runs while
    the interior planes are computed; the ghosts it delivers serve the next
    sweep. Bit-identical to the plain schedule."""
    if not overlap:
        done = 0
        while done < nsteps:
            n = min(depth, nsteps - done)
            exchanger.exchange()
            sim.run(n, sync=False)
            done += n
        return
    exchanger.exchange()  # ghosts of the current state
    done = 0
    while done < nsteps:
        n = min(depth, nsteps - done)
        sim.advance_begin(n)
        exchanger.start()
        sim.advance_end()
        exchanger.finish()
        done += n


class PeerExchange:
    """Direct halo push over peer memory (NVLink P2P, CUDA IPC): each rank
    exports IPC handles of its state buffers, all ranks gather them once
    (torch.distributed object collective), and each slab opens its two
    neighbours'. Afterwards no collective runs: yb_peer_step's sweep stores
    the boundary planes straight into the neighbours' ghost planes and orders
    the exchange through their flag words (run_steps_peer). Setup is
    collective: if any rank cannot export or map, every rank raises."""

    def __init__(self, sim, rank: int, world: int, group=None):
        self.sim = sim
        # every step is collective, so a failure on one rank raises on all of
        # them (callers may then fall back to HaloExchange together)
        why = ""
        try:
            mine = (sim.peer_export(), sim.nz)
        except Exception as e:  # noqa: BLE001
            mine, why = None, f"{type(e).__name__}: {e}"
        info = [None] * world
        dist.all_gather_object(info, mine, group=group)
        if not why:
            try:
                if rank > 0:
                    if info[rank - 1] is None:
                        raise RuntimeError("lower neighbour could not export its memory")
                    sim.peer_open(0, *info[rank - 1])
                if rank < world - 1:
                    if info[rank + 1] is None:
                        raise RuntimeError("upper neighbour could not export its memory")
                    sim.peer_open(1, *info[rank + 1])
            except Exception as e:  # noqa: BLE001
                why = f"{type(e).__name__}: {e}"
        whys = [None] * world
        dist.all_gather_object(whys, why, group=group)
        bad = [(r, w) for r, w in enumerate(whys) if w]
        if bad:
            raise RuntimeError(f"peer-memory exchange unavailable on rank {bad[0][0]}: {bad[0][1]}")


def run_steps_peer(sim, nsteps: int, depth: int, chained: bool = True):
    """run_steps for PeerExchange / peer_link'ed slabs: push the current
    boundary planes once, then (chained, two-step kernel) ALL the run's
    exchange periods in one persistent launch per rank (yb_peer_run: per sweep
    the boundary items wait in-kernel for the neighbours' previous sweep, store
    their boundary planes into the neighbours' ghost planes and signal); a
    trailing odd step, the one-step kernel and chained=False use one
    yb_peer_step per period instead (compute, exchange and ordering in one
    launch each). Every rank must make the same calls: chained launches of
    neighbouring ranks wait on each other, so they need the ranks on
    different GPUs (or, on one GPU, yb_peer_run over all slabs at once)."""
    sim.peer_push(False)
    done = 0
    if chained and depth == 2 and nsteps >= 2:
        n = nsteps // 2 * 2
        sim.peer_run(n)
        done = n
    while done < nsteps:
        n = min(depth, nsteps - done)
        sim.peer_step(n)
        done += n


def owned_planes(comp: int, nz_local: int, at_top: bool) -> int:
    """Planes of component `comp`'s dense slab array this rank owns: node-z
    components (ex, ey, hz) have nz_local+1 planes; the last belongs to the
    slab above unless this is the global top."""
    node_z = comp in (0, 1, 5)
    return nz_local + (1 if node_z and at_top else 0)
