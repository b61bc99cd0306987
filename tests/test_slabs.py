"""z-slab decomposition (§8(e)). CPU: the slab semantics (ghost planes,
recomputed top plane, global PEC) on the numpy slab oracle, and the
HaloExchange protocol across 2 processes over gloo, both bit-exact against
the single-domain C oracle. GPU: slabs of the CUDA path in one process on one
GPU, exchanging through device buffers, bit-exact against one domain."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1301_4539_b200.slabs import HaloExchange, partition


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint32), np.ascontiguousarray(b).view(np.uint32))


def test_partition():
    assert partition(10, 3) == [(0, 3), (3, 3), (6, 4)]
    assert partition(8, 8) == [(r, 1) for r in range(8)]
    with pytest.raises(ValueError):
        partition(3, 4)


TB2, FUSED = 0, 2  # include/yeeb200.h YB_VARIANT_* (ABI 3)
CASE = dict(nx=13, ny=11, nzg=17, steps=9, medium=(7, 7), fseed=8)


def reference_run(oracle, nx, ny, nzg, steps, medium, fseed, src=None):
    f = oracle.fill_fields(nx, ny, nzg, fseed)
    ca, cb, da, db = oracle.cell_coeffs(nx, ny, nzg, *medium)
    co = oracle.Coeffs(nx, ny, nzg, ca=ca, cb=cb, da=da, db=db)
    oracle.run(nx, ny, nzg, f, co, steps, sources=[oracle.Source(*src)] if src else None)
    return f


def assemble(oracle, nx, ny, nzg, slabs):
    out = oracle.zeros_state(nx, ny, nzg)
    for s in slabs:
        for c in range(6):
            (k0, k1), a = s.owned(c)
            out[c][k0:k1] = a
    return out


class DirectExchange:
    """In-process stand-in for HaloExchange (same pack/unpack protocol)."""

    def __init__(self, slabs):
        self.slabs = slabs

    def exchange(self):
        for lo, hi in zip(self.slabs[:-1], self.slabs[1:]):
            up = np.empty(lo.halo_bytes(1, False), np.uint8)
            down = np.empty(hi.halo_bytes(0, False), np.uint8)
            lo.halo_pack(1, up.ctypes.data)
            hi.halo_pack(0, down.ctypes.data)
            hi.halo_unpack(0, up.ctypes.data)
            lo.halo_unpack(1, down.ctypes.data)


def advance(exchange, slabs, steps, depth):
    done = 0
    while done < steps:
        n = min(depth, steps - done)
        exchange()
        for s in slabs:
            s.run(n)
        done += n


@pytest.mark.parametrize("depth", [1, 2])
@pytest.mark.parametrize("nranks", [1, 2, 3, 5])
def test_slab_oracle_matches_single_domain(oracle, nranks, depth):
    """Ghost-zone slabs: halo depth 1 (exchange every step) and 2 (every two
    steps, the two-step kernel's protocol)."""
    from oracle.slab_oracle import OracleSlab
    nx, ny, nzg, steps = CASE["nx"], CASE["ny"], CASE["nzg"], CASE["steps"]
    tab = oracle.gauss_table(steps)
    src = (2, 6, 5, 8, tab)
    f0 = oracle.fill_fields(nx, ny, nzg, CASE["fseed"])
    slabs = [OracleSlab(nx, ny, nzg, z0, n, medium=CASE["medium"], sources=[src], depth=depth)
             for z0, n in partition(nzg, nranks)]
    for s in slabs:
        s.load_global(f0)
    advance(DirectExchange(slabs).exchange, slabs, steps, depth)
    got = assemble(oracle, nx, ny, nzg, slabs)
    want = reference_run(oracle, nx, ny, nzg, steps, CASE["medium"], CASE["fseed"], src)
    for c in range(6):
        assert bits_equal(got[c], want[c]), c


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, result_path, depth, overlap=False):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import pyoracle as O
    from oracle.slab_oracle import OracleSlab
    from paper_1301_4539_b200.slabs import HaloExchange, partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nzg, steps = CASE["nx"], CASE["ny"], CASE["nzg"], CASE["steps"]
    z0, n = partition(nzg, world)[rank]
    tab = O.gauss_table(steps)
    slab = OracleSlab(nx, ny, nzg, z0, n, medium=CASE["medium"], sources=[(2, 6, 5, 8, tab)],
                      depth=depth)
    slab.load_global(O.fill_fields(nx, ny, nzg, CASE["fseed"]))
    hx = HaloExchange(slab, rank, world, "cpu")
    from paper_1301_4539_b200.slabs import run_steps
    run_steps(slab, hx, steps, depth, overlap=overlap)
    parts = [None] * world
    dist.all_gather_object(parts, [(slab.owned(c)[0], slab.owned(c)[1].copy()) for c in range(6)])
    if rank == 0:
        out = O.zeros_state(nx, ny, nzg)
        for p in parts:
            for c, ((k0, k1), a) in enumerate(p):
                out[c][k0:k1] = a
        np.savez(result_path, *out)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,depth,overlap", [(2, 1, False), (3, 1, False), (2, 2, False), (3, 2, False),
                                                 (2, 1, True), (3, 2, True)])
def test_gloo_halo_exchange_bit_exact(oracle, tmp_path, world, depth, overlap):
    """HaloExchange over torch.distributed (gloo, world_size 2/3, 127.0.0.1),
    halo depth 1 and 2; overlap: split sweeps with the exchange posted
    between the boundary and the interior part (run_steps(overlap=True))."""
    path = str(tmp_path / "res.npz")
    mp.spawn(_gloo_worker, args=(world, _free_port(), path, depth, overlap), nprocs=world, join=True)
    got = np.load(path)
    want = reference_run(oracle, CASE["nx"], CASE["ny"], CASE["nzg"], CASE["steps"], CASE["medium"],
                         CASE["fseed"], (2, 6, 5, 8, oracle.gauss_table(CASE["steps"])))
    for c in range(6):
        assert bits_equal(got[f"arr_{c}"], want[c]), c


class _DeviceExchange:
    """Single-GPU stand-in for HaloExchange between CUDA slabs (stream-ordered
    device copies between launches; no kernel waits on another)."""

    def __init__(self, sims):
        self.sims = sims
        self.bufs = []
        for lo, hi in zip(sims[:-1], sims[1:]):
            self.bufs.append((torch.empty(lo.halo_bytes(1, False), dtype=torch.uint8, device="cuda"),
                              torch.empty(hi.halo_bytes(0, False), dtype=torch.uint8, device="cuda")))

    def exchange(self):
        for (lo, hi), (up, down) in zip(zip(self.sims[:-1], self.sims[1:]), self.bufs):
            lo.halo_pack(1, up.data_ptr())
            hi.halo_pack(0, down.data_ptr())
            hi.halo_unpack(0, up.data_ptr())
            lo.halo_unpack(1, down.data_ptr())


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [FUSED, TB2])
@pytest.mark.parametrize("nranks,medium,fseed,src,upload", [(2, (7, 7), 8, True, False),
                                                            (3, (4, -1), None, True, False),
                                                            (4, (-1, -1), 5, False, False),
                                                            (3, (7, 7), 8, True, True)])
def test_gpu_slabs_bit_exact(yb, oracle, nranks, medium, fseed, src, variant, upload):
    """CUDA slabs (one-step fused, halo depth 1; two-step tb2, depth 2) in one
    process on one GPU, bit-exact against a single domain. upload: per-cell
    coefficients come from host arrays (slab layout: nz+4 cell planes)."""
    nx, ny, nzg, steps = 136, 40, 29, 11
    tab = oracle.gauss_table(steps)
    srcs = [(2, nx // 2, ny // 2, nzg // 2, tab)] if src else []
    sims = []
    for z0, n in partition(nzg, nranks):
        s = yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, zchunk=4, variant=variant)
        if upload:
            arrs = yb.host_medium_slab(nx, ny, nzg, z0 - 2, n + 4, *medium,
                                       [np.empty((n + 4, ny, nx), np.float32) for _ in range(4)])
            for q in range(4):
                s.set_cell_coeffs(q, arrs[q])
        else:
            s.generate_medium(*medium)
        for q in srcs:
            s.add_source(*q)
        if fseed is not None:
            s.fill(fseed)
        sims.append(s)
    ex = _DeviceExchange(sims)
    depth = sims[0].info()["halo_depth"]
    assert depth == (2 if variant == yb.VARIANT_TB2 else 1)
    done = 0
    while done < steps:
        n = min(depth, steps - done)
        ex.exchange()
        for s in sims:
            s.run(n)
        done += n
    out = oracle.zeros_state(nx, ny, nzg)
    for s in sims:
        d = s.download()
        at_top = s.z_offset + s.nz == nzg
        for c in range(6):
            node_z = c in (0, 1, 5)
            n = s.nz + (1 if node_z and at_top else 0)
            out[c][s.z_offset:s.z_offset + n] = d[c][:n]
    with yb.Simulation(nx, ny, nzg) as one:
        one.generate_medium(*medium)
        for q in srcs:
            one.add_source(*q)
        if fseed is not None:
            one.fill(fseed)
        one.run(steps)
        want = one.download()
    for c in range(6):
        assert bits_equal(out[c], want[c]), c
    for s in sims:
        s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [FUSED, TB2])
def test_gpu_slabs_stream_ordered(yb, oracle, variant):
    """Slabs on a shared caller stream: halo pack/unpack are stream-ordered
    (no host synchronisation between sweeps and exchanges) — same result."""
    nx, ny, nzg, steps = 136, 40, 29, 11
    tab = oracle.gauss_table(steps)
    srcs = [(2, nx // 2, ny // 2, nzg // 2, tab)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        sims = []
        for z0, n in partition(nzg, 3):
            s = yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, variant=variant)
            s.generate_medium(7, 7)
            for q in srcs:
                s.add_source(*q)
            s.fill(8)
            s.set_stream(st.cuda_stream)
            sims.append(s)
        ex = _DeviceExchange(sims)
        depth = sims[0].info()["halo_depth"]
        done = 0
        while done < steps:
            n = min(depth, steps - done)
            ex.exchange()
            for s in sims:
                s.run(n, sync=False)
            done += n
        st.synchronize()
    out = oracle.zeros_state(nx, ny, nzg)
    for s in sims:
        d = s.download()
        at_top = s.z_offset + s.nz == nzg
        for c in range(6):
            k = s.nz + (1 if c in (0, 1, 5) and at_top else 0)
            out[c][s.z_offset:s.z_offset + k] = d[c][:k]
        s.close()
    with yb.Simulation(nx, ny, nzg) as one:
        one.generate_medium(7, 7)
        for q in srcs:
            one.add_source(*q)
        one.fill(8)
        one.run(steps)
        want = one.download()
    for c in range(6):
        assert bits_equal(out[c], want[c]), c


class _DeviceExchangeSplit(_DeviceExchange):
    """start(): pack every slab (split sweeps: the new boundary planes) into
    the buffers; finish(): unpack — the in-process stand-in for posting NCCL
    transfers between advance_begin and advance_end."""

    def start(self):
        for (lo, hi), (up, down) in zip(zip(self.sims[:-1], self.sims[1:]), self.bufs):
            lo.halo_pack(1, up.data_ptr())
            hi.halo_pack(0, down.data_ptr())

    def finish(self):
        for (lo, hi), (up, down) in zip(zip(self.sims[:-1], self.sims[1:]), self.bufs):
            hi.halo_unpack(0, up.data_ptr())
            lo.halo_unpack(1, down.data_ptr())


@pytest.mark.gpu
@pytest.mark.parametrize("variant,nranks,nzg", [(FUSED, 3, 29), (TB2, 3, 29), (TB2, 2, 12), (TB2, 4, 23), (FUSED, 2, 5)])
def test_gpu_slabs_split_sweeps(yb, oracle, variant, nranks, nzg):
    """Split sweeps (yb_advance_begin / yb_advance_end: boundary planes first,
    exchange, interior) give the single-domain result bit for bit, including
    slabs too thin to have an interior."""
    nx, ny, steps = 136, 40, 11
    tab = oracle.gauss_table(steps)
    srcs = [(2, nx // 2, ny // 2, nzg // 2, tab)]
    sims = []
    for z0, n in partition(nzg, nranks):
        s = yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, variant=variant, zchunk=3)
        s.generate_medium(7, 7)
        for q in srcs:
            s.add_source(*q)
        s.fill(8)
        sims.append(s)
    ex = _DeviceExchangeSplit(sims)
    depth = sims[0].info()["halo_depth"]
    ex.exchange()
    done = 0
    while done < steps:
        n = min(depth, steps - done)
        for s in sims:
            s.advance_begin(n)
        ex.start()
        for s in sims:
            s.advance_end()
        ex.finish()
        done += n
    out = oracle.zeros_state(nx, ny, nzg)
    for s in sims:
        d = s.download()
        at_top = s.z_offset + s.nz == nzg
        for c in range(6):
            k = s.nz + (1 if c in (0, 1, 5) and at_top else 0)
            out[c][s.z_offset:s.z_offset + k] = d[c][:k]
        assert s.step_index == steps
        s.close()
    with yb.Simulation(nx, ny, nzg) as one:
        one.generate_medium(7, 7)
        for q in srcs:
            one.add_source(*q)
        one.fill(8)
        one.run(steps)
        want = one.download()
    for c in range(6):
        assert bits_equal(out[c], want[c]), c


@pytest.mark.gpu
def test_split_sweep_errors(yb):
    with yb.Simulation(40, 16, 10, z_offset=0, nz_global=20, variant=yb.VARIANT_FUSED) as s:
        with pytest.raises(yb.YeeInvalidArgument):
            s.advance_begin(2)  # the one-step kernel: depth 1
        with pytest.raises(yb.YeeInvalidArgument):
            s.advance_end()
        s.advance_begin(1)
        with pytest.raises(yb.YeeInvalidArgument):
            s.run(1)
        with pytest.raises(yb.YeeInvalidArgument):
            s.halo_unpack(0, 0)
        with pytest.raises(yb.YeeInvalidArgument):
            s.zero()
        with pytest.raises(yb.YeeInvalidArgument):
            s.download()
        s.advance_end()
        assert s.step_index == 1


@pytest.mark.gpu
@pytest.mark.parametrize("variant,nranks,nzg", [(TB2, 3, 29), (FUSED, 3, 29), (TB2, 2, 12), (TB2, 4, 23)])
def test_gpu_slabs_peer_push(yb, oracle, variant, nranks, nzg):
    """Direct peer-memory halo push (yb_peer_link within one process, one GPU):
    push / wait / split sweeps enqueued slab after slab on one stream, so every
    device-side wait is already satisfied when it runs (no kernel waits on a
    concurrent one). Bit-exact against one domain."""
    nx, ny, steps = 136, 40, 11
    tab = oracle.gauss_table(steps)
    srcs = [(2, nx // 2, ny // 2, nzg // 2, tab)]
    sims = []
    for z0, n in partition(nzg, nranks):
        s = yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, variant=variant, zchunk=3)
        s.generate_medium(7, 7)
        for q in srcs:
            s.add_source(*q)
        s.fill(8)
        sims.append(s)
    st = torch.cuda.Stream()
    for s in sims:
        s.set_stream(st.cuda_stream)
    for lo, hi in zip(sims[:-1], sims[1:]):
        lo.peer_link(1, hi)
        hi.peer_link(0, lo)
    depth = sims[0].info()["halo_depth"]
    for s in sims:
        s.peer_push(False)
    done = 0
    while done < steps:
        n = min(depth, steps - done)
        for s in sims:
            s.peer_wait()
            s.advance_begin(n)
        for s in sims:
            s.peer_push(False)
        for s in sims:
            s.advance_end()
        done += n
    out = oracle.zeros_state(nx, ny, nzg)
    for s in sims:
        s.synchronize()
        d = s.download()
        at_top = s.z_offset + s.nz == nzg
        for c in range(6):
            k = s.nz + (1 if c in (0, 1, 5) and at_top else 0)
            out[c][s.z_offset:s.z_offset + k] = d[c][:k]
    with yb.Simulation(nx, ny, nzg) as one:
        one.generate_medium(7, 7)
        for q in srcs:
            one.add_source(*q)
        one.fill(8)
        one.run(steps)
        want = one.download()
    for c in range(6):
        assert bits_equal(out[c], want[c]), c
    for s in sims:
        s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [FUSED, TB2])
def test_gpu_slabs_peer_quiescent_skip(yb, oracle, variant):
    """Peer-memory exchange with the quiescent skip on: the neighbours' stores
    into a slab's ghost planes must reach its quiescent map (yb_peer_wait
    rescans them), else a boundary item whose only nonzero input came from
    the neighbour is skipped and the wave never enters the slab. Zero fields
    and one point source in the bottom slab: every other slab starts all-zero
    and only the exchange can wake it. Bit-exact against one domain."""
    nx, ny, nzg, nranks, steps = 136, 40, 30, 3, 24
    tab = oracle.gauss_table(steps)
    src = (2, nx // 2, ny // 2, 6, tab)
    sims = []
    for z0, n in partition(nzg, nranks):
        s = yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, variant=variant, zchunk=3)
        s.generate_medium(7, -1)
        s.add_source(*src)
        s.set_quiescent_skip(True)
        sims.append(s)
    st = torch.cuda.Stream()
    for s in sims:
        s.set_stream(st.cuda_stream)
    for lo, hi in zip(sims[:-1], sims[1:]):
        lo.peer_link(1, hi)
        hi.peer_link(0, lo)
    depth = sims[0].info()["halo_depth"]
    for s in sims:
        s.peer_push(False)
    done = 0
    while done < steps:
        n = min(depth, steps - done)
        for s in sims:
            s.peer_wait()
            s.advance_begin(n)
        for s in sims:
            s.peer_push(False)
        for s in sims:
            s.advance_end()
        done += n
    out = oracle.zeros_state(nx, ny, nzg)
    for s in sims:
        s.synchronize()
        d = s.download()
        at_top = s.z_offset + s.nz == nzg
        for c in range(6):
            k = s.nz + (1 if c in (0, 1, 5) and at_top else 0)
            out[c][s.z_offset:s.z_offset + k] = d[c][:k]
    assert sims[0].info()["skipped_items"] > 0  # the skip was active
    for s in sims:
        s.close()
    with yb.Simulation(nx, ny, nzg) as one:
        one.generate_medium(7, -1)
        one.add_source(*src)
        one.run(steps)
        want = one.download()
    assert any(np.any(out[c][20:] != 0) for c in range(6))  # the wave reached the top slab
    for c in range(6):
        assert bits_equal(out[c], want[c]), c


@pytest.mark.gpu
def test_peer_errors(yb):
    with yb.Simulation(40, 16, 10) as one:
        with pytest.raises(yb.YeeInvalidArgument):
            one.peer_push()
    a = yb.Simulation(40, 16, 10, z_offset=0, nz_global=20)
    b = yb.Simulation(40, 16, 10, z_offset=10, nz_global=20)
    with pytest.raises(yb.YeeInvalidArgument):
        a.peer_link(0, b)  # nothing below the global bottom
    c = yb.Simulation(32, 16, 10, z_offset=10, nz_global=20)
    with pytest.raises(yb.YeeInvalidArgument):
        a.peer_link(1, c)  # x extents differ
    assert len(a.peer_export()) == yb.lib().yb_peer_handle_bytes()
    for s in (a, b, c):
        s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("fold", [True, False])
@pytest.mark.parametrize("variant,nranks,nzg,steps", [(TB2, 3, 29, 11), (TB2, 2, 12, 10), (TB2, 4, 23, 9), (FUSED, 3, 29, 7),
                                                       (2, 3, 150, 8)])
def test_gpu_slabs_peer_step(yb, oracle, monkeypatch, fold, variant, nranks, nzg, steps):
    """Exchange fused into the sweep (yb_peer_step): the two-step kernel stores
    its boundary planes straight into the linked neighbours' ghost planes, and
    (fold) its bottom / top z-chunk items wait for and signal the neighbours
    themselves. One process, one GPU, all slabs on one stream, stepped one after
    another (every device-side wait already satisfied when it runs). Bit-exact
    against one domain."""
    import torch
    if not fold:
        monkeypatch.setenv("YB_PEER_NOFOLD", "1")
    nx, ny = 136, 40
    tab = oracle.gauss_table(steps)
    srcs = [(2, nx // 2, ny // 2, nzg // 2, tab)]
    sims = []
    for z0, n in partition(nzg, nranks):
        s = yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, variant=variant)
        s.generate_medium(7, 7)
        for q in srcs:
            s.add_source(*q)
        s.fill(8)
        sims.append(s)
    st = torch.cuda.Stream()
    for s in sims:
        s.set_stream(st.cuda_stream)
    for lo, hi in zip(sims[:-1], sims[1:]):
        lo.peer_link(1, hi)
        hi.peer_link(0, lo)
    depth = sims[0].info()["halo_depth"]
    for s in sims:
        s.peer_push(False)
    done = 0
    while done < steps:
        n = min(depth, steps - done)
        for s in sims:
            s.peer_step(n)
        done += n
    out = oracle.zeros_state(nx, ny, nzg)
    for s in sims:
        s.synchronize()
        d = s.download()
        at_top = s.z_offset + s.nz == nzg
        for c in range(6):
            k = s.nz + (1 if c in (0, 1, 5) and at_top else 0)
            out[c][s.z_offset:s.z_offset + k] = d[c][:k]
    with yb.Simulation(nx, ny, nzg) as one:
        one.generate_medium(7, 7)
        for q in srcs:
            one.add_source(*q)
        one.fill(8)
        one.run(steps)
        want = one.download()
    for c in range(6):
        assert bits_equal(out[c], want[c]), c
    for s in sims:
        s.close()


@pytest.mark.gpu
@pytest.mark.parametrize("nranks,nzg,steps,medium,fseed,zchunk", [
    (2, 12, 10, (7, 7), 8, 0),       # thin slabs: one z-chunk each (bottom = top chunk)
    (3, 29, 16, (7, 7), 8, 0),
    (4, 23, 8, (4, -1), None, 0),    # zero start, point source, Cb only
    (3, 150, 12, (7, 7), 8, 0),      # multi-chunk slabs, interior chunks between the boundary ones
    (2, 61, 20, (-1, -1), 5, 7),     # vacuum, ragged chunks (31 = 4 x 7 + 3, 30 = 4 x 7 + 2)
    (4, 67, 14, (7, 7), 8, 4),       # more items than CTAs per sweep
])
def test_gpu_slabs_peer_run_chained(yb, oracle, nranks, nzg, steps, medium, fseed, zchunk):
    """Chained exchange periods (yb_peer_run, k_tb2 MODE 4): all slabs of the
    decomposition run in ONE persistent launch on the one GPU — the emulation
    of nranks ranks prescribed for fewer GPUs than ranks: every sweep's
    boundary items wait in-kernel for the neighbour slab's previous sweep,
    store their boundary planes into its ghost planes and signal, the sweeps
    follow each other through the device-side neighbourhood counts. Bit-exact
    against one domain (which itself matches the oracle, test_parity_gpu)."""
    nx, ny = 136, 40
    tab = oracle.gauss_table(steps + 4)
    srcs = [(2, nx // 2, ny // 2, nzg // 2, tab)] if fseed is None else []
    sims = []
    for z0, n in partition(nzg, nranks):
        s = yb.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, zchunk=zchunk, variant=TB2)
        s.generate_medium(*medium)
        for q in srcs:
            s.add_source(*q)
        if fseed is not None:
            s.fill(fseed)
        sims.append(s)
    for lo, hi in zip(sims[:-1], sims[1:]):
        lo.peer_link(1, hi)
        hi.peer_link(0, lo)
    for s in sims:
        s.peer_push(False)
    yb.peer_run(sims, steps // 2 * 2 - 2)  # one launch of several periods ...
    yb.peer_run(sims, 2)                   # ... and one more (state, counters, flags carried over)
    out = oracle.zeros_state(nx, ny, nzg)
    for s in sims:
        s.synchronize()
        assert s.step_index == steps // 2 * 2
        d = s.download()
        at_top = s.z_offset + s.nz == nzg
        for c in range(6):
            k = s.nz + (1 if c in (0, 1, 5) and at_top else 0)
            out[c][s.z_offset:s.z_offset + k] = d[c][:k]
    with yb.Simulation(nx, ny, nzg) as one:
        one.generate_medium(*medium)
        for q in srcs:
            one.add_source(*q)
        if fseed is not None:
            one.fill(fseed)
        one.run(steps // 2 * 2)
        want = one.download()
    for c in range(6):
        assert bits_equal(out[c], want[c]), c
    for s in sims:
        s.close()


@pytest.mark.gpu
def test_peer_run_errors(yb):
    with yb.Simulation(16, 8, 6, z_offset=0, nz_global=12) as a, \
            yb.Simulation(16, 8, 6, z_offset=6, nz_global=12) as b:
        with pytest.raises(yb.YeeError):
            yb.peer_run([a], 0)  # nothing to advance
        a.peer_link(1, b)
        b.peer_link(0, a)
        with pytest.raises(yb.YeeError):
            yb.peer_run([a, b], 3)  # odd step count
        with pytest.raises(yb.YeeError):
            yb.peer_run([a, a], 2)  # listed twice


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 3])
def test_gpu_peer_run_single_domain(yb, oracle, n):
    """yb_peer_run over unlinked single-domain handles: a chain of n independent
    domains in one launch (n = 1: the rank's direct-parameter MODE 4 kernel;
    n = 3: the parameter-array kernel of the emulation) equals yb_advance."""
    nx, ny, nz, steps = 136, 40, 37, 8
    sims = []
    for q in range(n):
        s = yb.Simulation(nx, ny, nz, variant=TB2)
        s.generate_medium(7, 7)
        s.fill(8 + q)
        sims.append(s)
    yb.peer_run(sims, steps)
    for q, s in enumerate(sims):
        got = s.download()
        with yb.Simulation(nx, ny, nz) as one:
            one.generate_medium(7, 7)
            one.fill(8 + q)
            one.run(steps)
            want = one.download()
        for c in range(6):
            assert bits_equal(got[c], want[c]), (q, c)
        s.close()


def _ipc_worker(rank, world, port, result_path, variant, steps):
    """One slab per process, all on cuda:0, linked through CUDA IPC
    (PeerExchange). Ranks take turns — each period rank r steps while the
    others idle, with a device sync and a gloo barrier between turns — so every
    device-side wait is already satisfied when it runs and no kernel waits on
    a concurrently running one."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1301_4539_b200 as Y
    from oracle import pyoracle as O
    from paper_1301_4539_b200.slabs import PeerExchange, partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    nx, ny, nzg = 136, 40, 37
    z0, n = partition(nzg, world)[rank]
    s = Y.Simulation(nx, ny, n, z_offset=z0, nz_global=nzg, variant=variant)
    s.generate_medium(7, 7)
    s.add_source(2, nx // 2, ny // 2, nzg // 2, O.gauss_table(steps))
    s.fill(8)
    PeerExchange(s, rank, world)
    depth = s.info()["halo_depth"]

    def turns(fn):
        for r in range(world):
            if r == rank:
                fn()
                s.synchronize()
            dist.barrier()

    turns(lambda: s.peer_push(False))
    done = 0
    while done < steps:
        k = min(depth, steps - done)
        turns(lambda: s.peer_step(k))
        done += k
    d = s.download()
    at_top = z0 + n == nzg
    mine = [(z0, d[c][:n + (1 if c in (0, 1, 5) and at_top else 0)].copy()) for c in range(6)]
    parts = [None] * world
    dist.all_gather_object(parts, mine)
    if rank == 0:
        out = O.zeros_state(nx, ny, nzg)
        for p in parts:
            for c, (k0, a) in enumerate(p):
                out[c][k0:k0 + a.shape[0]] = a
        np.savez(result_path, *out)
    dist.barrier()
    s.close()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("variant,world,steps", [(TB2, 2, 10), (TB2, 3, 9), (FUSED, 2, 5)])
def test_gpu_ipc_peer_exchange(yb, oracle, tmp_path, variant, world, steps):
    """The cross-process path of --exchange p2p: IPC handles exchanged over
    gloo, opened with cudaIpcOpenMemHandle, then yb_peer_step per period (the
    two-step sweep stores its boundary planes into the other process's ghost
    planes and signals its flag word). Bit-exact against one domain."""
    path = str(tmp_path / "ipc.npz")
    mp.spawn(_ipc_worker, args=(world, _free_port(), path, variant, steps), nprocs=world, join=True)
    got = np.load(path)
    nx, ny, nzg = 136, 40, 37
    with yb.Simulation(nx, ny, nzg) as one:
        one.generate_medium(7, 7)
        one.add_source(2, nx // 2, ny // 2, nzg // 2, oracle.gauss_table(steps))
        one.fill(8)
        one.run(steps)
        want = one.download()
    for c in range(6):
        assert bits_equal(got[f"arr_{c}"], want[c]), c


@pytest.mark.gpu
def test_gpu_peer_wait_times_out(yb):
    """A neighbour that never publishes: the sweep's in-kernel wait gives up
    (bounded, ~15 s) and the error surfaces at the next synchronize instead of
    hanging the device."""
    a = yb.Simulation(136, 16, 40, z_offset=0, nz_global=80, variant=yb.VARIANT_TB2)
    b = yb.Simulation(136, 16, 40, z_offset=40, nz_global=80, variant=yb.VARIANT_TB2)
    a.peer_link(1, b)
    b.peer_link(0, a)
    a.peer_push(False)
    a.peer_step(2)  # b never pushed: a's top-chunk items wait for b's flag
    with pytest.raises(yb.YeeError):
        a.synchronize()
    for s in (a, b):
        s.close()


class _FakePeerSim:
    """Host-side stand-in for PeerExchange's setup logic (no GPU): rank
    `fail_rank` cannot map its neighbours' memory."""

    def __init__(self, rank, fail_rank, fail_at):
        self.rank, self.fail_rank, self.fail_at, self.nz, self.opened = rank, fail_rank, fail_at, 5, []

    def peer_export(self):
        if self.rank == self.fail_rank and self.fail_at == "export":
            raise RuntimeError("cudaIpcGetMemHandle failed")
        return b"h%d" % self.rank

    def peer_open(self, side, handles, nz):
        if self.rank == self.fail_rank and self.fail_at == "open":
            raise RuntimeError("cudaIpcOpenMemHandle failed")
        self.opened.append((side, handles, nz))


def _peer_setup_worker(rank, world, port, fail_rank, fail_at, result_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1301_4539_b200.slabs import PeerExchange
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sim = _FakePeerSim(rank, fail_rank, fail_at)
    try:
        PeerExchange(sim, rank, world)
        out = "ok " + ",".join(f"{s}:{h.decode()}" for s, h, _ in sim.opened)
    except RuntimeError as e:
        out = "raised " + str(e)
    dist.barrier()  # every rank reached here: no collective was left unmatched
    with open(f"{result_path}.{rank}", "w") as f:
        f.write(out)
    dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank,fail_at", [(-1, None), (1, "open"), (0, "export"), (2, "open")])
def test_peer_exchange_setup_is_collective(tmp_path, fail_rank, fail_at):
    """PeerExchange over gloo (world 3, no GPU): handles reach the right
    neighbours; when one rank cannot export or map, every rank raises (so
    bench.py --exchange auto falls back to NCCL on all ranks together)."""
    world = 3
    path = str(tmp_path / "setup")
    mp.spawn(_peer_setup_worker, args=(world, _free_port(), fail_rank, fail_at, path), nprocs=world, join=True)
    outs = [open(f"{path}.{r}").read() for r in range(world)]
    if fail_rank < 0:
        assert outs == ["ok 1:h1", "ok 0:h0,1:h2", "ok 0:h1"]
    else:
        assert all(o.startswith("raised peer-memory exchange unavailable") for o in outs), outs
