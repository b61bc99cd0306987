"""Multi-sweep launches under concurrent load on one GPU: two (or three) handles, each with its
own stream, run their persistent multi-sweep launches at the same time from separate host threads.
The second launch's CTAs only become resident as the first one's retire, so its in-kernel
dependency waits (globaltimer-bounded, yb_tb2.cu `wait_neighbours`) see long, irregular delays;
every dependency still points at an item a resident CTA holds, so no wait may time out and the
results must equal the solo runs bit for bit. Also a streamed run (tile-row upload + readback
words polled in-kernel and by the copy stream) next to a plain run."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def make(yb, nx, ny, nz, seed):
    s = yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2)
    s.generate_medium(seed, seed)
    s.fill(seed + 10)
    return s


@pytest.mark.parametrize("nsims", [2, 3])
def test_concurrent_multisweep_launches(yb, nsims):
    nx, ny, nz, steps = 512, 256, 96, 60
    solo = []
    for q in range(nsims):
        with make(yb, nx, ny, nz, q + 1) as s:
            s.run(steps)
            solo.append(s.download())
    sims = [make(yb, nx, ny, nz, q + 1) for q in range(nsims)]
    errs = [None] * nsims
    start = threading.Barrier(nsims)

    def work(q):
        try:
            start.wait()
            for _ in range(3):  # 3 x 20 steps: several launches per handle interleave
                sims[q].run(steps // 3)
        except Exception as e:  # noqa: BLE001 - reported below
            errs[q] = e

    th = [threading.Thread(target=work, args=(q,)) for q in range(nsims)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    try:
        assert errs == [None] * nsims, errs
        for q in range(nsims):
            got = sims[q].download()
            for c in range(6):
                assert np.array_equal(bits(got[c]), bits(solo[q][c])), (q, c)
    finally:
        for s in sims:
            s.close()


def test_streamed_run_next_to_a_plain_run(yb, monkeypatch):
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("YB_UP_STREAM", "1")
    nx, ny, nz, steps = 256, 256, 64, 40

    def pin(a):
        t = torch.empty(a.shape, dtype=torch.float32).pin_memory()
        t.numpy()[...] = a
        return t.numpy()

    med = yb.host_medium_slab(nx, ny, nz, 0, nz, 2, 2, [np.empty((nz, ny, nx), np.float32) for _ in range(4)])
    cells = {q: pin(med[q]) for q in range(4)}
    fields = [np.empty(yb.comp_extents(nx, ny, nz, c)[::-1], np.float32) for c in range(6)]
    yb.host_fields_slab(nx, ny, nz, 0, nz, 3, out=fields)
    pf = [pin(a) for a in fields]
    out = [torch.empty(a.shape, dtype=torch.float32).pin_memory().numpy() for a in fields]
    with yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2) as s:
        s.set_cell_coeffs_many(cells)
        s.upload(pf)
        s.run(steps)
        want = s.download()
    with make(yb, 512, 256, 96, 7) as other:
        other.run(60)
        want_other = other.download()
    a = yb.Simulation(nx, ny, nz, variant=yb.VARIANT_TB2)
    b = make(yb, 512, 256, 96, 7)
    errs = []
    start = threading.Barrier(2)

    def run_a():
        try:
            start.wait()
            a.run_streamed(steps, cells, pf, out=out)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    def run_b():
        try:
            start.wait()
            b.run(60)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run_a), threading.Thread(target=run_b)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    try:
        assert not errs, errs
        assert a.info()["streamed_uploads"] == 1
        got_b = b.download()
        for c in range(6):
            assert np.array_equal(bits(out[c]), bits(want[c])), c
            assert np.array_equal(bits(got_b[c]), bits(want_other[c])), c
    finally:
        a.close()
        b.close()
