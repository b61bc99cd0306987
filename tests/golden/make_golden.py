"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
i.e. /root/reference/proj/include compiled by oracle/Makefile).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures are committed; tests compare the C oracle and the GPU path to
them without needing the reference at run time.

Cases (all fp32, Standard step order, schedule.hpp:171-210):
  axis_src    12x10x9 unit grid (make_uniform_grid semantics, safety 0.99),
              seeded random fields, config Gaussian source on Ez at the
              centre, 20 steps through apply_ampere_range / apply_pec_boundary
              / += src / apply_faraday_range.
  stretched   11x9x8 non-uniform dx/dy/dz (build_coefficients per axis),
              seeded random fields, 15 steps, no source.
  sim_refsrc  16^3 zero fields, yeeblock::Simulation<float> Standard with the
              reference's own SourceSpec (differentiated Gaussian), 30 steps;
              also the per-step increments inject_current adds.
  kat_hz      4^3, c*dt/h = 0.5, hz(2,2,2)=1, Ampere only
              (kernel_test.cpp:84-106).
  kat_faraday 4^3, c*dt/h = 0.5, ey(1,1,2)=1 then ez(1,2,1)=1, Faraday only
              (kernel_test.cpp:108-130).
  energy      total_energy (fields.hpp:116-146): (a) 13x11x9 stretched
              spacing, seeded E/H and a seeded H snapshot -> one value;
              (b) 20^3 unit grid, Gaussian Ez source for 30 steps then free,
              the leapfrog invariant after each of 60 single steps (the
              measure_energy_drift pattern, bench.hpp:273-303).
  bench_case  the reference bench harness's run_case (bench.hpp:105-127):
              cube cavity make_uniform_grid<float>(N, 1, c0, 0.99), default
              source (Ez pulse at the centre) and six default probes ->
              checksum and the format_probe_records text, for two configs.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrs):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrs)
    print("wrote", name)


def fields_dict(prefix, f):
    return {f"{prefix}_{O.COMP_NAMES[c]}": f[c] for c in range(6)}


def main():
    O.build()
    assert O.have_ref(), "oracle/_ref/libyeeref.so missing (needs /root/reference)"

    # axis_src
    nx, ny, nz = 12, 10, 9
    f0 = O.fill_fields(nx, ny, nz, 11)
    tab = O.gauss_table(20)
    src = O.Source(2, nx // 2, ny // 2, nz // 2, tab)
    f = [a.copy() for a in f0]
    O.ref_run_kernels(nx, ny, nz, f, 20, source=src)
    save("axis_src", dims=np.array([nx, ny, nz]), steps=np.array(20), seed=np.array(11),
         src=np.array([2, nx // 2, ny // 2, nz // 2]), table=tab,
         digest=np.array(O.ref_digest(nx, ny, nz, f), dtype=np.uint64),
         **fields_dict("in", f0), **fields_dict("out", f))

    # stretched
    nx, ny, nz = 11, 9, 8
    dx = np.linspace(0.8, 1.3, nx).astype(np.float32)
    dy = np.linspace(0.5, 2.0, ny).astype(np.float32)
    dz = np.full(nz, 1.25, np.float32)
    dt = O.ref_stable_dt(nx, ny, nz, dx, dy, dz, 1.0, 0.9)
    cdx, cdy, cdz = O.ref_coefficients(nx, ny, nz, dx, dy, dz, dt)
    f0 = O.fill_fields(nx, ny, nz, 12)
    f = [a.copy() for a in f0]
    O.ref_run_kernels(nx, ny, nz, f, 15, dx=dx, dy=dy, dz=dz, dt=dt)
    save("stretched", dims=np.array([nx, ny, nz]), steps=np.array(15), seed=np.array(12),
         cdx=cdx, cdy=cdy, cdz=cdz, dt=np.array(dt, np.float32),
         digest=np.array(O.ref_digest(nx, ny, nz, f), dtype=np.uint64),
         **fields_dict("in", f0), **fields_dict("out", f))

    # sim_refsrc: reference Simulation + reference SourceSpec
    n = 16
    dt = O.ref().yr_uniform_dt(n, 1.0, 1.0, 0.99)
    amp, sigma, t0, active = 1.0, 3.0 * dt, 12.0 * dt, 25
    f = O.zeros_state(n, n, n)
    _, dig = O.ref_simulation(n, n, n, f, 30, source=(2, 8, 8, 8, amp, sigma, t0, active))
    table = O.ref_source_table(n, n, n, 2, 8, 8, 8, amp, sigma, t0, active, float(np.float32(dt)), 30)
    save("sim_refsrc", dims=np.array([n, n, n]), steps=np.array(30),
         src=np.array([2, 8, 8, 8]), wave=np.array([amp, sigma, t0, active, float(np.float32(dt))]),
         table=table, digest=np.array(dig, dtype=np.uint64), **fields_dict("out", f))

    # kat_hz: Ampere only, c*dt/h = 0.5
    n = 4
    f = O.zeros_state(n, n, n)
    f[5][2, 2, 2] = 1.0  # hz(i=2,j=2,k=2)
    ones = np.ones(n, np.float32)
    O.ref_run_kernels(n, n, n, f, 1, dx=ones, dy=ones, dz=ones, dt=0.5, phases=1)
    save("kat_hz", dims=np.array([n, n, n]), **fields_dict("out", f))

    # kat_faraday: Faraday only
    f = O.zeros_state(n, n, n)
    f[1][2, 1, 1] = 1.0  # ey(1,1,2)
    O.ref_run_kernels(n, n, n, f, 1, dx=ones, dy=ones, dz=ones, dt=0.5, phases=4)
    g = O.zeros_state(n, n, n)
    g[2][1, 2, 1] = 1.0  # ez(1,2,1)
    O.ref_run_kernels(n, n, n, g, 1, dx=ones, dy=ones, dz=ones, dt=0.5, phases=4)
    save("kat_faraday", dims=np.array([n, n, n]), **fields_dict("ey", f), **fields_dict("ez", g))

    # energy
    nx, ny, nz = 13, 11, 9
    dx = np.linspace(0.7, 1.4, nx).astype(np.float32)
    dy = np.linspace(1.2, 0.6, ny).astype(np.float32)
    dz = np.linspace(0.9, 1.1, nz).astype(np.float32)
    f = O.fill_fields(nx, ny, nz, 31)
    prev = O.fill_fields(nx, ny, nz, 32)[3:]
    e_static = O.ref_total_energy(nx, ny, nz, f, prev, dx, dy, dz)
    n, steps = 20, 60
    tab = O.gauss_table(30, t0=12.0, w=4.0)
    src = O.Source(2, n // 2, n // 2, n // 2, tab)
    g = O.zeros_state(n, n, n)
    series = []
    for t in range(steps):
        h = [a.copy() for a in g[3:]]
        O.ref_run_kernels(n, n, n, g, 1, step0=t, source=src)
        series.append(O.ref_total_energy(n, n, n, g, h))
    save("energy", dims=np.array([nx, ny, nz]), dx=dx, dy=dy, dz=dz, static=np.array(e_static),
         seeds=np.array([31, 32]), n=np.array(n), steps=np.array(steps), table=tab,
         series=np.array(series), **fields_dict("out", g))

    # bench_case
    cases = [(24, 40, 25, 8.0, 1.0, 5), (32, 60, 50, 8.0, 1.0, 20)]
    out = {}
    for q, (n, st, ss, sd, amp, stride) in enumerate(cases):
        chk, text = O.ref_run_case(n, st, source_steps=ss, sigma_dt=sd, amplitude=amp, probe_stride=stride)
        out[f"case{q}"] = np.array([n, st, ss, stride])
        out[f"case{q}_params"] = np.array([sd, amp])
        out[f"case{q}_checksum"] = np.array(chk)
        out[f"case{q}_probes"] = np.array(text)
    save("bench_case", ncases=np.array(len(cases)), **out)


if __name__ == "__main__":
    main()
