"""bench-cli (bench.hpp:41-391) on the B200 path:
paper_1301_4539_b200/yb_bench, built over the drop-in shim. CPU: it builds,
predict mode, flag errors. GPU: the reference harness's own run_case results
(checksum + probe text, tests/golden/bench_case.npz) are reproduced by every
variant; measure-mode CSV shape; energy drift."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_1301_4539_b200", "yb_bench")
GOLD = os.path.join(ROOT, "tests", "golden", "bench_case.npz")


@pytest.fixture(scope="module")
def cli(yb):
    if not os.path.exists(EXE):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1301_4539_b200", "csrc")], check=True,
                       capture_output=True)
    assert os.path.exists(EXE)
    return EXE


def run(cli, *args, check=True):
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check:
        assert r.returncode == 0, r.stderr
    return r


def test_cli_predict(cli):
    out = run(cli, "--mode", "predict", "--size", "256", "--hbm-gbs", "6000").stdout
    assert "fused" in out and "tb2" in out and "naive" in out
    line = [ln for ln in out.splitlines() if ln.startswith("tb2")][0].split()
    assert float(line[1]) == 24.0 and abs(float(line[2]) - 250.0) < 0.1


def test_cli_flag_errors(cli):
    assert run(cli, "--precision", "double", check=False).returncode == 2
    assert run(cli, "--case", "sphere", check=False).returncode == 2
    assert run(cli, "--variant", "tiled", check=False).returncode == 2
    assert run(cli, "--steps", "0", check=False).returncode == 2
    assert run(cli, "--bogus", "1", check=False).returncode == 2


@pytest.mark.gpu
def test_cli_verify_matches_reference_run_case(cli, tmp_path):
    """Every variant reproduces the reference harness's run_case checksum and
    probe file bit for bit (verify mode compares them with each other)."""
    d = np.load(GOLD)
    for q in range(int(d["ncases"])):
        n, steps, ss, stride = (int(v) for v in d[f"case{q}"])
        sd, amp = (float(v) for v in d[f"case{q}_params"])
        pf = tmp_path / f"probes{q}.tsv"
        out = run(cli, "--mode", "verify", "--size", n, "--steps", steps, "--source-steps", ss,
                  "--sigma-dt", sd, "--amplitude", amp, "--probe-stride", stride,
                  "--variant", "fused,tb2,naive", "--probes", pf).stdout
        assert "verify: PASS" in out and "FAIL" not in out, out
        assert f"checksum {str(d[f'case{q}_checksum'])}" in out, out
        assert pf.read_text() == str(d[f"case{q}_probes"])


@pytest.mark.gpu
def test_cli_measure_csv(cli, tmp_path):
    out = tmp_path / "t.csv"
    run(cli, "--mode", "measure", "--size", "48", "--steps", "10", "--variant", "fused,tb2,naive",
        "--out", out)
    lines = out.read_text().splitlines()
    assert lines[0] == "case,split,cores,precision,variant,mcs,total_s,vol_s,vol_pct,checksum"
    rows = [ln.split(",") for ln in lines[1:]]
    assert [r[4] for r in rows] == ["fused", "tb2", "naive"]
    assert len({r[9] for r in rows}) == 1  # checksum column constant across variants
    for r in rows:
        mcs, total = float(r[5]), float(r[6])
        assert abs(mcs - 48 ** 3 * 10 / total / 1e6) <= 0.005 * mcs + 0.01
    md = tmp_path / "t.md"
    run(cli, "--mode", "measure", "--size", "16", "--steps", "4", "--variant", "fused", "--out", md)
    assert md.read_text().startswith("| case | split |")


@pytest.mark.gpu
def test_cli_energy_drift(cli):
    """64^3, 1000 steps, single precision: drift < 1e-4."""
    out = run(cli, "--mode", "energy", "--size", "64", "--steps", "1000", "--source-steps", "50").stdout
    drift = float(out.strip().split()[-1])
    assert 0.0 <= drift < 1e-4, out
