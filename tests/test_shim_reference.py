"""The reference's OWN unit tests (/root/reference/proj/tests/grid_test.cpp and
kernel_test.cpp, Catch2), compiled unmodified against the B200 drop-in:
include/yeeb200/compat/yeeblock/*.hpp forward the reference's header names to
the shim (namespace yeeblock -> yeeb200), include/yeeb200/compat/catch2/ is a
small Catch2-compatible harness (Catch2 is not in this image), and the
binary links libyeeb200.so. The kernel tests run in double precision: the
range operations (apply_ampere_range / apply_faraday_range / apply_pec_boundary
/ update_e_box) and total_energy execute as fp64 device kernels on the
caller's host FieldSet (yb_fs_apply, yb_fs_total_energy).

Recipe: tests/cpp/Makefile (run by __graft_entry__.build() here, where the
reference sources exist); the binary tests/cpp/_ref/ref_unit_tests is
git-ignored and travels to the GPU box with the tree."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "_ref", "ref_unit_tests")
REF_TESTS = "/root/reference/proj/tests"

# test cases that touch no device code: grid setup, extents, the range checks
# (thrown before any copy), soft-source and probe arithmetic on host arrays, digests
HOST_ONLY = ["build_coefficients", "stable_dt", "make_uniform_grid", "staggered extents",
             "range ops reject", "inject_current", "sample_probes", "probe records", "field digest"]


def binary():
    if os.path.isdir(REF_TESTS):
        r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
    if not os.path.exists(EXE):
        pytest.skip("reference unit tests not built (needs /root/reference/proj/tests at build time)")
    return EXE


def run(*args):
    return subprocess.run([binary(), *args], capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("name", HOST_ONLY)
def test_reference_unit_tests_host_side(yb, name):
    r = run(name)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "All tests passed" in r.stdout and " 0 test cases" not in r.stdout, r.stdout


@pytest.mark.gpu
def test_reference_unit_tests_all_on_gpu(yb):
    """Every test case of grid_test.cpp + kernel_test.cpp passes (16 cases)."""
    r = run()
    assert r.returncode == 0, r.stdout + r.stderr
    assert "All tests passed: 16 test cases" in r.stdout, r.stdout
