"""CPU tests of the drop-in boundary: libyeeb200.so builds for sm_100a, loads,
exports every symbol include/yeeb200.h declares, and fails loudly (no CPU
fallback) when no GPU is present."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "yeeb200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|size_t)\s+(yb_\w+)\(", txt, re.M)))


def test_header_symbols_listed(yb):
    syms = header_symbols()
    assert len(syms) >= 20
    assert sorted(yb.ABI_SYMBOLS) == syms


def test_library_exports_all_symbols(yb):
    L = C.CDLL(yb.LIB_PATH)
    for s in header_symbols():
        assert hasattr(L, s), s
    assert L.yb_abi_version() == 5


def test_library_is_sm100a_only(yb):
    out = subprocess.run(["cuobjdump", "--list-elf", yb.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_sass_uses_tma(yb):
    out = subprocess.run(["cuobjdump", "-sass", yb.LIB_PATH], capture_output=True, text=True)
    assert "UTMALDG.3D" in out.stdout
    assert "SYNCS.PHASECHK.TRANS64.TRYWAIT" in out.stdout


def test_no_oracle_in_product():
    # the product library and package never reference the oracle
    pkg = os.path.join(ROOT, "paper_1301_4539_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "yee_oracle" not in txt and "pyoracle" not in txt and "liboracle" not in txt, f


def test_fails_loudly_without_gpu(yb):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(yb.YeeError):
        yb.Simulation(8, 8, 8)


def test_invalid_arguments_rejected_before_gpu(yb):
    with pytest.raises(yb.YeeInvalidArgument):
        yb.Simulation(0, 8, 8)


def build_shim_kat(tmp_path):
    exe = os.path.join(str(tmp_path), "shim_kat")
    r = subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "shim_kat.cpp"),
                        "-L", os.path.join(ROOT, "paper_1301_4539_b200"), "-lyeeb200",
                        "-Wl,-rpath," + os.path.join(ROOT, "paper_1301_4539_b200"), "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_cpp_shim_compiles(yb, tmp_path):
    """The C++ drop-in (include/yeeb200/yeeblock.hpp) builds against the C-ABI."""
    assert os.path.exists(build_shim_kat(tmp_path))
