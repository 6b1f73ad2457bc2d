"""The C++ drop-in headers (include/xbarsim/*.hpp) compile against the C ABI
and behave like the reference's API: tests/cpp/test_cpp_api.cpp, built with
g++ here and run in 'cpu' mode (validation / exception mapping) or, on a
B200, 'gpu' mode (CrossbarLinear bit-exact against the oracle)."""
import os
import subprocess

import pytest

from helpers import ROOT

LIB = os.path.join(ROOT, "paper_2002_11151_b200", "_lib")
ORC = os.path.join(ROOT, "oracle", "_build")


def _build(tmp_path):
    exe = str(tmp_path / "test_cpp_api")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_cpp_api.cpp"), "-o", exe, "-L", LIB, "-lxbarsim_b200", "-L", ORC,
           "-loracle", f"-Wl,-rpath,{LIB}", f"-Wl,-rpath,{ORC}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_headers_compile_and_map_errors(tmp_path, oracle_build):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_crossbar_linear_bit_exact_vs_oracle(tmp_path, oracle_build):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


def _build_um(tmp_path):
    exe = str(tmp_path / "test_update_mapping")
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_update_mapping.cpp"), "-o", exe, "-L", LIB, "-lxbarsim_b200",
           f"-Wl,-rpath,{LIB}"]
    subprocess.run(cmd, check=True)
    return exe


def test_cpp_update_mapping_validation(tmp_path):
    """The restated reference test_update.cpp / test_mapping.cpp compile
    against include/xbarsim/; validation cases run without a GPU."""
    r = subprocess.run([_build_um(tmp_path), "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_update_mapping_on_gpu(tmp_path):
    """Every restated test_update.cpp / test_mapping.cpp case on the GPU."""
    r = subprocess.run([_build_um(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
