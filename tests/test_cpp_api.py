"""GPU: build and run the C++ parity suite (tests/cpp/test_gpu_api.cpp) that
exercises the dcd::gpu host API exactly as the reference's doctest suites
exercise dcd:: (same cases, GPU tolerances, identical exception texts)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_gpu_api.cpp")
PKG = os.path.join(ROOT, "paper_1902_08653_b200")
ORACLE = os.path.join(ROOT, "oracle")


def build(out):
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", SRC,
           "-o", out, "-L", PKG, "-ldcdg", f"-Wl,-rpath,{PKG}", os.path.join(ORACLE, "libdcdoracle.so"),
           f"-Wl,-rpath,{ORACLE}", "-L", "/usr/local/cuda/lib64", "-lcudart"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_cpp_suite_compiles(tmp_path):
    build(str(tmp_path / "test_gpu_api"))


@pytest.mark.gpu
def test_cpp_suite_passes(tmp_path):
    exe = str(tmp_path / "test_gpu_api")
    build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout
