"""GPU: build and run the C++ parity suite (tests/cpp/test_gpu_api.cpp) that
exercises the dcd::gpu host API exactly as the reference's doctest suites
exercise dcd:: (same cases, GPU tolerances, identical exception texts)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_gpu_api.cpp")
BENCH_SRC = os.path.join(ROOT, "tests", "cpp", "bench_cpp_api.cpp")
PKG = os.path.join(ROOT, "paper_1902_08653_b200")
ORACLE = os.path.join(ROOT, "oracle")


def build(out, src=SRC):
    cmd = ["g++", "-std=c++20", "-O2", "-pthread", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           src, "-o", out, "-L", PKG, "-ldcdg", f"-Wl,-rpath,{PKG}", os.path.join(ORACLE, "libdcdoracle.so"),
           f"-Wl,-rpath,{ORACLE}", "-L", "/usr/local/cuda/lib64", "-lcudart", "-ldl"]
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


def test_cpp_latency_bench_compiles(tmp_path):
    build(str(tmp_path / "bench_cpp_api"), BENCH_SRC)


@pytest.mark.gpu
def test_cpp_latency_bench_runs(tmp_path):
    """The drop-in surface's per-call and batched-round timing program
    (numbers for DESIGN.md come from its full run; --quick here)."""
    import json
    exe = str(tmp_path / "bench_cpp_api")
    build(exe, BENCH_SRC)
    r = subprocess.run([exe, "--quick"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    print(out)
    assert out["per_call_us"]["decentralized_cd_detect_uniform"] > 0
    assert out["batched_round"]["detect_us_per_subcarrier"] > 0
