"""GPU parity of the CUDA hot path against the CPU oracle (the C restatement
pinned bit-exactly to the reference), on the reference's own seeded
Rayleigh/QAM/AWGN inputs (make_batch + run_uplink_round's observation,
src/cluster.cpp:80-105,142-145), through the C ABI.

Tolerances (north_star / BASELINE.md §4): per-problem relative error
||x_gpu - x_ref|| / ||x_ref|| <= 1e-5 for fp32 and <= 2e-2 for fp16 (half2),
the fp16 path also against the reference's fp16 full-storage emulation.
"""
import numpy as np
import pytest

from helpers import (FP16, FP64, FULL_STORAGE, MESSAGES, OPTIMAL, TOL_FP16, TOL_FP32, UNIFORM, batch, qam_symbols,
                     rel_err, to_dev, to_host)

pytestmark = pytest.mark.gpu

# (C, B_c, U): register-resident specialisations and generic-path shapes
SHAPES = [
    (8, 32, 16),   # north-star target B=256 U=16 C=8
    (2, 32, 8),    # config 1 (B=64 U=8 C=2) / paper B_c=32 U=8
    (8, 16, 16),   # B=128 C=8
    (4, 64, 16),   # B=256 C=4
    (2, 64, 8),
    (3, 24, 6),    # generic (odd sizes)
    (1, 128, 16),  # generic, B=128 C=1
    (4, 20, 5),    # generic
    (4, 32, 32),   # configs[4]: B=128 U=32 C=4
    (2, 64, 32),   # B=128 U=32 C=2
    (8, 16, 32),   # B=128 U=32 C=8 (downlink infeasible: B_c < U)
    (2, 256, 16),  # B=512 C=2: multi-warp (2 warps per problem)
    (1, 128, 32),  # multi-warp, U=32
    (2, 256, 32),  # multi-warp, 4 warps
    (1, 512, 32),  # multi-warp, 8 warps
    (1, 512, 16),
    (1, 1024, 16),
]


@pytest.mark.parametrize("shape,S", [((8, 32, 16), 1200), ((1, 256, 16), 1400), ((1, 512, 32), 400)],
                         ids=lambda v: str(v))
def test_persistent_grid_loops(engine, port, shape, S):
    """More problems than resident warps/CTAs: every persistent worker runs
    several problems through its staging slot (prefetch + phase flips)."""
    C, Bc, U = shape
    b = batch(C, Bc, U, S=S, seed=77)
    xhat, local, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
    r = engine.ul_detect(to_dev(b["h_tiles"]), to_dev(b["y"]), n0=b["n0"], K=3)
    sym = qam_symbols(S, U)
    x, g = port.dl_precode_batch(b["h_tiles"], sym, float(np.sqrt(U)), 3)
    d = engine.dl_precode(to_dev(b["h_tiles"]), to_dev(sym), rho=float(np.sqrt(U)), K=3)
    engine.sync()
    assert rel_err(to_host(r.x_local), local) <= TOL_FP32
    assert rel_err(to_host(d.x), x) <= TOL_FP32
    assert np.max(np.abs(d.gain.cpu().numpy() - g) / np.abs(g)) <= TOL_FP32


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"C{s[0]}_Bc{s[1]}_U{s[2]}")
@pytest.mark.parametrize("fusion", ["uniform", "optimal"])
def test_uplink_fp32(engine, port, shape, fusion):
    C, Bc, U = shape
    b = batch(C, Bc, U, S=48)
    fu = UNIFORM if fusion == "uniform" else OPTIMAL
    xhat, local, s2 = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, fu)
    r = engine.ul_detect(to_dev(b["h_tiles"]), to_dev(b["y"]), n0=b["n0"], K=3, fusion=fusion)
    engine.sync()
    assert rel_err(to_host(r.x_local), local) <= TOL_FP32
    assert rel_err(to_host(r.xhat), xhat) <= TOL_FP32
    if fusion == "optimal":
        got = r.sigma2.cpu().numpy()
        assert np.max(np.abs(got - s2) / s2) <= TOL_FP32


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"C{s[0]}_Bc{s[1]}_U{s[2]}")
def test_uplink_fp16(engine, port, shape):
    C, Bc, U = shape
    b = batch(C, Bc, U, S=48)
    xhat, local, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
    xhat16, local16, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM, FP16, FULL_STORAGE)
    r = engine.ul_detect(to_dev(b["h_tiles"], "fp16", True), to_dev(b["y"], "fp16", True), n0=b["n0"], K=3,
                         fusion="uniform")
    engine.sync()
    assert rel_err(to_host(r.x_local), local) <= TOL_FP16
    assert rel_err(to_host(r.x_local), local16) <= TOL_FP16
    assert rel_err(to_host(r.xhat), xhat) <= TOL_FP16


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"C{s[0]}_Bc{s[1]}_U{s[2]}")
@pytest.mark.parametrize("fmt", ["fp32", "fp16"])
def test_downlink(engine, port, shape, fmt):
    C, Bc, U = shape
    if Bc < U:
        pytest.skip("downlink needs B_c >= U")
    b = batch(C, Bc, U, S=48)
    sym = qam_symbols(48, U)
    rho = float(np.sqrt(U))  # harness.cpp:159, rho = sqrt(U * Ex)
    x, g = port.dl_precode_batch(b["h_tiles"], sym, rho, 3)
    r = engine.dl_precode(to_dev(b["h_tiles"], fmt, True), to_dev(sym, fmt), rho=rho, K=3)
    engine.sync()
    tol = TOL_FP32 if fmt == "fp32" else TOL_FP16
    assert rel_err(to_host(r.x), x) <= tol
    got_g = r.gain.cpu().numpy()
    assert np.max(np.abs(got_g - g) / np.abs(g)) <= tol
    if fmt == "fp16":
        x16, _ = port.dl_precode_batch(b["h_tiles"], sym, rho, 3, FP16, FULL_STORAGE)
        assert rel_err(to_host(r.x), x16) <= TOL_FP16


def test_target_shape_large_batch(engine, port):
    """North-star shape at a few thousand problems, fp32 UL+DL in one go."""
    b = batch(8, 32, 16, S=400, seed=11)
    xhat, local, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
    r = engine.ul_detect(to_dev(b["h_tiles"]), to_dev(b["y"]), n0=b["n0"], K=3)
    engine.sync()
    assert rel_err(to_host(r.x_local), local) <= TOL_FP32
    assert rel_err(to_host(r.xhat), xhat) <= TOL_FP32
