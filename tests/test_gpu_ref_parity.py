"""GPU parity DIRECTLY against the reference: the unmodified reference sources
compiled here (oracle/_ref/libdcdref.so, built by `make -C oracle ref` and
shipped to the GPU box with the snapshot) — its own make_batch and uplink
observation (src/cluster.cpp:80-105,142-145) for the inputs and its own
decentralized_cd_detect / decentralized_cd_precode (src/detect.cpp:147-189,
src/precode.cpp:136-169) for the expected outputs — against the CUDA path
through the C ABI.  This closes the link that test_gpu_parity.py makes
transitively (CUDA == C restatement == reference).

Shapes: the north-star target (B=256, U=16, C=8) and BASELINE configs[0]
(B=64, U=8, C=2).  Tolerances: north_star's 1e-5 (fp32) and 2e-2 (fp16, the
half2 path also against the reference's own binary16 full-storage emulation).
"""
import numpy as np
import pytest

from helpers import TOL_FP16, TOL_FP32, rel_err, to_dev, to_host
from oracle.oracle import FP16, FULL_STORAGE, OPTIMAL, UNIFORM, Oracle, available, reference_batch

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not available("reference"), reason="oracle/_ref/libdcdref.so not built")]

SHAPES = [(8, 32, 16), (2, 32, 8)]  # (C, B_c, U): target, configs[0]
S = 40


@pytest.fixture(scope="module")
def ref():
    return Oracle("reference")


def _batch(shape, seed):
    C, Bc, U = shape
    return reference_batch(C, Bc, U, 16, S, seed, kind="reference")


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"C{s[0]}_Bc{s[1]}_U{s[2]}")
@pytest.mark.parametrize("fusion", ["uniform", "optimal"])
def test_uplink_fp32_against_reference(engine, ref, shape, fusion):
    b = _batch(shape, 21)
    fu = UNIFORM if fusion == "uniform" else OPTIMAL
    xhat, local, s2 = ref.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, fu)
    r = engine.ul_detect(to_dev(b["h_tiles"]), to_dev(b["y"]), n0=b["n0"], K=3, fusion=fusion)
    engine.sync()
    assert rel_err(to_host(r.x_local), local) <= TOL_FP32
    assert rel_err(to_host(r.xhat), xhat) <= TOL_FP32
    if fusion == "optimal":
        got = r.sigma2.cpu().numpy().reshape(s2.shape)
        assert np.max(np.abs(got - s2) / s2) <= TOL_FP32


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"C{s[0]}_Bc{s[1]}_U{s[2]}")
def test_downlink_fp32_against_reference(engine, ref, shape):
    C, Bc, U = shape
    b = _batch(shape, 22)
    sym = b["x_true"]  # the reference's own QAM symbols
    rho = float(np.sqrt(U))  # harness.cpp:159
    x, g = ref.dl_precode_batch(b["h_tiles"], sym, rho, 3)
    d = engine.dl_precode(to_dev(b["h_tiles"]), to_dev(sym), rho=rho, K=3)
    engine.sync()
    assert rel_err(to_host(d.x), x) <= TOL_FP32
    assert np.max(np.abs(d.gain.cpu().numpy() - g) / np.abs(g)) <= TOL_FP32


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"C{s[0]}_Bc{s[1]}_U{s[2]}")
@pytest.mark.parametrize("alg", ["sweep", "gram"])
def test_fp16_against_reference_and_its_emulation(engine, ref, shape, alg):
    """half2 sweep kernels (the paper's fp16 arithmetic) and the default fp16
    kernels: within 2e-2 of the reference in fp64 AND of the reference's own
    binary16 full-storage emulation (precision.cpp:43-72)."""
    C, Bc, U = shape
    b = _batch(shape, 23)
    xhat, local, _ = ref.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
    _, local16, _ = ref.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM, FP16, FULL_STORAGE)
    sym = b["x_true"]
    rho = float(np.sqrt(U))
    x, _ = ref.dl_precode_batch(b["h_tiles"], sym, rho, 3)
    x16, _ = ref.dl_precode_batch(b["h_tiles"], sym, rho, 3, FP16, FULL_STORAGE)
    prev = engine.fp16_algorithm
    engine.set_fp16_algorithm(alg)
    try:
        r = engine.ul_detect(to_dev(b["h_tiles"], "fp16", True), to_dev(b["y"], "fp16", True), n0=b["n0"], K=3)
        d = engine.dl_precode(to_dev(b["h_tiles"], "fp16", True), to_dev(sym, "fp16"), rho=rho, K=3)
        engine.sync()
    finally:
        engine.set_fp16_algorithm(prev)
    assert rel_err(to_host(r.x_local), local) <= TOL_FP16
    assert rel_err(to_host(r.x_local), local16) <= TOL_FP16
    assert rel_err(to_host(r.xhat), xhat) <= TOL_FP16
    assert rel_err(to_host(d.x), x) <= TOL_FP16
    assert rel_err(to_host(d.x), x16) <= TOL_FP16


def test_hard_decisions_match_the_reference_slicer(engine, ref):
    """Target shape: GPU fused estimates, unbiased by the device mmse_bias and
    sliced on the device, against the reference's own fused estimates sliced by
    the reference's Constellation::slice with the reference's bias factors —
    identical labels except at decision-boundary ties (counted)."""
    b = _batch((8, 32, 16), 24)
    xhat, _, _ = ref.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
    r = engine.ul_detect(to_dev(b["h_tiles"]), to_dev(b["y"]), n0=b["n0"], K=3)
    beta = engine.mmse_bias(to_dev(b["h_tiles"]), n0=b["n0"])
    labels = engine.slice(r.xhat, beta, qam=16).cpu().numpy().reshape(S, -1)
    engine.sync()
    want = np.zeros_like(labels)
    pts = ref.qam_points(16)
    ties = 0
    for s in range(S):
        bf = ref.mmse_bias_factors(b["h_full"][s], b["n0"], 1.0)
        z = xhat[s] / bf
        want[s] = ref.slice(16, z)
        d = np.abs(z[:, None] - pts[None, :]) ** 2
        d.sort(axis=1)
        ties += int(np.sum(d[:, 1] - d[:, 0] <= 1e-4 * d[:, 1]))
    mismatches = int(np.sum(labels != want))
    assert mismatches <= ties, (mismatches, ties)
