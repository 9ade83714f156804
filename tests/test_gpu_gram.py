"""The Gram-space fp16 kernels (dcdg_gram_kernels.cuh).  Uplink (ul_gram_f16):
G = H^H H and z = H^H y on the tensor cores, Alg. 1's sweeps (detect.cpp:67-110)
in c = H^H r.  Downlink (dl_gram_f16): Alg. 2's dual sweeps (precode.cpp:52-99)
in w = H^H x = G a, then x = H a, power_scale and the effective gain.  Checked against the CPU oracle on the reference's seeded
batches at the fp16 tolerance (2e-2, against both the fp64 reference and its
fp16 full-storage emulation), against the half2 sweep kernel, and at
convergence against the exact L-MMSE solution of the stored fp16 inputs."""
import numpy as np
import pytest

from helpers import FP16, FULL_STORAGE, OPTIMAL, TOL_FP16, UNIFORM, batch, qam_symbols, rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


def _run(engine, b, alg, K=3, n0=None):
    engine.set_fp16_algorithm(alg)
    try:
        r = engine.ul_detect(to_dev(b["h_tiles"], "fp16", True), to_dev(b["y"], "fp16", True),
                             n0=b["n0"] if n0 is None else n0, K=K)
        engine.sync()
    finally:
        engine.set_fp16_algorithm("gram")
    return to_host(r.x_local), to_host(r.xhat)


def test_dispatch_names(engine):
    from paper_1902_08653_b200._lib import FP16 as F16
    assert engine.kernel_name(0, 32, 16, F16).startswith("ul_gram_f16")
    engine.set_fp16_algorithm("sweep")
    try:
        assert engine.kernel_name(0, 32, 16, F16).startswith("ul_reg_f16")
    finally:
        engine.set_fp16_algorithm("gram")
    assert engine.kernel_name(1, 32, 16, F16).startswith("dl_gram_f16")
    engine.set_fp16_algorithm("sweep")
    try:
        assert engine.kernel_name(1, 32, 16, F16).startswith("dl_reg_f16")
    finally:
        engine.set_fp16_algorithm("gram")
    # other shapes keep their kernels
    assert not engine.kernel_name(0, 32, 8, F16).startswith("ul_gram")
    assert not engine.kernel_name(1, 32, 8, F16).startswith("dl_gram")
    with pytest.raises(ValueError):
        engine.set_fp16_algorithm("tensor")


@pytest.mark.parametrize("C,S,K", [(8, 48, 3), (8, 1200, 3), (3, 7, 3), (1, 5, 1), (8, 64, 8)],
                         ids=lambda v: str(v))
def test_gram_vs_oracle(engine, port, C, S, K):
    """Target tile (B_c=32, U=16); S*C not a multiple of the 4 problems of a
    set exercises the zero-filled TMA rows; S=1200 the persistent loop."""
    b = batch(C, 32, 16, S=S, seed=11 + S)
    xhat, local, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, K, UNIFORM)
    _, local16, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, K, UNIFORM, FP16, FULL_STORAGE)
    xl, xh = _run(engine, b, "gram", K)
    assert rel_err(xl, local) <= TOL_FP16
    assert rel_err(xl, local16) <= TOL_FP16
    assert rel_err(xh, xhat) <= TOL_FP16


def test_gram_more_accurate_than_half2(engine, port):
    """fp32 accumulation of exact fp16 products: the Gram path sits closer to
    the fp64 reference than the half2 arithmetic path (same fp16 inputs)."""
    b = batch(8, 32, 16, S=256, seed=5)
    _, local, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
    g, _ = _run(engine, b, "gram")
    s, _ = _run(engine, b, "sweep")
    eg, es = rel_err(g, local), rel_err(s, local)
    assert eg <= TOL_FP16 and es <= TOL_FP16
    assert eg < es
    assert rel_err(g, s) <= TOL_FP16


def test_gram_noiseless_and_convergence(engine, port):
    """N0 = 0 (kappa = 0, m_j = 1/||h_j||^2) and T = 200 sweeps, which reach the
    exact L-MMSE solution (acceptance criterion 1) of the fp16-stored channel
    within the fp16 output rounding."""
    b = batch(2, 32, 16, S=16, seed=3)
    h16 = b["h_tiles"].astype(np.complex64)
    h16 = (h16.real.astype(np.float16).astype(np.float64) + 1j * h16.imag.astype(np.float16).astype(np.float64))
    y16 = b["y"].astype(np.complex64)
    y16 = (y16.real.astype(np.float16).astype(np.float64) + 1j * y16.imag.astype(np.float16).astype(np.float64))
    xl, _ = _run(engine, b, "gram", K=200)
    S, C, U, Bc = h16.shape
    worst = 0.0
    for s in range(S):
        for c in range(C):
            Hm = h16[s, c].T  # B_c x U
            x = np.linalg.solve(Hm.conj().T @ Hm + b["n0"] * np.eye(U), Hm.conj().T @ y16[s, c])
            worst = max(worst, np.linalg.norm(xl[s, c] - x) / np.linalg.norm(x))
    assert worst <= 2e-3
    _, local0, _ = port.ul_detect_batch(b["h_tiles"], b["y"], 0.0, 1.0, 3, UNIFORM)
    xl0, _ = _run(engine, b, "gram", K=3, n0=0.0)
    assert rel_err(xl0, local0) <= TOL_FP16


def _run_dl(engine, b, sym, alg, rho, K=3, gain=True):
    engine.set_fp16_algorithm(alg)
    try:
        r = engine.dl_precode(to_dev(b["h_tiles"], "fp16", True), to_dev(sym, "fp16"), rho=rho, K=K, want_gain=gain)
        engine.sync()
    finally:
        engine.set_fp16_algorithm("gram")
    return to_host(r.x), (r.gain.cpu().numpy() if gain else None)


@pytest.mark.parametrize("C,S,K", [(8, 48, 3), (8, 1200, 3), (3, 7, 3), (1, 5, 1), (8, 64, 8)],
                         ids=lambda v: str(v))
def test_dl_gram_vs_oracle(engine, port, C, S, K):
    """Target tile; ragged sets (S*C not a multiple of 4), the persistent loop,
    C=1 and more sweeps.  Precoder, per-subcarrier effective gain, and the
    per-cluster power rho/sqrt(C) (precode.cpp:155) of the fp16 output."""
    U = 16
    b = batch(C, 32, U, S=S, seed=21 + S)
    sym = qam_symbols(S, U, seed=S)
    rho = float(np.sqrt(U))
    x, g = port.dl_precode_batch(b["h_tiles"], sym, rho, K)
    x16, _ = port.dl_precode_batch(b["h_tiles"], sym, rho, K, FP16, FULL_STORAGE)
    got, gg = _run_dl(engine, b, sym, "gram", rho, K)
    assert rel_err(got, x) <= TOL_FP16
    assert rel_err(got, x16) <= TOL_FP16
    assert np.max(np.abs(gg - g) / np.abs(g)) <= TOL_FP16
    pw = np.linalg.norm(got.reshape(S, C, -1), axis=-1)
    assert np.max(np.abs(pw - rho / np.sqrt(C))) <= 2e-3 * rho


def test_dl_gram_more_accurate_than_half2(engine, port):
    U = 16
    b = batch(8, 32, U, S=256, seed=9)
    sym = qam_symbols(256, U, seed=4)
    rho = float(np.sqrt(U))
    x, _ = port.dl_precode_batch(b["h_tiles"], sym, rho, 3)
    g, _ = _run_dl(engine, b, sym, "gram", rho)
    s, _ = _run_dl(engine, b, sym, "sweep", rho)
    eg, es = rel_err(g, x), rel_err(s, x)
    assert eg <= TOL_FP16 and es <= TOL_FP16
    assert eg < es
    assert rel_err(g, s) <= TOL_FP16


def test_dl_gram_raw_beamformer_and_convergence(engine):
    """rho = 0 returns the unscaled cd_precode beamformer; T = 200 sweeps reach
    zero-forcing of the stored fp16 channel (H^H x = s, precode.cpp:339-359
    analogue), within the fp16 output rounding."""
    U, S, C = 16, 16, 2
    b = batch(C, 32, U, S=S, seed=5)
    sym = qam_symbols(S, U, seed=2)
    got, _ = _run_dl(engine, b, sym, "gram", 0.0, K=200, gain=False)
    h16 = b["h_tiles"].astype(np.complex64)
    h16 = h16.real.astype(np.float16).astype(np.float64) + 1j * h16.imag.astype(np.float16).astype(np.float64)
    s16 = sym.astype(np.complex64)
    s16 = s16.real.astype(np.float16).astype(np.float64) + 1j * s16.imag.astype(np.float16).astype(np.float64)
    worst = 0.0
    xs = got.reshape(S, C, 32)
    for s in range(S):
        for c in range(C):
            Hm = h16[s, c].T  # B_c x U
            recv = Hm.conj().T @ xs[s, c]
            worst = max(worst, np.linalg.norm(recv - s16[s]) / np.linalg.norm(s16[s]))
    assert worst <= 5e-3


def test_dl_gram_zero_row_message(engine):
    """A zero channel column raises the reference's runtime_error text naming
    the lowest zero user (precode.cpp:74-76)."""
    from paper_1902_08653_b200 import NumericError
    U, S, C = 16, 8, 8
    b = batch(C, 32, U, S=S, seed=1)
    h = b["h_tiles"].copy()
    h[3, 5, 9, :] = 0
    h[3, 5, 11, :] = 0
    b = dict(b, h_tiles=h)
    sym = qam_symbols(S, U, seed=1)
    with pytest.raises(NumericError, match="cd_precode: user 9 has an all-zero channel row") as ei:
        _run_dl(engine, b, sym, "gram", 4.0)
    assert ei.value.problem == 3 * C + 5
    engine.sync()


def test_dl_gram_zero_beamformer(engine):
    """All-zero symbols give x = 0, which power_scale rejects (precode.cpp:107-108)."""
    from paper_1902_08653_b200 import NumericError
    U, S, C = 16, 4, 8
    b = batch(C, 32, U, S=S, seed=2)
    sym = qam_symbols(S, U, seed=3)
    sym[1] = 0
    with pytest.raises(NumericError, match="power_scale: zero beamformer cannot be scaled") as ei:
        _run_dl(engine, b, sym, "gram", 4.0)
    assert ei.value.problem == 1 * C
    engine.sync()


@pytest.mark.parametrize("C,S", [(8, 48), (3, 7), (8, 1200)], ids=lambda v: str(v))
def test_gram_optimal_fusion_fused_variance(engine, port, C, S):
    """Optimal fusion on the Gram kernel: post_eq_variance (detect.cpp:112-130)
    from the kernel's own Gram by the in-place sweep operator, fp16 wire
    rounding of sigma^2, then the weighted fusion; against the fp64 reference,
    its fp16 full-storage emulation, and the standalone variance kernel."""
    U = 16
    b = batch(C, 32, U, S=S, seed=31 + S)
    xhat, local, s2 = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, OPTIMAL)
    xhat16, _, s216 = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, OPTIMAL, FP16, FULL_STORAGE)
    H16 = to_dev(b["h_tiles"], "fp16", True)
    r = engine.ul_detect(H16, to_dev(b["y"], "fp16", True), n0=b["n0"], K=3, fusion="optimal")
    engine.sync()
    assert engine.kernel_name(0, 32, 16, 1).startswith("ul_gram_f16")
    got = r.sigma2.cpu().numpy()
    assert np.max(np.abs(got - s2) / s2) <= TOL_FP16
    assert np.max(np.abs(got - s216) / s216) <= TOL_FP16
    standalone = engine.post_eq_variance(H16, n0=b["n0"]).cpu().numpy()
    assert np.max(np.abs(got - standalone) / standalone) <= 2e-3  # both on the fp16 grid
    assert rel_err(to_host(r.xhat), xhat) <= TOL_FP16
    assert rel_err(to_host(r.xhat), xhat16) <= TOL_FP16
    assert rel_err(to_host(r.x_local), local) <= TOL_FP16
