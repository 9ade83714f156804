"""GPU: hard decisions of the CUDA path equal the reference's, except at
decision-boundary ties, which are counted and reported (north_star).

Uplink: slice(x̂_u / β_u) with β from the reference's full-H MMSE bias factors
(run_uplink_round, src/cluster.cpp:196-203; mmse_bias_factors,
src/detect.cpp:227-242), nearest point with ties to the lowest label
(Constellation::slice, src/mimo.cpp:111-122).
Downlink: the genie-rescaled receive y0/β with β = Re(s^H y0)/||s||^2
(downlink_receive_and_ber, src/precode.cpp:204-233), noiseless here so the
comparison isolates the precoder.

A mismatch counts as a tie when the reference value's two nearest
constellation points are closer to equidistant than the numeric tolerance
allows: |d1 - d2| <= tol * (d1 + d2) with tol = 1e-4 (fp32) / 5e-2 (fp16)."""
import numpy as np
import pytest

from helpers import UNIFORM, FP16, FULL_STORAGE, batch, to_dev, to_host

pytestmark = pytest.mark.gpu


def _near_tie(port, y, qam, tol):
    pts = port.qam_points(qam)
    d = np.sort(np.abs(y[:, None] - pts[None, :]) ** 2, axis=1)
    return np.abs(d[:, 0] - d[:, 1]) <= tol * (d[:, 0] + d[:, 1])


def _compare(port, got, ref, qam, tol):
    lg, lr = port.slice(qam, got), port.slice(qam, ref)
    mism = lg != lr
    ties = _near_tie(port, ref, qam, tol)
    return int(mism.sum()), int((mism & ties).sum()), int(mism.size)


@pytest.mark.parametrize("fmt,snr_db,qam", [("fp32", 10.0, 16), ("fp32", 25.0, 64), ("fp16", 10.0, 16)])
def test_uplink_hard_decisions(engine, port, fmt, snr_db, qam, record_property):
    C, Bc, U, S = 8, 32, 16, 300
    b = batch(C, Bc, U, qam=qam, S=S, seed=17, snr_db=snr_db)
    if fmt == "fp32":
        xr, _, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
    else:
        xr, _, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM, FP16, FULL_STORAGE)
    r = engine.ul_detect(to_dev(b["h_tiles"], fmt, True), to_dev(b["y"], fmt, True), n0=b["n0"], K=3)
    engine.sync()
    xg = to_host(r.xhat)
    beta = np.stack([port.mmse_bias_factors(b["h_full"][s], b["n0"], 1.0) for s in range(S)])
    tol = 1e-4 if fmt == "fp32" else 5e-2
    mism, ties, n = _compare(port, (xg / beta).ravel(), (xr / beta).ravel(), qam, tol)
    record_property("uplink_mismatches", mism)
    record_property("uplink_ties", ties)
    print(f"uplink {fmt} {qam}-QAM @{snr_db} dB: {n} decisions, {mism} differ, {ties} of them at ties")
    assert mism == ties


@pytest.mark.parametrize("fmt", ["fp32", "fp16"])
def test_downlink_hard_decisions(engine, port, fmt, record_property):
    C, Bc, U, S, qam = 8, 32, 16, 300, 16
    b = batch(C, Bc, U, qam=qam, S=S, seed=19)
    sym = b["x_true"]  # QAM symbols of the batch's payload bits
    rho = float(np.sqrt(U))
    if fmt == "fp32":
        xr, _ = port.dl_precode_batch(b["h_tiles"], sym, rho, 3)
    else:
        xr, _ = port.dl_precode_batch(b["h_tiles"], sym, rho, 3, FP16, FULL_STORAGE)
    d = engine.dl_precode(to_dev(b["h_tiles"], fmt, True), to_dev(sym, fmt), rho=rho, K=3)
    engine.sync()
    xg = to_host(d.x)
    tol = 1e-4 if fmt == "fp32" else 5e-2
    tot = [0, 0, 0]
    for s in range(S):
        hdl = b["h_full"][s].conj().T  # U x B
        out = []
        for x in (xg[s].ravel(), xr[s].ravel()):
            y0 = hdl @ x
            beta = np.real(np.vdot(sym[s], y0)) / np.real(np.vdot(sym[s], sym[s]))
            out.append(y0 / beta)
        m, t, n = _compare(port, out[0], out[1], qam, tol)
        tot = [tot[0] + m, tot[1] + t, tot[2] + n]
    record_property("downlink_mismatches", tot[0])
    record_property("downlink_ties", tot[1])
    print(f"downlink {fmt}: {tot[2]} decisions, {tot[0]} differ, {tot[1]} of them at ties")
    assert tot[0] == tot[1]
