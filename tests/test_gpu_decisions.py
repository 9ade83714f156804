"""GPU: the device hard-decision path against the oracle —
full-H MMSE bias factors (mmse_bias_factors, src/detect.cpp:227-242), the QAM
slicer (Constellation::slice, src/mimo.cpp:111-122: bit-exact labels on the
same inputs, exact decision-boundary ties to the lowest label), bit-error
counting, a full uplink BER round, and the downlink genie receive
(downlink_receive_and_ber, src/precode.cpp:204-233)."""
import numpy as np
import pytest
import torch

from helpers import UNIFORM, batch, rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("C,Bc,U", [(8, 32, 16), (2, 32, 8), (3, 24, 6)])
def test_mmse_bias_factors(engine, port, C, Bc, U):
    b = batch(C, Bc, U, S=24, seed=41)
    beta = engine.mmse_bias(to_dev(b["h_tiles"]), n0=b["n0"]).cpu().numpy()
    engine.sync()
    ref = np.stack([port.mmse_bias_factors(b["h_full"][s], b["n0"], 1.0) for s in range(24)])
    assert np.max(np.abs(beta - ref) / ref) <= 1e-5
    ones = engine.mmse_bias(to_dev(b["h_tiles"]), n0=0.0).cpu().numpy()
    assert np.all(ones == 1.0)


@pytest.mark.parametrize("qam", [4, 16, 64])
def test_slicer_bit_exact_including_ties(engine, port, qam):
    rng = np.random.default_rng(qam)
    pts = port.qam_points(qam)
    # random points plus exact midpoints between neighbouring levels (ties)
    x = (rng.standard_normal(4000) + 1j * rng.standard_normal(4000)) * 0.8
    lv = np.unique(pts.real)
    mids = (lv[:-1] + lv[1:]) / 2
    ties = np.array([complex(m, l) for m in mids for l in lv] + [complex(l, m) for m in mids for l in lv] +
                    [complex(m, n) for m in mids for n in mids])
    x = np.concatenate([x, ties]).astype(np.complex64)
    beta = rng.uniform(0.6, 1.0, x.size).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    bt = torch.from_numpy(beta).cuda()
    got = engine.slice(xt, bt, qam=qam).cpu().numpy()
    engine.sync()
    want = port.slice(qam, x.astype(np.complex128) / beta.astype(np.float64))
    assert np.array_equal(got, want)
    got0 = engine.slice(xt, None, qam=qam).cpu().numpy()
    assert np.array_equal(got0, port.slice(qam, x.astype(np.complex128)))


def test_uplink_ber_round(engine, port):
    """Device BER == reference BER for the decentralized detector (bit
    errors identical except where a decision sits at a tie)."""
    C, Bc, U, S, qam = 8, 32, 16, 400, 16
    b = batch(C, Bc, U, qam=qam, S=S, seed=43, snr_db=4.0)
    xhat, labels, errs = engine.uplink_round(to_dev(b["h_tiles"]), to_dev(b["y"]),
                                             torch.from_numpy(b["bits"]).cuda(), n0=b["n0"], qam=qam)
    engine.sync()
    xr, _, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
    beta = np.stack([port.mmse_bias_factors(b["h_full"][s], b["n0"], 1.0) for s in range(S)])
    ref_labels = port.slice(qam, (xr / beta).ravel()).reshape(S, U)
    bps = 4
    ref_bits = ((ref_labels[..., None] >> np.arange(bps - 1, -1, -1)) & 1).reshape(S, -1)
    ref_errs = int((ref_bits != b["bits"]).sum())
    got_labels = labels.cpu().numpy()
    mism = int((got_labels != ref_labels).sum())
    print(f"uplink round @4 dB: {S * U * bps} bits, device errors {int(errs.item())}, reference {ref_errs}, "
          f"{mism} decisions differ")
    assert mism == 0
    assert int(errs.item()) == ref_errs
    assert rel_err(to_host(xhat), xr) <= 1e-5


def test_downlink_receive(engine, port):
    C, Bc, U, S, qam = 8, 32, 16, 200, 16
    b = batch(C, Bc, U, qam=qam, S=S, seed=47)
    sym = b["x_true"]
    H = to_dev(b["h_tiles"])
    st = to_dev(sym)
    d = engine.dl_precode(H, st, rho=float(np.sqrt(U)), K=3)
    rng = np.random.default_rng(5)
    noise = ((rng.standard_normal((S, U)) + 1j * rng.standard_normal((S, U))) * np.sqrt(0.05 / 2)).astype(np.complex64)
    labels, beta, flagged = engine.dl_receive(H, d.x, st, torch.view_as_real(torch.from_numpy(noise).cuda()), qam=qam)
    engine.sync()
    x = to_host(d.x)
    pts = port.qam_points(qam)
    mism = ties = 0
    for s in range(S):
        y0 = b["h_full"][s].conj().T @ x[s].ravel()  # the same beamformer through an fp64 receive
        bref = np.real(np.vdot(sym[s], y0)) / np.real(np.vdot(sym[s], sym[s]))
        assert abs(beta[s].item() - bref) <= 1e-5 * abs(bref)
        yr = (y0 + noise[s]) / bref
        want = port.slice(qam, yr)
        diff = labels[s].cpu().numpy() != want
        dist = np.sort(np.abs(yr[:, None] - pts[None, :]) ** 2, axis=1)
        near = np.abs(dist[:, 0] - dist[:, 1]) <= 1e-4 * (dist[:, 0] + dist[:, 1])
        mism += int(diff.sum())
        ties += int((diff & near).sum())
    assert mism == ties  # fp32 receive vs fp64: only decision-boundary ties may differ
    assert not flagged.any()
    # zero beamformer -> flagged, labels 0xff
    z = torch.zeros_like(d.x)
    l2, b2, f2 = engine.dl_receive(H, z, st, qam=qam)
    engine.sync()
    assert f2.all() and (l2 == 0xFF).all()
