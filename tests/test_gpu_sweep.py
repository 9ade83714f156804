"""GPU: the BER-sweep building blocks — device-side
synthesis, the matched-filter and exact baselines against the oracle, the
flagged-trial error rule, and the sweep driver's end-to-end behaviour."""
import math

import numpy as np
import pytest
import torch

from helpers import TOL_FP32, batch, qam_symbols, rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


def _stack_full(h_tiles_s):
    """[C, U, Bc] tiles of one subcarrier -> full B x U channel (rows stacked)."""
    return np.concatenate([t.T for t in h_tiles_s], axis=0)


# ---- synthesis -------------------------------------------------------------
def test_synth_statistics_and_model(engine, port):
    S, C, Bc, U, qam, n0 = 2000, 4, 32, 8, 16, 0.5
    b = engine.synth(S, C, Bc, U, qam=qam, n0=n0, seed=5, uplink=True, downlink=True)
    engine.sync()
    H = b["H"].cpu().numpy()
    assert abs(np.mean(np.abs(H) ** 2) - 1.0) < 0.01 and abs(np.mean(H)) < 0.01
    assert abs(np.mean(H.real ** 2) - 0.5) < 0.01 and abs(np.mean(H.real * H.imag)) < 0.01
    bits = b["bits"].cpu().numpy()
    assert set(np.unique(bits)) <= {0, 1} and abs(bits.mean() - 0.5) < 0.01
    # symbols are the Gray-QAM points of the MSB-first bit labels (modulate, mimo.cpp:124-139)
    bps = 4
    labels = (bits.reshape(S, U, bps) * (1 << np.arange(bps - 1, -1, -1))).sum(-1)
    pts = port.qam_points(qam)
    sym = b["sym"].cpu().numpy()
    assert np.allclose(sym, pts[labels], atol=1e-6)
    # y = H x + n with n ~ CN(0, n0)
    y = b["y"].cpu().numpy()
    hx = np.einsum("scub,su->scb", H, sym)
    noise = (y - hx).ravel()
    assert abs(np.mean(np.abs(noise) ** 2) - n0) < 0.02 * n0
    nd = b["noise_dl"].cpu().numpy()
    assert abs(np.mean(np.abs(nd) ** 2) - n0) < 0.05 * n0


def test_synth_is_deterministic_and_layout_independent(engine):
    kw = dict(qam=64, n0=0.2, seed=99, first_trial=(3 << 32) + 17)
    a = engine.synth(64, 4, 32, 16, **kw)
    b = engine.synth(64, 4, 32, 16, **kw)
    c = engine.synth(64, 1, 128, 16, **kw)  # centralized layout, same antennas
    d = engine.synth(64, 4, 32, 16, **{**kw, "first_trial": kw["first_trial"] + 1})
    engine.sync()
    assert torch.equal(a["H"], b["H"]) and torch.equal(a["y"], b["y"]) and torch.equal(a["bits"], b["bits"])
    full_a = a["H"].permute(0, 2, 1, 3).reshape(64, 16, 128)  # [S, U, B] rows in cluster order
    assert torch.equal(full_a, c["H"].reshape(64, 16, 128))
    assert torch.equal(a["y"].reshape(64, 128), c["y"].reshape(64, 128))
    assert torch.equal(a["H"][1:], d["H"][:-1])  # trial t+1 of run a is trial t of run d


# ---- baselines vs the oracle ---------------------------------------------------
def test_mf_detect_and_precode_match_oracle(engine, port):
    C, Bc, U, S = 4, 32, 8, 24
    b = batch(C, Bc, U, S=S, seed=41)
    x = engine.mf_detect(to_dev(b["h_tiles"]), to_dev(b["y"]))
    sym = qam_symbols(S, U)
    rho = math.sqrt(U)
    xd = engine.mf_precode(to_dev(b["h_tiles"]), to_dev(sym), rho=rho)
    engine.sync()
    ref = np.stack([port.mf_detect([b["h_tiles"][s, c].T for c in range(C)], [b["y"][s, c] for c in range(C)])
                    for s in range(S)])
    assert rel_err(to_host(x), ref) <= TOL_FP32
    refd = np.stack([port.mf_precode([b["h_tiles"][s, c].conj() for c in range(C)], sym[s], rho) for s in range(S)])
    assert rel_err(to_host(xd).reshape(S, -1), refd) <= TOL_FP32


@pytest.mark.parametrize("C,Bc,U", [(4, 32, 8), (8, 32, 16), (2, 64, 32), (3, 24, 6)])
def test_exact_solvers_match_oracle(engine, port, C, Bc, U):
    S = 24
    b = batch(C, Bc, U, S=S, seed=43, snr_db=8.0)
    x = engine.lmmse_exact(to_dev(b["h_tiles"]), to_dev(b["y"]), n0=b["n0"])
    sym = qam_symbols(S, U)
    rho = math.sqrt(U)
    xd = engine.zf_exact(to_dev(b["h_tiles"]), to_dev(sym), rho=rho)
    engine.sync()
    ref = np.stack([port.lmmse_exact(_stack_full(b["h_tiles"][s]), b["y"][s].ravel(), b["n0"], 1.0)
                    for s in range(S)])
    assert rel_err(to_host(x), ref) <= 1e-4  # fp32 Cholesky of a B x U Gram (condition-dependent)
    refd = np.stack([port.power_scale(port.zf_exact(_stack_full(b["h_tiles"][s]).conj().T, sym[s]), rho)
                     for s in range(S)])
    assert rel_err(to_host(xd).reshape(S, -1), refd) <= 1e-4


def test_zf_exact_rank_deficient_raises_reference_text(engine):
    from paper_1902_08653_b200 import NumericError
    b = batch(2, 32, 8, S=4, seed=3)
    h = b["h_tiles"].copy()
    h[1, :, 5, :] = h[1, :, 4, :]  # users 4 and 5 share a channel on subcarrier 1
    engine.zf_exact(to_dev(h), to_dev(qam_symbols(4, 8)), rho=1.0)
    with pytest.raises(NumericError, match="zf_exact: channel rows are rank deficient") as ei:
        engine.sync()
    assert ei.value.problem == 1


def test_flagged_labels_count_half_the_bits(engine):
    labels = torch.tensor([[0xFF, 3], [0, 0xFF]], dtype=torch.uint8, device="cuda")
    bits = torch.zeros((2, 2 * 4), dtype=torch.uint8, device="cuda")
    e = engine.bit_errors(labels, bits, qam=16)
    engine.sync()
    assert int(e.item()) == 2 + 2 + 2  # two flagged symbols x bps/2, label 3 = 0b0011 vs 0000


# ---- the sweep driver ----------------------------------------------------------
def test_sweep_uplink_orders_methods(engine):
    from paper_1902_08653_b200.harness import SweepSpec, curve_of, run_ber_sweep
    spec = SweepSpec(direction="uplink", methods=("dcd", "cd", "exact", "mf"), users=8, cluster_size=32,
                     clusters=4, snr_db=(4, 8), t_max=(3,), min_bits=200_000, seed=71)
    pts = run_ber_sweep(spec, engine)
    ber = {(p.method, p.snr_db): p.ber for p in pts}
    for s in (4, 8):
        assert ber[("exact", s)] <= ber[("dcd", s)] * 1.15 + 1e-4
        assert ber[("dcd", s)] < ber[("mf", s)]
    assert curve_of(pts, "dcd", 3)[1][1] < curve_of(pts, "dcd", 3)[0][1]
    assert all(p.bits >= 200_000 for p in pts)
    dcd = [p for p in pts if p.method == "dcd"][0]
    assert dcd.message_bytes == (200_000 + 31) // 32 * 4 * (8 * 16 + 1 * 8)  # U complex + sigma^2 per cluster


def test_sweep_downlink_flags_and_orders(engine):
    from paper_1902_08653_b200.harness import SweepSpec, run_ber_sweep
    spec = SweepSpec(direction="downlink", methods=("dcd", "exact", "mf"), users=8, cluster_size=32, clusters=4,
                     snr_db=(6,), t_max=(3,), min_bits=200_000, seed=72)
    pts = {p.method: p for p in run_ber_sweep(spec, engine)}
    assert pts["exact"].ber <= pts["dcd"].ber * 1.15 + 1e-4 < pts["mf"].ber
    assert pts["dcd"].flagged_trials == 0


def test_exact_beats_matched_filter_at_high_snr(engine):
    # test_harness.cpp:173-191
    from paper_1902_08653_b200.harness import SweepSpec, run_ber_sweep
    spec = SweepSpec(methods=("exact", "mf"), users=4, cluster_size=16, clusters=2, snr_db=(12.0,), min_bits=40000,
                     seed=9)
    pts = {p.method: p.ber for p in run_ber_sweep(spec, engine)}
    assert pts["exact"] < pts["mf"] and pts["mf"] > 1e-3


def test_downlink_zf_error_free_at_high_snr(engine):
    # test_harness.cpp:193-208
    from paper_1902_08653_b200.harness import SweepSpec, run_ber_sweep
    spec = SweepSpec(direction="downlink", methods=("exact",), users=4, cluster_size=32, clusters=1,
                     snr_db=(10.0, 30.0), min_bits=20000, seed=11)
    pts = run_ber_sweep(spec, engine)
    assert pts[1].ber <= pts[0].ber and pts[1].errors == 0 and pts[0].flagged_trials == 0


def test_sweeps_are_reproducible_to_the_csv_bytes(engine, tmp_path):
    # test_harness.cpp:140-171
    from paper_1902_08653_b200.harness import SweepSpec, run_ber_sweep
    spec = SweepSpec(methods=("dcd", "exact"), users=4, cluster_size=16, clusters=2, snr_db=(4.0, 8.0),
                     t_max=(2,), min_bits=20000, seed=5)
    a, b = tmp_path / "a.csv", tmp_path / "b.csv"
    r1, r2 = run_ber_sweep(spec, engine, str(a)), run_ber_sweep(spec, engine, str(b))
    assert [(p.errors, p.bits) for p in r1] == [(p.errors, p.bits) for p in r2]
    assert a.read_bytes() == b.read_bytes() and len(r1) == 4
    assert all(p.bits >= spec.min_bits for p in r1)


@pytest.mark.parametrize("direction", ["uplink", "downlink"])
def test_convergence_study_medians_shrink(engine, direction):
    # test_harness.cpp:242-262 (fp32 floor instead of fp64)
    from paper_1902_08653_b200.harness import SweepSpec, run_convergence_study
    spec = SweepSpec(direction=direction, users=8, cluster_size=32, clusters=1, snr_db=(8.0,), t_max=(6,),
                     min_bits=10000, seed=13)
    pts = run_convergence_study(spec, engine, instances=40)
    assert [p.t for p in pts] == list(range(1, 7))
    for i, p in enumerate(pts):
        assert 0.0 <= p.median <= p.p95
        if i:
            assert p.median <= pts[i - 1].median * (1 + 1e-6) + 2e-6
    assert pts[-1].median < 0.05 * pts[0].median
