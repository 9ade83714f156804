"""CPU: host logic of the GPU sweep driver against the reference's own known
answers (tests/test_harness.cpp, tests/test_cluster.cpp:201-230) and the
oracle; no device calls."""
import math

import pytest

from paper_1902_08653_b200.harness import (SweepSpec, analytic_qam_ber, message_bytes_per_trial, snr_at_ber,
                                           snr_to_n0)


def q_func(x):
    return 0.5 * math.erfc(x / math.sqrt(2.0))


def test_analytic_qam_ber_closed_forms():
    # test_harness.cpp:45-58
    assert analytic_qam_ber(4, 4.0) == pytest.approx(q_func(2.0), rel=1e-12)
    for gamma in (2.0, 10.0, 40.0):
        a = math.sqrt(gamma / 5.0)
        want = 0.75 * q_func(a) + 0.5 * q_func(3 * a) - 0.25 * q_func(5 * a)
        assert analytic_qam_ber(16, gamma) == pytest.approx(want, rel=1e-12)
    assert analytic_qam_ber(16, 1e6) < 1e-12
    assert analytic_qam_ber(64, 10.0) > analytic_qam_ber(16, 10.0)
    with pytest.raises(ValueError):
        analytic_qam_ber(8, 1.0)


def test_snr_at_ber_log_interpolation():
    # test_harness.cpp:82-91
    curve = [(0.0, 1e-2), (2.0, 1e-4)]
    assert snr_at_ber(curve, 1e-3) == pytest.approx(1.0, rel=1e-12)
    assert snr_at_ber(curve, 1e-2) == pytest.approx(0.0, abs=1e-9)
    assert snr_at_ber(curve + [(4.0, 0.0)], 1e-3) == pytest.approx(1.0, rel=1e-12)
    assert math.isnan(snr_at_ber(curve, 1e-6))
    assert math.isnan(snr_at_ber([(0.0, 1e-2)], 1e-3))


@pytest.mark.parametrize("kw,msg", [
    (dict(min_bits=100), "min_bits must be at least 10000"),
    (dict(direction="downlink", users=8, cluster_size=4, min_bits=10000), "B_c >= U"),
    (dict(qam_order=32), "order must be 4, 16 or 64"),
    (dict(max_trials=0), r"max_trials must be in \[1, 2\^32-1\]"),
    (dict(t_max=(3, 0)), "T_max entries must be >= 1"),
    (dict(methods=()), "no methods selected"),
])
def test_spec_validation(kw, msg):
    # test_harness.cpp:103-128 (and SweepSpec::validate texts, harness.cpp:41-62)
    with pytest.raises(ValueError, match=msg):
        SweepSpec(**kw).validate()
    ok = SweepSpec(min_bits=10000)
    ok.validate()
    assert ok.antennas == 128


def test_interconnect_bytes_kat():
    # test_cluster.cpp:201-230: B=128, C=4, U=8, 1200 subcarriers
    kw = dict(users=8, cluster_size=32, clusters=4)
    assert 1200 * message_bytes_per_trial(SweepSpec(**kw, precision="fp32", fusion="uniform"), "dcd") == 307200
    assert 1200 * message_bytes_per_trial(SweepSpec(**kw, precision="fp16", fusion="uniform"), "dcd") == 153600
    assert (1200 * message_bytes_per_trial(SweepSpec(**kw, precision="fp32", fusion="optimal"), "dcd")
            == 307200 + 4 * 1200 * 4)
    # centralized methods forward B_c raw samples per cluster (cluster.cpp:176-186)
    assert message_bytes_per_trial(SweepSpec(**kw, precision="fp32"), "exact") == 4 * 32 * 8


def test_snr_to_n0_matches_oracle(port):
    for snr in (-3.0, 0.0, 7.5, 30.0):
        assert snr_to_n0(snr, 8, 1.0) == port.snr_to_n0(snr, 8, 1.0)
