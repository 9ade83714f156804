"""CPU: the oracle (plain-C restatement, oracle/dcd_oracle.c) reproduces every
golden vector that the UNMODIFIED reference produced (tests/golden/, generated
by tests/golden/make_golden.py through oracle/_ref/libdcdref.so with the
scalar kernel backend) — bit for bit, including the reference's exception
types and texts.  When the reference library itself is present it is
re-checked too."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import Oracle, available

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden():
    g = np.load(GOLD)
    return {k: g[k] for k in g.files}


@pytest.fixture(scope="module")
def golden_errs():
    with open(os.path.join(HERE, "golden", "golden_errors.json")) as f:
        return json.load(f)


def _compute(kind):
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "golden", "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    o = Oracle(kind)
    o.set_backend("scalar")
    return mg.compute(o)


@pytest.fixture(scope="module")
def port_results():
    return _compute("port")


def test_golden_backend_is_scalar(golden_errs):
    assert golden_errs["backend"] == "scalar"


def test_port_bit_exact_on_every_golden_array(golden, port_results):
    out, _ = port_results
    assert set(out) == set(golden)
    bad = [k for k in golden if not np.array_equal(golden[k], out[k])]
    assert not bad, f"oracle differs from the reference on: {bad[:10]}"


def test_port_reproduces_reference_errors(golden_errs, port_results):
    _, errs = port_results
    assert errs == golden_errs["errors"]


def test_known_answers_from_reference_tests(golden):
    """KATs quoted by the reference's own tests (test_kernels.cpp:77-106,
    test_precode.cpp:286-302, test_detect.cpp:249-288)."""
    o = Oracle("port")
    assert o.f16_bits_to_f64(o.f64_to_f16_bits(2049.0)) == 2048.0
    assert o.f16_bits_to_f64(o.f64_to_f16_bits(65520.0)) == np.inf
    assert o.f16_bits_to_f64(o.f64_to_f16_bits(2 ** -25)) == 0.0
    assert np.signbit(o.f16_bits_to_f64(o.f64_to_f16_bits(-0.0)))
    x = o.power_scale(np.array([3.0, 4.0j]), 2.0)
    assert abs(x[0] - 1.2) <= 1e-15 and abs(x[1] - 1.6j) <= 1e-15
    w = o.fusion_weights(np.array([1.0, 1.0, 2.0]))
    assert np.allclose(w, [0.4, 0.4, 0.2], rtol=1e-15, atol=0)


@pytest.mark.skipif(not available("reference"), reason="oracle/_ref not built (needs /root/reference)")
def test_reference_library_still_matches_golden(golden):
    out, _ = _compute("reference")
    bad = [k for k in golden if not np.array_equal(golden[k], out[k])]
    assert not bad, bad[:10]
