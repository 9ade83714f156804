"""The reference's acceptance criteria 1, 2, 7, 8 and 9 (tests/acceptance.cpp,
device analogues in scripts/acceptance_gpu.py) as GPU tests; criteria 3-6 (BER
gaps) are covered by test_gpu_sweep.py and the acceptance script."""
import importlib.util
import os

import pytest

pytestmark = pytest.mark.gpu

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_spec = importlib.util.spec_from_file_location("acceptance_gpu", os.path.join(_ROOT, "scripts", "acceptance_gpu.py"))
acc = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(acc)


def test_criterion_1_convergence_to_the_exact_solvers(engine):
    r = acc.criterion_1(engine)
    assert r["pass"], r


def test_criterion_2_single_cluster_equivalence(engine):
    r = acc.criterion_2(engine)
    assert r["pass"], r


def test_criterion_7_message_accounting(engine):
    r = acc.criterion_7(engine)
    assert r["pass"], r


def test_criterion_8_sweep_level_invariants(engine):
    r = acc.criterion_8(engine, instances=30)
    assert r["pass"], r


def test_criterion_9_per_cluster_rate_stable(engine):
    r = acc.criterion_9(engine, S=33600, reps=5)
    assert r["pass"], r
