"""GPU: the per-update trace kernels behind SweepObserver (detect.hpp:28-36).

The reference hooks every coordinate update (detect.cpp:106 hands the
observer x and the maintained residual r, precode.cpp:95 x and no residual);
its DescentProbe and ZeroingProbe suites (tests/test_detect.cpp:149-200,
tests/test_precode.cpp:170-224) check per-update invariants.  Here the same
invariants are checked on the device traces with fp32 tolerances, and the
traces are checked against the oracle's per-update iterates (its cd_detect /
cd_precode stopped after every update count) and the batched kernels.
"""
import numpy as np
import pytest

from helpers import TOL_FP32, batch, qam_symbols, rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(32, 16), (16, 4), (24, 6), (64, 8)], ids=lambda s: f"Bc{s[0]}_U{s[1]}")
def test_uplink_trace_descends_and_keeps_the_residual(engine, port, shape):
    Bc, U = shape
    b = batch(1, Bc, U, S=2, seed=31)
    h = b["h_tiles"][0, 0]          # [U, Bc]: column j of the B_c x U block
    y = b["y"][0, 0]
    n0, K = b["n0"], 3
    xt, rt = engine.ul_trace(to_dev(h), to_dev(y), n0=n0, K=K)
    xt, rt = to_host(xt), to_host(rt)
    Hm = h.T                        # B_c x U
    kappa = n0
    j_prev = float(np.vdot(y, y).real)
    for e in range(K * U):
        x = xt[e]
        res = y - Hm @ x
        # the maintained residual equals y - H x (DescentProbe's second check)
        assert np.linalg.norm(res - rt[e]) <= 1e-5 * (1 + np.linalg.norm(y))
        # every update descends the L-MMSE objective
        j = float(np.vdot(res, res).real + kappa * np.vdot(x, x).real)
        assert j <= j_prev + 1e-5 * float(np.vdot(y, y).real)
        j_prev = j
        # the trace is the reference's iterate after this many updates
        t, jj = divmod(e, U)
        if jj == U - 1:
            want = port.cd_detect(Hm, y, n0, 1.0, t + 1)
            assert rel_err(x, want) <= TOL_FP32
    # and ends where the batched kernel ends
    r = engine.ul_detect(to_dev(b["h_tiles"][:1, :1]), to_dev(b["y"][:1, :1]), n0=n0, K=K)
    assert rel_err(xt[-1], to_host(r.x_local)[0, 0]) <= TOL_FP32


@pytest.mark.parametrize("shape", [(32, 16), (12, 3), (20, 7)], ids=lambda s: f"Bc{s[0]}_U{s[1]}")
def test_downlink_trace_zeroes_each_constraint(engine, port, shape):
    Bc, U = shape
    b = batch(1, Bc, U, S=2, seed=41)
    h = b["h_tiles"][0, 0]          # uplink tile [U, Bc]; H_dl = conj rows
    s = qam_symbols(1, U, seed=3)[0]
    K = 3
    xt = to_host(engine.dl_trace(to_dev(h), to_dev(s), K=K))
    Hdl = np.conj(h)                # U x B_c downlink block (precode.cpp:19-27)
    for e in range(K * U):
        u = e % U
        x = xt[e]
        # the updated user's constraint is zeroed (ZeroingProbe)
        nrm = np.linalg.norm(Hdl[u])
        assert abs(Hdl[u] @ x - s[u]) / nrm <= 1e-5 * (1 + abs(s[u]) / nrm)
        if u == U - 1:
            # sweep boundary: x in the row space of H_dl
            px = np.linalg.pinv(Hdl) @ (Hdl @ x)
            assert np.linalg.norm(x - px) <= 1e-5 * (1 + np.linalg.norm(x))
            want = port.cd_precode(Hdl, s, e // U + 1)
            assert rel_err(x, want) <= TOL_FP32
