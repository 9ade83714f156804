#!/usr/bin/env python
"""Generate the golden vectors that pin the CPU oracle (oracle/dcd_oracle.c).

Every array here is produced by the UNMODIFIED reference library — the
/root/reference/proj sources compiled by oracle/Makefile into
oracle/_ref/libdcdref.so — with its kernel table pinned to the scalar backend
(src/kernels/dispatch.cpp:63-69), which is the reference's bit-reproducibility
backend.  Run in the build container (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

Outputs tests/golden/golden.npz and tests/golden/golden_errors.json.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import (FP16, FP32, FP64, FULL_STORAGE, MESSAGES, OPTIMAL, UNIFORM, OracleError,  # noqa: E402
                           Oracle, reference_batch)


def compute(ref):
    """All golden cases through oracle `ref` (reference or port); deterministic."""
    out = {}
    errs = {}
    rng = np.random.default_rng(20250101)

    def cn(*shape):
        return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)

    # --- RNG streams (rng.cpp) and key derivation
    out["derive_seed"] = np.array([ref.derive_seed(m, p, i) for m in (0, 1, 12345, 2**63 + 7)
                                   for p in (1, 2, 3, 4) for i in (0, 1, 99, 2**40)], dtype=np.uint64)
    for kind, name in ((0, "uniform"), (1, "gaussian"), (2, "bits")):
        out[f"rng_{name}"] = ref.rng_draw(987654321, kind, 700)

    # --- binary16 conversion KATs (kernels_scalar.cpp:43-90, test_kernels.cpp:77-106)
    f16_in = np.array([0.0, -0.0, 1.0, 2049.0, 2049.0 + 2**-14, 2049.0 - 2**-14, 65504.0, 65519.99, 65520.0,
                       2**-24, 2**-25, 2**-25 * 1.0000001, 3 * 2**-26, 1e-8, 0.1, -0.3333333333333333,
                       np.pi, 1e5, np.inf, -np.inf, 6.1035156e-05, 6.0975552e-05, 5.9604645e-08, 0.99951171875,
                       0.999755859375, 1.00048828125] + list(rng.standard_normal(64) * 8.0))
    out["f16_in"] = f16_in
    out["f16_bits"] = np.array([ref.f64_to_f16_bits(x) for x in f16_in], dtype=np.uint16)
    out["f16_round"] = ref.round_precision(f16_in, FP16)
    out["f32_round"] = ref.round_precision(f16_in, FP32)

    # --- vector kernels (kernels_scalar.cpp:9-41)
    a, b = cn(37), cn(37)
    out["k_a"], out["k_b"] = a, b
    out["k_cdotc"] = np.array([ref.cdotc(a, b)])
    out["k_caxpy"] = ref.caxpy(0.3 - 1.7j, a, b)
    out["k_norm2sq"] = np.array([ref.norm2sq(a)])

    # --- system model: make_batch + uplink observation (cluster.cpp:80-105,142-145)
    h, bits = ref.make_batch(2, 4, 3, 16, 3, 77, 5)
    out["mb_h"], out["mb_bits"] = h, bits
    n0 = ref.snr_to_n0(6.0, 3, 1.0)
    out["mb_n0"] = np.array([n0])
    out["mb_y"] = np.stack([ref.uplink_observe(h[s], bits[s], 16, n0, 77, 5 + s)[0] for s in range(3)])
    out["qam4"], out["qam16"], out["qam64"] = ref.qam_points(4), ref.qam_points(16), ref.qam_points(64)
    ys = cn(200) * 1.5
    out["slice_y"] = ys
    out["slice16"] = ref.slice(16, ys).astype(np.int64)
    out["slice64"] = ref.slice(64, ys).astype(np.int64)
    tie = np.array([0.0 + 0.0j, 2 / np.sqrt(10) + 0j, 0 + 2j / np.sqrt(10)])  # exact decision-boundary ties
    out["slice_tie_y"], out["slice_tie16"] = tie, ref.slice(16, tie).astype(np.int64)

    # --- uplink (detect.cpp)
    shapes = [(32, 8), (16, 4), (24, 6), (64, 16), (8, 8)]
    for (B, U) in shapes:
        H = cn(B, U)
        y = cn(B)
        out[f"ul_h_{B}_{U}"], out[f"ul_y_{B}_{U}"] = H, y
        for (fmt, scope) in ((FP64, MESSAGES), (FP32, FULL_STORAGE), (FP16, FULL_STORAGE)):
            for K in (1, 3):
                out[f"cd_detect_{B}_{U}_{fmt}{scope}_{K}"] = ref.cd_detect(H, y, 0.3, 1.0, K, fmt, scope)
        out[f"lmmse_{B}_{U}"] = ref.lmmse_exact(H, y, 0.3, 1.0)
        out[f"pev_{B}_{U}"] = np.array([ref.post_eq_variance(H, 0.3, 1.0)])
        out[f"bias_{B}_{U}"] = ref.mmse_bias_factors(H, 0.3, 1.0)
        # downlink on the same block: H_dl = H^H (U x B)
        Hdl = H.conj().T
        s = cn(U)
        out[f"dl_s_{B}_{U}"] = s
        if B >= U:
            for (fmt, scope) in ((FP64, MESSAGES), (FP16, FULL_STORAGE)):
                for K in (1, 3):
                    out[f"cd_precode_{B}_{U}_{fmt}{scope}_{K}"] = ref.cd_precode(Hdl, s, K, fmt, scope)
            out[f"zf_{B}_{U}"] = ref.zf_exact(Hdl, s)
    out["fw_in"] = np.array([0.5, 1.5, 0.25, 2.0, 1e-3, 7.0])
    out["fw"] = ref.fusion_weights(out["fw_in"])
    x = cn(33)
    out["ps_in"] = x
    out["ps"] = ref.power_scale(x, 2.5)

    # --- decentralized wrappers: config-1 shape (B=64, U=8, C=2) and target (B=256, U=16, C=8)
    for (C, BC, U, S, tag) in ((2, 32, 8, 6, "c1"), (8, 32, 16, 3, "tgt"), (3, 8, 4, 4, "small")):
        b = reference_batch(C, BC, U, 16, S, 1234, 8.0, kind=ref.kind)
        out[f"dec_{tag}_h"], out[f"dec_{tag}_y"], out[f"dec_{tag}_x"] = b["h_tiles"], b["y"], b["x_true"]
        out[f"dec_{tag}_n0"] = np.array([b["n0"]])
        for fusion in (UNIFORM, OPTIMAL):
            for (fmt, scope) in ((FP64, MESSAGES), (FP16, MESSAGES), (FP16, FULL_STORAGE), (FP32, FULL_STORAGE)):
                xh, loc, s2 = ref.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, fusion, fmt, scope)
                key = f"dec_{tag}_ul_{fusion}_{fmt}{scope}"
                out[key + "_xhat"], out[key + "_local"] = xh, loc
                if fusion == OPTIMAL:
                    out[key + "_sigma2"] = s2
            xd, g = ref.dl_precode_batch(b["h_tiles"], b["x_true"], np.sqrt(U), 3)
            out[f"dec_{tag}_dl_x"], out[f"dec_{tag}_dl_gain"] = xd, g
            xd16, g16 = ref.dl_precode_batch(b["h_tiles"], b["x_true"], np.sqrt(U), 3, FP16, FULL_STORAGE)
            out[f"dec_{tag}_dl16_x"], out[f"dec_{tag}_dl16_gain"] = xd16, g16

    # --- error behaviour (exception type and text)
    def capture(name, fn):
        try:
            fn()
            errs[name] = None
        except OracleError as e:
            errs[name] = [e.kind, str(e)]

    Hz = cn(8, 2)
    Hz[:, 1] = 0
    capture("precode_zero_row", lambda: ref.cd_precode(Hz.conj().T, cn(2), 3))
    capture("detect_tmax0", lambda: ref.cd_detect(cn(8, 2), cn(8), 0.1, 1.0, 0))
    capture("detect_neg_n0", lambda: ref.cd_detect(cn(8, 2), cn(8), -0.1, 1.0, 3))
    capture("detect_ex0", lambda: ref.cd_detect(cn(8, 2), cn(8), 0.1, 0.0, 3))
    capture("pev_n0_0", lambda: ref.post_eq_variance(cn(8, 2), 0.0, 1.0))
    capture("fw_bad", lambda: ref.fusion_weights(np.array([1.0, 0.0])))
    capture("fw_empty", lambda: ref.fusion_weights(np.zeros(0)))
    capture("ps_zero", lambda: ref.power_scale(np.zeros(4, complex), 1.0))
    capture("ps_rho0", lambda: ref.power_scale(cn(4), 0.0))
    capture("dec_precode_undersized",
            lambda: ref.decentralized_cd_precode([cn(8, 32), cn(8, 32), cn(8, 4)], cn(8), 1.0, 3))
    capture("dec_detect_empty", lambda: ref.decentralized_cd_detect([], [], 0.1, 1.0, 3))

    # --- matched-filter baselines (detect.cpp:191-218, precode.cpp:171-202);
    # appended last so the earlier arrays keep their random draws
    mh = [cn(32, 8) for _ in range(4)]
    my = [cn(32) for _ in range(4)]
    ms = cn(8)
    out["mf_h"] = np.stack(mh)
    out["mf_y"] = np.stack(my)
    out["mf_s"] = ms
    out["mf_detect"] = ref.mf_detect(mh, my)
    out["mf_precode"] = ref.mf_precode([h.conj().T for h in mh], ms, np.sqrt(8))
    mz = [h.copy() for h in mh]
    for h in mz:
        h[:, 3] = 0
    capture("mf_zero_energy", lambda: ref.mf_detect(mz, my))
    capture("mf_zero_beamformer", lambda: ref.mf_precode([np.zeros((8, 32), complex)] + [h.conj().T for h in mh[1:]],
                                                          ms, 1.0))

    return out, errs


def main():
    ref = Oracle("reference")
    ref.set_backend("scalar")
    out, errs = compute(ref)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden_errors.json"), "w") as f:
        json.dump({"backend": ref.backend(), "errors": errs}, f, indent=1, sort_keys=True)
    print(f"wrote {len(out)} arrays, {len(errs)} error cases")


if __name__ == "__main__":
    main()
