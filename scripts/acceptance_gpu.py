"""The reference's acceptance criteria (tests/acceptance.cpp) on the GPU path.
Criteria 3-6 (:180-291) run the GPU sweep driver with the reference's sweep
specs (users 8, B_c 32, C 4, 16-QAM, 1e6 bits per point, seeds 71/73).
Criteria 1, 2, 7, 8, 9 are their device analogues:
  1 (:111-139)  T=200 reaches the exact solvers (device Cholesky) — fp32 limit
                1e-5 instead of the fp64 1e-8;
  2 (:144-179)  a single-cluster decentralized call equals the cluster's own
                result (uplink bitwise, downlink fused power scaling vs a separate
                power_scale within fp32 rounding);
  7 (:296-353)  the interconnect byte model is exact (C in {1,4,8}, fp32/fp16,
                uniform/optimal);
  8 (:402-475)  invariants at sweep granularity (per-update observers cannot run
                on the GPU): the L-MMSE objective never increases from sweep to
                sweep, and the downlink beamformer stays in the channel's row
                space with the last-updated user's constraint zeroed;
  9 (:480-513)  per-cluster throughput at C=4 vs C=8 within 20%.
Prints the [PASS]/[FAIL] lines and writes a JSON summary.

    python scripts/acceptance_gpu.py [out.json]

The reference's own run of these criteria (this container, 8-core Xeon): UL gap
1.42 dB, DL gap 0.90 dB, fp16 gap 0.00 dB."""
import dataclasses
import json
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1902_08653_b200 import Engine  # noqa: E402
from paper_1902_08653_b200.harness import SweepSpec, curve_of, run_ber_sweep, snr_at_ber  # noqa: E402


def ber_at_snr(curve, snr):
    """acceptance.cpp:64-74: log-linear read-out inside the grid."""
    c = sorted(curve)
    for (s0, b0), (s1, b1) in zip(c, c[1:]):
        if s0 <= snr <= s1:
            if b0 <= 0.0 or b1 <= 0.0:
                return min(b0, b1)
            w = (snr - s0) / (s1 - s0)
            return math.exp((1.0 - w) * math.log(b0) + w * math.log(b1))
    return math.nan


def _rel(a, b):
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    return float(np.max(np.linalg.norm((a - b).reshape(a.shape[0], -1), axis=1) /
                        np.linalg.norm(b.reshape(b.shape[0], -1), axis=1)))


def criterion_1(eng):
    """100 instances, B=128 (one cluster), U=8, N0=0.1, T=200 vs the exact solvers."""
    S, BC, U = 100, 128, 8
    d = eng.synth(S, 1, BC, U, n0=0.1, seed=10000, uplink=True, downlink=True)
    H, y, sym = d["H"], d["y"], d["sym"]
    cd = eng.ul_detect(H, y, n0=0.1, K=200, want_local=False).xhat
    ex = eng.lmmse_exact(H, y, n0=0.1)
    cdp = eng.dl_precode(H, sym, rho=0.0, K=200, want_gain=False).x
    zf = eng.zf_exact(H, sym, rho=0.0)
    eng.sync()
    wu, wd = _rel(cd.cpu().numpy(), ex.cpu().numpy()), _rel(cdp.cpu().numpy(), zf.cpu().numpy())
    return {"pass": bool(wu <= 1e-5 and wd <= 1e-5), "worst_ul": wu, "worst_dl": wd, "limit_fp32": 1e-5}


def criterion_2(eng):
    """50 instances of one 32x8 cluster: decentralized == the cluster's own result."""
    S, BC, U = 50, 32, 8
    d = eng.synth(S, 1, BC, U, n0=0.2, seed=20000, uplink=True, downlink=True)
    H, y, sym = d["H"], d["y"], d["sym"]
    r = eng.ul_detect(H, y, n0=0.2, K=3)
    dl = eng.dl_precode(H, sym, rho=math.sqrt(8.0), K=3, want_gain=False).x
    raw = eng.dl_precode(H, sym, rho=0.0, K=3, want_gain=False).x
    eng.power_scale(raw, math.sqrt(8.0))
    eng.sync()
    ul_mis = int((torch.view_as_real(r.xhat) != torch.view_as_real(r.x_local[:, 0])).any(dim=-1).any(dim=-1).sum())
    dl_err = _rel(dl.cpu().numpy(), raw.cpu().numpy())
    return {"pass": bool(ul_mis == 0 and dl_err <= 1e-6), "ul_bitwise_mismatches": ul_mis, "dl_rel_vs_power_scale": dl_err}


def criterion_7(eng):
    """The MessageLog byte model over the GPU uplink (DistributedCD.traffic)."""
    from paper_1902_08653_b200 import to_fp16_pairs
    from paper_1902_08653_b200.distributed import CudaCompute, DistributedCD, partition
    U, S = 8, 300
    ok, notes = True, []
    for nc in (1, 4, 8):
        d = eng.synth(S, nc, 32, U, n0=0.5, seed=600 + nc)
        got = {}
        for fmt in ("fp32", "fp16"):
            H, y = (d["H"], d["y"]) if fmt == "fp32" else (to_fp16_pairs(d["H"]), to_fp16_pairs(d["y"]))
            for fusion in ("uniform", "optimal"):
                dcd = DistributedCD(partition(nc, 1, 0, S), CudaCompute(eng))
                dcd.uplink(H, y, n0=0.5, K=3, fusion=fusion)
                got[(fmt, fusion)] = dcd.traffic.uplink_payload_bytes
        want = {("fp32", "uniform"): nc * S * U * 8, ("fp16", "uniform"): nc * S * U * 4,
                ("fp32", "optimal"): nc * S * (U * 8 + 4), ("fp16", "optimal"): nc * S * (U * 4 + 2)}
        for k, v in want.items():
            if got[k] != v:
                ok = False
                notes.append(f"C={nc} {k}: {got[k]} != {v}")
        if got[("fp16", "uniform")] * 2 != got[("fp32", "uniform")]:
            ok = False
            notes.append(f"C={nc}: fp16 bytes not half of fp32")
    eng.sync()
    return {"pass": ok, "notes": notes or ["C in {1,4,8}, fp32/fp16, uniform/optimal exact"]}


def criterion_8(eng, instances=100):
    """Sweep-level invariants on random shapes u in 4..8, b in {4u, 5u, 6u}."""
    rng = np.random.default_rng(30000)
    desc_bad = row_bad = zero_bad = 0
    worst_zero = worst_row = 0.0
    for inst in range(instances):
        u = int(4 + rng.integers(0, 5))
        b = int(4 * u + rng.integers(0, 3) * u)
        d = eng.synth(1, 1, b, u, n0=0.2, seed=30000 + inst, uplink=True, downlink=True)
        H, y, sym = d["H"], d["y"], d["sym"]
        Hn = H[0, 0].cpu().numpy().astype(np.complex128).T          # b x u (column j = user j)
        yn = y[0, 0].cpu().numpy().astype(np.complex128)
        kappa = 0.2
        j_prev = float(np.vdot(yn, yn).real)
        for K in range(1, 7):
            x = eng.ul_detect(H, y, n0=kappa, K=K, want_local=False).xhat[0].cpu().numpy().astype(np.complex128)
            r = yn - Hn @ x
            j = float(np.vdot(r, r).real + kappa * np.vdot(x, x).real)
            if j > j_prev + 1e-6 * float(np.vdot(yn, yn).real):  # fp32 slack
                desc_bad += 1
            j_prev = j
        xd = eng.dl_precode(H, sym, rho=0.0, K=2, want_gain=False).x[0, 0].cpu().numpy().astype(np.complex128)
        # row space of H_dl = column space of the uplink block: x = Hn w
        w, *_ = np.linalg.lstsq(Hn, xd, rcond=None)
        row = float(np.linalg.norm(xd - Hn @ w) / np.linalg.norm(xd))
        worst_row = max(worst_row, row)
        row_bad += int(row > 1e-5)
        # the last user updated in the final sweep has its constraint zeroed:
        # h~_u^H x = s~_u with h~_u = h_u / ||h_u||, s~_u = s_u / ||h_u||
        hu = Hn[:, u - 1]
        su = sym[0, u - 1].item()
        zres = abs(np.vdot(hu, xd) - su) / max(abs(su), 1e-30)
        worst_zero = max(worst_zero, float(zres))
        zero_bad += int(zres > 1e-5)
    eng.sync()
    return {"pass": bool(desc_bad == 0 and row_bad == 0 and zero_bad == 0), "instances": instances,
            "descent_violations": desc_bad, "row_space_violations": row_bad, "zeroing_violations": zero_bad,
            "worst_row_space_rel": worst_row, "worst_zeroing_rel": worst_zero}


def criterion_9(eng, S=67200, reps=10):
    """per_cluster_rate (harness.cpp:357-358: subcarriers/s x clusters, i.e.
    cluster-problems/s) at C=4 vs C=8, 32x8 clusters.
    Both batches (0.6 / 1.2 GB) exceed the 126 MB L2, so repeated launches do
    not favour the smaller one."""
    rates = {}
    for nc in (4, 8):
        d = eng.synth(S, nc, 32, 8, n0=0.5, seed=77)
        fn = lambda: eng.ul_detect(d["H"], d["y"], n0=0.5, K=3, want_local=False)  # noqa: E731
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / reps * 1e-3
        rates[nc] = S / t * nc
    spread = abs(rates[4] - rates[8]) / max(rates[4], rates[8])
    return {"pass": bool(spread <= 0.2), "per_cluster_rate_c4": rates[4], "per_cluster_rate_c8": rates[8],
            "spread": spread, "subcarriers": S}


def criteria_3_to_5(eng):
    """Criteria 3-5 on the reference's sweep spec (acceptance.cpp:180-260):
    returns ({3: .., 4: .., 5: ..}, curves, points)."""
    results = {}
    ul = SweepSpec(direction="uplink", methods=("dcd", "exact", "mf"), users=8, cluster_size=32, clusters=4,
                   snr_db=(2, 3, 4, 5, 6, 7, 8), t_max=(3, 4), min_bits=1_000_000, seed=71)
    pts = run_ber_sweep(ul, eng)
    ul200 = dataclasses.replace(ul, methods=("dcd",), snr_db=(5, 6, 7), t_max=(200,))
    pts200 = run_ber_sweep(ul200, eng)
    dl = dataclasses.replace(ul, direction="downlink", methods=("dcd", "exact", "mf"), t_max=(3,))
    dpts = run_ber_sweep(dl, eng)

    curves = {"ul_dcd3": curve_of(pts, "dcd", 3), "ul_dcd4": curve_of(pts, "dcd", 4),
              "ul_exact": curve_of(pts, "exact", 0), "ul_mf": curve_of(pts, "mf", 0),
              "ul_dcd200": curve_of(pts200, "dcd", 200), "dl_dcd3": curve_of(dpts, "dcd", 3),
              "dl_exact": curve_of(dpts, "exact", 0), "dl_mf": curve_of(dpts, "mf", 0)}

    # 3: T=3 within 2 dB of the exact methods at BER 1e-3 (acceptance.cpp:225-239)
    ul_d, ul_e = snr_at_ber(curves["ul_dcd3"], 1e-3), snr_at_ber(curves["ul_exact"], 1e-3)
    dl_d, dl_e = snr_at_ber(curves["dl_dcd3"], 1e-3), snr_at_ber(curves["dl_exact"], 1e-3)
    gu, gd = ul_d - ul_e, dl_d - dl_e
    ok3 = all(map(math.isfinite, (gu, gd))) and -0.5 <= gu <= 2.0 and -0.5 <= gd <= 2.0
    results[3] = {"pass": ok3, "ul_dcd3_db": ul_d, "ul_exact_db": ul_e, "gap_ul_db": gu, "dl_dcd3_db": dl_d,
                  "dl_exact_db": dl_e, "gap_dl_db": gd}
    # 4: MF floors >= 1e-2 at the crossing SNR (acceptance.cpp:241-251)
    mu, md = ber_at_snr(curves["ul_mf"], ul_d), ber_at_snr(curves["dl_mf"], dl_d)
    ok4 = all(map(math.isfinite, (mu, md))) and mu >= 1e-2 and md >= 1e-2
    results[4] = {"pass": ok4, "ul_mf_ber": mu, "dl_mf_ber": md}
    # 5: uplink T=4 within 0.5 dB of T=200 (acceptance.cpp:253-260)
    c4, c200 = snr_at_ber(curves["ul_dcd4"], 1e-3), snr_at_ber(curves["ul_dcd200"], 1e-3)
    ok5 = math.isfinite(c4 - c200) and abs(c4 - c200) <= 0.5
    results[5] = {"pass": ok5, "t4_db": c4, "t200_db": c200, "gap_db": c4 - c200}
    return results, curves, pts + pts200 + dpts


def criterion_6(eng):
    """binary16 full-storage penalty <= 0.3 dB (acceptance.cpp:265-291); the
    fp16 'full' scope runs the half2 sweep kernels (fp16 arithmetic)."""
    s6 = SweepSpec(direction="uplink", methods=("dcd",), users=8, cluster_size=32, clusters=2,
                   snr_db=(6, 7, 8, 9, 10, 11, 12), t_max=(3,), min_bits=1_000_000, seed=73)
    c64 = snr_at_ber(curve_of(run_ber_sweep(s6, eng), "dcd", 3), 1e-3)
    c16 = snr_at_ber(curve_of(run_ber_sweep(dataclasses.replace(s6, precision="fp16", scope="full"), eng), "dcd", 3),
                     1e-3)
    ok6 = math.isfinite(c16 - c64) and c16 - c64 <= 0.3
    return {"pass": ok6, "fp16_db": c16, "fp64_db": c64, "gap_db": c16 - c64}


def main():
    eng = Engine(0)
    t0 = time.time()
    results, curves, all_pts = criteria_3_to_5(eng)
    t_main = time.time() - t0
    t1 = time.time()
    results[6] = criterion_6(eng)
    t6 = time.time() - t1

    t_other = time.time()
    results[1] = criterion_1(eng)
    results[2] = criterion_2(eng)
    results[7] = criterion_7(eng)
    results[8] = criterion_8(eng)
    results[9] = criterion_9(eng)
    t_other = time.time() - t_other

    names = {1: "oracle convergence at T=200 (fp32)", 2: "single-cluster equivalence",
             3: "T=3 within 2 dB of the exact methods at BER 1e-3",
             4: "matched filter floors 10x above 1e-3 at the crossing SNR",
             5: "uplink T=4 within 0.5 dB of full convergence", 6: "binary16 full-storage penalty at most 0.3 dB",
             7: "interconnect accounting is exact", 8: "sweep-level invariants hold on random instances",
             9: "per-cluster throughput stable across cluster counts"}
    for k in sorted(results):
        r = results[k]
        detail = ", ".join(f"{a}={v:.3g}" if isinstance(v, float) else f"{a}={v}" for a, v in r.items() if a != "pass")
        print(f"[{'PASS' if r['pass'] else 'FAIL'}] {k}: {names[k]} ({detail})")
    device_s = sum(p.seconds for p in all_pts)
    summary = {"criteria": results, "wall_s_criteria_3_5": t_main, "wall_s_criterion_6": t6,
               "wall_s_criteria_1_2_7_8_9": t_other,
               "device_s_criteria_3_5": device_s, "points": len(all_pts),
               "curves": curves,
               "reference_cpu_probe": {"acceptance_total_s": 273, "ul_gap_db": 1.42, "dl_gap_db": 0.90,
                                       "fp16_gap_db": 0.00, "source": "SURVEY.md §4 (criteria 1-9, 8-core host)"}}
    print(json.dumps({k: v for k, v in summary.items() if k != "curves"}))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(summary, f, indent=1)
    return 0 if all(r["pass"] for r in results.values()) else 1


if __name__ == "__main__":
    sys.exit(main())
