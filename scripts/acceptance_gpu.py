"""Acceptance criteria 3-6 of the reference (tests/acceptance.cpp:180-291) on
the GPU sweep driver, with the reference's sweep specs (users 8, B_c 32, C 4,
16-QAM, 1e6 bits per point, seeds 71/73).  Prints the [PASS]/[FAIL] lines and
writes a JSON summary.

    python scripts/acceptance_gpu.py [out.json]

The reference's own run of these criteria (this container, 8-core Xeon): UL gap
1.42 dB, DL gap 0.90 dB, fp16 gap 0.00 dB."""
import dataclasses
import json
import math
import os
import sys
import time

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


def main():
    eng = Engine(0)
    results = {}
    t0 = time.time()
    ul = SweepSpec(direction="uplink", methods=("dcd", "exact", "mf"), users=8, cluster_size=32, clusters=4,
                   snr_db=(2, 3, 4, 5, 6, 7, 8), t_max=(3, 4), min_bits=1_000_000, seed=71)
    pts = run_ber_sweep(ul, eng)
    ul200 = dataclasses.replace(ul, methods=("dcd",), snr_db=(5, 6, 7), t_max=(200,))
    pts200 = run_ber_sweep(ul200, eng)
    dl = dataclasses.replace(ul, direction="downlink", methods=("dcd", "exact", "mf"), t_max=(3,))
    dpts = run_ber_sweep(dl, eng)
    t_main = time.time() - t0

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
    # 6: binary16 full-storage penalty <= 0.3 dB (acceptance.cpp:265-291)
    t1 = time.time()
    s6 = SweepSpec(direction="uplink", methods=("dcd",), users=8, cluster_size=32, clusters=2,
                   snr_db=(6, 7, 8, 9, 10, 11, 12), t_max=(3,), min_bits=1_000_000, seed=73)
    c64 = snr_at_ber(curve_of(run_ber_sweep(s6, eng), "dcd", 3), 1e-3)
    c16 = snr_at_ber(curve_of(run_ber_sweep(dataclasses.replace(s6, precision="fp16", scope="full"), eng), "dcd", 3),
                     1e-3)
    ok6 = math.isfinite(c16 - c64) and c16 - c64 <= 0.3
    results[6] = {"pass": ok6, "fp16_db": c16, "fp64_db": c64, "gap_db": c16 - c64}
    t6 = time.time() - t1

    names = {3: "T=3 within 2 dB of the exact methods at BER 1e-3",
             4: "matched filter floors 10x above 1e-3 at the crossing SNR",
             5: "uplink T=4 within 0.5 dB of full convergence", 6: "binary16 full-storage penalty at most 0.3 dB"}
    for k in (3, 4, 5, 6):
        r = results[k]
        detail = ", ".join(f"{a}={v:.3g}" for a, v in r.items() if a != "pass")
        print(f"[{'PASS' if r['pass'] else 'FAIL'}] {k}: {names[k]} ({detail})")
    device_s = sum(p.seconds for p in pts + pts200 + dpts)
    summary = {"criteria": results, "wall_s_criteria_3_5": t_main, "wall_s_criterion_6": t6,
               "device_s_criteria_3_5": device_s, "points": len(pts) + len(pts200) + len(dpts),
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
