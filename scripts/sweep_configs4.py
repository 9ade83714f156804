"""BASELINE configs[4]: scaling sweep B in {128,256,512} x U in {16,32} x
C in {1,2,4,8}, 64-QAM, K=3, fp32, one GPU holding all C clusters.  For each
shape: UL and DL CD-kernel time, Gbps (S*U*log2(64)/t), batch latency
(kernel + fusion / gain) and fraction of the measured HBM roofline.  The
downlink needs B_c >= U (precode.cpp:147-151); infeasible shapes are reported
as such.  usage: python scripts/sweep_configs4.py [out.json] [U filter, e.g. 32]"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import peaks  # noqa: E402
from paper_1902_08653_b200 import Engine, kernel_name  # noqa: E402

BITS = 6  # 64-QAM
dev = torch.device("cuda", 0)
eng = Engine(0)
hbm, _ = peaks()
st = torch.cuda.current_stream()


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


rows = []
UF = [int(sys.argv[2])] if len(sys.argv) > 2 else (16, 32)
for B in (128, 256, 512):
    for U in UF:
        for C in (1, 2, 4, 8):
            Bc = B // C
            per = (Bc * U + Bc + U) * 8
            S = max(1024, int(400e6 / (C * per)) // 64 * 64)
            g = torch.Generator(device=dev)
            g.manual_seed(B * 100 + U * 10 + C)
            H = torch.randn((S, C, U, Bc), dtype=torch.complex64, device=dev, generator=g)
            y = torch.randn((S, C, Bc), dtype=torch.complex64, device=dev, generator=g)
            s = torch.randn((S, U), dtype=torch.complex64, device=dev, generator=g)
            n0 = U / 10 ** (15 / 10)
            row = {"B": B, "U": U, "C": C, "B_c": Bc, "S": S, "problems": S * C, "bytes_per_problem": per}
            k = timed(lambda: eng.ul_detect(H, y, n0=n0, K=3, want_xhat=False))
            lat = timed(lambda: eng.ul_detect(H, y, n0=n0, K=3))
            row["ul"] = {"kernel": kernel_name("ul", Bc, U, "fp32"), "kernel_ms": round(k, 4),
                         "batch_ms": round(lat, 4), "Gbps": round(S * U * BITS / (lat * 1e-3) / 1e9, 3),
                         "roofline_frac": round(S * C * per / (k * 1e-3) / 1e9 / hbm, 4)}
            if Bc >= U:
                k = timed(lambda: eng.dl_precode(H, s, rho=math.sqrt(U), K=3, want_gain=False))
                lat = timed(lambda: eng.dl_precode(H, s, rho=math.sqrt(U), K=3))
                row["dl"] = {"kernel": kernel_name("dl", Bc, U, "fp32"), "kernel_ms": round(k, 4),
                             "batch_ms": round(lat, 4), "Gbps": round(S * U * BITS / (lat * 1e-3) / 1e9, 3),
                             "roofline_frac": round(S * C * per / (k * 1e-3) / 1e9 / hbm, 4)}
            else:
                row["dl"] = "infeasible: B_c < U (local zero-forcing needs B_c >= U, precode.cpp:147-151)"
            eng.sync()
            rows.append(row)
            print(json.dumps(row), flush=True)
            del H, y, s
            torch.cuda.empty_cache()
out = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] != "-" else None
if out:
    json.dump({"peak_hbm_gbs": hbm, "fmt": "fp32", "K": 3, "qam": 64, "rows": rows}, open(out, "w"), indent=1)
