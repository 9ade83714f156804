"""Quick kernel timing at the north-star shape: achieved algorithmic GB/s of the
UL/DL CD kernels (fp32, fp16), alone and with the cross-cluster stage
(uniform fusion / effective gain).  usage: python scripts/kbench.py [S] [reps]"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_inputs  # noqa: E402
from paper_1902_08653_b200 import Engine, to_fp16, to_fp16_pairs  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 16800
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
eng = Engine(0)
H, y, x, n0 = make_inputs(S, 8, dev, 1)
out = {"lib": os.environ.get("DCDG_LIB_PATH", "default")}
for fmt in ("fp32", "fp16", "fp16sweep"):
    Hh, yh, xh = (H, y, x) if fmt == "fp32" else (to_fp16_pairs(H), to_fp16_pairs(y), to_fp16(x))
    if fmt != "fp32" and hasattr(eng, "set_fp16_algorithm"):
        eng.set_fp16_algorithm("sweep" if fmt == "fp16sweep" else "gram")
    esz = 8 if fmt == "fp32" else 4
    nbytes = S * 8 * (32 * 16 + 32 + 16) * esz
    for d in ("ul", "dl", "ul+fusion", "dl+gain"):
        def run():
            if d == "ul":
                eng.ul_detect(Hh, yh, n0=n0, K=3, want_xhat=False)
            elif d == "dl":
                eng.dl_precode(Hh, xh, rho=4.0, K=3, want_gain=False)
            elif d == "ul+fusion":
                eng.ul_detect(Hh, yh, n0=n0, K=3)
            else:
                eng.dl_precode(Hh, xh, rho=4.0, K=3)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[f"{d}_{fmt}"] = {"ms": round(ms, 4), "GBps": round(nbytes / ms / 1e6, 1), "frac": round(nbytes / ms / 1e6 / 6546.6, 3)}
eng.sync()
print(json.dumps(out))
