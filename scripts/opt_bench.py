"""Time optimal-fusion uplink detection (CD + post_eq_variance + fusion) at the
north-star shape, fp32 and fp16: python scripts/opt_bench.py [S]
(set DCDG_LIB_PATH to compare builds)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_inputs  # noqa: E402
from paper_1902_08653_b200 import Engine, to_fp16_pairs  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 16800
eng = Engine(0)
H, y, x, n0 = make_inputs(S, 8, torch.device("cuda", 0), 1)
out = {"lib": os.environ.get("DCDG_LIB_PATH", "default")}
for fmt, Hh, yh in (("fp32", H, y), ("fp16", to_fp16_pairs(H), to_fp16_pairs(y))):
    for _ in range(3):
        r = eng.ul_detect(Hh, yh, n0=n0, K=3, fusion="optimal")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        r = eng.ul_detect(Hh, yh, n0=n0, K=3, fusion="optimal")
    e1.record()
    torch.cuda.synchronize()
    out[f"opt_{fmt}_ms"] = round(e0.elapsed_time(e1) / 10, 4)
    out[f"opt_{fmt}_sigma2_checksum"] = float(r.sigma2.double().sum())
eng.sync()
print(json.dumps(out))
