"""Cost of the fused peer-memory exchange at the north-star shape on one GPU:
the window path (CD kernel with the exchange epilogue + owner fusion, world 1)
against the plain path (CD kernel + fusion), uplink and downlink, CUDA events.
usage: python scripts/xchg_bench.py [S] [reps] > profiles/…json"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_inputs  # noqa: E402
from paper_1902_08653_b200 import Engine, ExchangeWindow  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 16800
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
eng = Engine(0)
H, y, x, n0 = make_inputs(S, 8, dev, 1)
w = ExchangeWindow(eng, 1, 0, S=S, C_total=8, U=16)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = {"S": S, "problems": S * 8, "shape": "B_c=32 U=16 C=8 K=3 fp32"}
out["ul_plain_ms"] = timed(lambda: eng.ul_detect(H, y, n0=n0, K=3, want_local=False))
out["ul_window_ms"] = timed(lambda: w.ul_detect(H, y, c0=0, C_total=8, n0=n0, K=3))
rho = math.sqrt(16)
out["dl_plain_ms"] = timed(lambda: eng.dl_precode(H, x, rho=rho, K=3, want_gain=True))
out["dl_window_ms"] = timed(lambda: w.dl_precode(H, x, root=0, c0=0, C_total=8, rho=rho, K=3))
eng.sync()
a = eng.ul_detect(H, y, n0=n0, K=3, want_local=False).xhat
b = w.ul_detect(H, y, c0=0, C_total=8, n0=n0, K=3)
eng.sync()
out["ul_bitwise_equal"] = bool(torch.equal(torch.view_as_real(a), torch.view_as_real(b)))
out = {k: (round(v, 5) if isinstance(v, float) else v) for k, v in out.items()}
print(json.dumps(out))
