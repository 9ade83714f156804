"""Lab: configs[0] tile (B_c=32, U=8, C=2) kernel time at two batch sizes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from bench import make_inputs, peaks, alg_bytes_per_problem, _time_stream  # noqa: E402
from paper_1902_08653_b200 import Engine  # noqa: E402

eng = Engine(0)
dev = torch.device("cuda", 0)
hbm, _ = peaks()
out = {"lib": os.environ.get("DCDG_LIB_PATH", "default"), "kernel": eng.kernel_name(0, 32, 8, 0)}
for S in (16800, 67200):
    H, y, _, n0 = make_inputs(S, 2, dev, 77, u=8, bc=32)
    fn = lambda: eng.ul_detect(H, y, n0=n0, K=3, want_xhat=False)  # noqa: E731
    for _ in range(3):
        fn()
    ms = _time_stream(fn, torch.cuda.current_stream(dev), 20)
    out[f"S{S}_ms"] = round(ms, 5)
    out[f"S{S}_frac"] = round(S * 2 * alg_bytes_per_problem(32, 8, 8) / (ms * 1e-3) / 1e9 / hbm, 4)
print(json.dumps(out))
