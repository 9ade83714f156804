"""Lab: optimal vs uniform fusion batch time across tile shapes (fp32)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from bench import make_inputs, _time_stream  # noqa: E402
from paper_1902_08653_b200 import Engine  # noqa: E402

eng = Engine(0)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
out = {}
for (C, Bc, U, S) in ((2, 32, 8, 16800), (8, 32, 16, 16800), (8, 16, 16, 16800), (4, 64, 16, 16800), (4, 32, 32, 8400)):
    H, y, _, n0 = make_inputs(S, C, dev, 5, u=U, bc=Bc)
    row = {"kernel": eng.kernel_name(0, Bc, U, 0)}
    for fu in ("uniform", "optimal"):
        fn = lambda: eng.ul_detect(H, y, n0=n0, K=3, fusion=fu)  # noqa: E731
        for _ in range(3):
            fn()
        row[fu + "_ms"] = round(_time_stream(fn, st, 10), 4)
    out[f"C{C}_Bc{Bc}_U{U}_S{S}"] = row
    del H, y
print(json.dumps(out, indent=0))
