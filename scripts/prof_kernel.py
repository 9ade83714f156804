"""Launch one CD-path kernel a few times for an ncu capture.
usage: python scripts/prof_kernel.py [ul|opt|dl|dlg|pev] [fp32|fp16] [reps] [S] [C B_c U]
Default shape: the north star (C=8, B_c=32, U=16, S=16800 -> 134 400 problems);
other shapes are synthesised on the device (dcdg_synth)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import make_inputs  # noqa: E402
from paper_1902_08653_b200 import Engine, to_fp16, to_fp16_pairs  # noqa: E402

direction = sys.argv[1] if len(sys.argv) > 1 else "ul"
fmt = sys.argv[2] if len(sys.argv) > 2 else "fp32"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
S = int(sys.argv[4]) if len(sys.argv) > 4 else 16800
dev = torch.device("cuda", 0)
eng = Engine(0)
if len(sys.argv) > 7:
    C, Bc, U = (int(v) for v in sys.argv[5:8])
    b = eng.synth(S, C, Bc, U, qam=16, n0=U / 10.0, seed=1, uplink=True, downlink=True)
    H, y, x, n0 = b["H"], b["y"], b["sym"], U / 10.0
else:
    U = 16
    H, y, x, n0 = make_inputs(S, 8, dev, 1)
if fmt == "fp16":
    H, y, x = to_fp16_pairs(H), to_fp16_pairs(y), to_fp16(x)
for _ in range(reps):
    if direction == "ul":
        eng.ul_detect(H, y, n0=n0, K=3, fusion="uniform", want_xhat=False)
    elif direction == "opt":  # optimal fusion: CD + post_eq_variance (fused at the north-star tile)
        eng.ul_detect(H, y, n0=n0, K=3, fusion="optimal", want_xhat=False)
    elif direction == "pev":
        eng.post_eq_variance(H, n0=n0)
    elif direction == "dlg":  # downlink with the effective-gain share
        eng.dl_precode(H, x, rho=math.sqrt(U), K=3, want_gain=True)
    else:
        eng.dl_precode(H, x, rho=math.sqrt(U), K=3, want_gain=False)
eng.sync()
torch.cuda.synchronize()
print("done", direction, fmt, eng.launches)
