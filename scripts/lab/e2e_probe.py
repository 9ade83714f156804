"""Where the e2e step's time goes beyond the PCIe copy bound (lab):
bench.measure_e2e as is, plus the host-side cost of one chunk's enqueue."""
import os
import sys
import time
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1902_08653_b200 import Engine  # noqa: E402

dev = torch.device("cuda", 0)
S = 16800
eng = Engine(0)
H, y, x, n0 = bench.make_inputs(S, 8, dev, 1)
part = types.SimpleNamespace(S=S, S_local=S, own_lo=0, own_hi=S)
for rep in range(3):
    r = bench.measure_e2e(eng, None, part, H, y, n0, "uniform", 1, dev, 5, lambda: torch.cuda.synchronize(dev))
    print("e2e", r["ms_per_step"], "copy", r["h2d_copy_only_ms"], "frac", r["frac_of_copy_bound"], flush=True)
# host cost of the per-chunk calls with no pending copies
cs = S // 8
st = torch.cuda.Stream(dev)
with torch.cuda.stream(st):
    for _ in range(3):
        eng.ul_detect(H[:cs], y[:cs], n0=n0, K=3, want_local=False, stream=st)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(8):
        eng.ul_detect(H[i * cs:(i + 1) * cs], y[i * cs:(i + 1) * cs], n0=n0, K=3, want_local=False, stream=st)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
print("host enqueue of 8 chunk calls %.1f us, until done %.1f us" % ((t1 - t) * 1e6, (t2 - t) * 1e6))
# GPU time of one chunk call
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    e0.record(st)
    for i in range(8):
        eng.ul_detect(H[i * cs:(i + 1) * cs], y[i * cs:(i + 1) * cs], n0=n0, K=3, want_local=False, stream=st)
    e1.record(st)
torch.cuda.synchronize()
print("8 chunk calls on the GPU %.1f us" % (e0.elapsed_time(e1) * 1e3))
