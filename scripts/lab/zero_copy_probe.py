"""Lab: the CD kernels reading H, y straight from pinned (UVA-mapped) host
memory and writing their results to pinned host memory — one subcarrier per
call (the reference's per-call granularity), no cudaMemcpy: per-call latency
and bitwise agreement with the device-resident call."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from bench import make_inputs  # noqa: E402
from paper_1902_08653_b200 import Engine  # noqa: E402
from paper_1902_08653_b200._lib import lib, FP32, FUSION_UNIFORM  # noqa: E402

eng = Engine(0)
dev = torch.device("cuda", 0)
S, Cn, U, Bc = 1, 8, 16, 32
H, y, _, n0 = make_inputs(S, Cn, dev, 3)
Hh, yh = H.cpu().pin_memory(), y.cpu().pin_memory()
xl_h = torch.empty((S, Cn, U), dtype=torch.complex64).pin_memory()
xh_h = torch.empty((S, U), dtype=torch.complex64).pin_memory()
xl_d = torch.empty((S, Cn, U), dtype=torch.complex64, device=dev)
xh_d = torch.empty((S, U), dtype=torch.complex64, device=dev)
st = torch.cuda.current_stream(dev)
sp = C.c_void_p(st.cuda_stream)
L = lib()


def call(Hp, yp, xlp, xhp):
    rc = L.dcdg_ul_detect(eng._ctx, C.c_void_p(Hp), C.c_void_p(yp), S, Cn, Cn, Bc, U, 3, float(n0), 1.0, FP32,
                          FUSION_UNIFORM, C.c_void_p(xlp), None, C.c_void_p(xhp), None, sp)
    assert rc == 0, L.dcdg_last_error()


out = {}
call(H.data_ptr(), y.data_ptr(), xl_d.data_ptr(), xh_d.data_ptr())
call(Hh.data_ptr(), yh.data_ptr(), xl_h.data_ptr(), xh_h.data_ptr())
st.synchronize()
out["bitwise_equal"] = bool(torch.equal(xh_h, xh_d.cpu()) and torch.equal(xl_h, xl_d.cpu()))
for name, args in (("zero_copy", (Hh, yh, xl_h, xh_h)), ("device_resident", (H, y, xl_d, xh_d))):
    ts = []
    for _ in range(300):
        t0 = time.perf_counter()
        call(*(a.data_ptr() for a in args))
        st.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    out[name + "_us_median"] = round(ts[len(ts) // 2] * 1e6, 2)
print(json.dumps(out))
