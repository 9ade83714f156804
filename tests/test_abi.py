"""CPU: the C-ABI library (paper_1902_08653_b200/libdcdg.so) loads, exports
every entry point include/dcdg.h declares plus the C++ host API of
include/dcd_gpu.hpp, validates arguments with the reference's exception texts
before touching a device, and fails loudly (no CPU fallback) without a GPU."""
import ctypes as C
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

from paper_1902_08653_b200 import _lib  # noqa: E402
from paper_1902_08653_b200._lib import DCDG_EINVAL, FP16, FP32, FUSION_OPTIMAL, FUSION_UNIFORM  # noqa: E402

HEADER = os.path.join(ROOT, "include", "dcdg.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dcdg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_expected_surface():
    syms = declared_symbols()
    for s in ("dcdg_init", "dcdg_ul_detect", "dcdg_dl_precode", "dcdg_fuse", "dcdg_post_eq_variance",
              "dcdg_power_scale", "dcdg_fusion_weights", "dcdg_sync_status", "dcdg_convert"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_cpp_host_api_is_exported():
    out = subprocess.run(["nm", "-DC", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in ("dcd::gpu::cd_detect(", "dcd::gpu::decentralized_cd_detect(", "dcd::gpu::cd_precode(",
                 "dcd::gpu::decentralized_cd_precode(", "dcd::gpu::power_scale(", "dcd::gpu::post_eq_variance(",
                 "dcd::gpu::fusion_weights(", "dcd::gpu::DeviceBatch::detect(", "dcd::gpu::DeviceBatch::precode("):
        assert name in out, name


def test_abi_version():
    assert _lib.lib().dcdg_abi_version() == 1


def _err(rc, expect_code, text):
    assert rc == expect_code
    assert _lib.lib().dcdg_last_error().decode() == text


NULL = None
DUMMY = C.c_void_p(16)  # non-null pointer that is never dereferenced (validation fails first)


def ul(**kw):
    a = dict(ctx=NULL, H=DUMMY, y=DUMMY, S=4, C=2, C_total=2, Bc=32, U=8, K=3, n0=0.1, ex=1.0, fmt=FP32,
             fusion=FUSION_UNIFORM)
    a.update(kw)
    return _lib.lib().dcdg_ul_detect(a["ctx"], a["H"], a["y"], a["S"], a["C"], a["C_total"], a["Bc"], a["U"], a["K"],
                                     a["n0"], a["ex"], a["fmt"], a["fusion"], None, None, None, None, None)


def dl(**kw):
    a = dict(ctx=NULL, H=DUMMY, s=DUMMY, S=4, C=2, C_total=2, Bc=32, U=8, K=3, rho=1.0, fmt=FP32, x=DUMMY)
    a.update(kw)
    return _lib.lib().dcdg_dl_precode(a["ctx"], a["H"], a["s"], a["S"], a["C"], a["C_total"], a["Bc"], a["U"],
                                      a["K"], a["rho"], a["fmt"], a["x"], None, None, None)


def test_uplink_argument_errors_use_reference_texts():
    # detect.cpp:12-19,71-72,115-116,150-151 (texts pinned in tests/golden/golden_errors.json)
    _err(ul(K=0), DCDG_EINVAL, "cd_detect: need at least one sweep")
    _err(ul(n0=-0.1), DCDG_EINVAL, "detector: need N0 >= 0 and E_x > 0")
    _err(ul(ex=0.0), DCDG_EINVAL, "detector: need N0 >= 0 and E_x > 0")
    _err(ul(C=0), DCDG_EINVAL, "decentralized_cd_detect: no clusters")
    _err(ul(Bc=0), DCDG_EINVAL, "detector: empty channel matrix")
    _err(ul(fusion=FUSION_OPTIMAL, n0=0.0), DCDG_EINVAL, "post_eq_variance: need N0 > 0 and E_x > 0")
    _err(ul(fmt=FP16, Bc=31), DCDG_EINVAL, "dcdg: fp16 row-pair planar tiles need an even antenna count B_c")
    _err(ul(), DCDG_EINVAL, "dcdg: null context")  # valid arguments, no device context


def test_downlink_argument_errors_use_reference_texts():
    # precode.cpp:11-16,57-58,143-151,101-104
    _err(dl(Bc=4, U=8), DCDG_EINVAL,
         "decentralized_cd_precode: cluster 0 has 4 antennas for 8 users; local zero-forcing needs B_c >= U")
    _err(dl(K=0), DCDG_EINVAL, "cd_precode: need at least one sweep")
    _err(dl(rho=-1.0), DCDG_EINVAL, "power_scale: amplitude must be positive")
    _err(dl(C=0), DCDG_EINVAL, "decentralized_cd_precode: no clusters")


def test_power_scale_and_fusion_weight_errors():
    L = _lib.lib()
    _err(L.dcdg_power_scale(NULL, DUMMY, 1, 4, 0.0, FP32, None), DCDG_EINVAL, "power_scale: amplitude must be positive")
    _err(L.dcdg_power_scale(NULL, DUMMY, 1, 0, 1.0, FP32, None), DCDG_EINVAL, "power_scale: empty beamformer")
    _err(L.dcdg_fusion_weights(NULL, DUMMY, 1, 0, DUMMY, None), DCDG_EINVAL, "fusion_weights: no clusters")


def test_kernel_dispatch_table():
    assert _lib.kernel_name(0, 32, 16, FP32) == "ul_tmh_f32<32,16,8>"  # half of the tile in TMEM
    assert _lib.kernel_name(1, 32, 16, FP32) == "dl_reg_f32<32,16,8>"
    assert _lib.kernel_name(0, 32, 16, FP16) == "ul_reg_f16<32,16,4>"
    assert _lib.kernel_name(0, 32, 8, FP32) == "ul_reg_f32<32,8,4>"
    assert _lib.kernel_name(0, 24, 6, FP32) == "ul_generic_f32"
    assert _lib.kernel_name(1, 512, 32, FP16) == "dl_generic_f16"


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_a_device():
    from paper_1902_08653_b200 import CudaError, Engine
    assert _lib.lib().dcdg_device_count() == 0
    with pytest.raises(CudaError, match="no CPU fallback"):
        Engine(0)


def test_missing_library_fails_loudly():
    env = dict(os.environ, DCDG_LIB_PATH="/nonexistent/libdcdg.so")
    code = "import paper_1902_08653_b200._lib as l; l.lib()"
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True)
    assert r.returncode != 0 and "no CPU fallback" in r.stderr


def test_exchange_window_argument_errors_before_any_device_work():
    """dcdg_xwin_create / dcdg_ul_detect_xchg validate on the host (the fused
    cross-GPU exchange, include/dcdg.h)."""
    L = _lib.lib()
    w = C.c_void_p()
    _err(L.dcdg_xwin_create(None, 9, 0, 1024, C.byref(w)), DCDG_EINVAL,
         "dcdg_xwin_create: need 1 <= world <= 8 and 0 <= rank < world")
    _err(L.dcdg_xwin_create(None, 2, 2, 1024, C.byref(w)), DCDG_EINVAL,
         "dcdg_xwin_create: need 1 <= world <= 8 and 0 <= rank < world")
    _err(L.dcdg_xwin_create(None, 2, 0, 0, C.byref(w)), DCDG_EINVAL, "dcdg_xwin_create: empty window")
    dummy = C.c_void_p(16)
    _err(L.dcdg_ul_detect_xchg(None, None, dummy, dummy, 16, 4, 0, 8, 32, 16, 0, 1.0, 1.0, FP32, FUSION_UNIFORM,
                               dummy, None), DCDG_EINVAL, "cd_detect: need at least one sweep")
    _err(L.dcdg_ul_detect_xchg(None, None, dummy, dummy, 16, 4, 0, 8, 32, 16, 3, 1.0, 1.0, FP32, FUSION_UNIFORM,
                               dummy, None), DCDG_EINVAL, "dcdg_ul_detect_xchg: null exchange window")
