"""Batched device API over the dcdg C ABI (torch tensors are only device
memory and streams here).

Tensor conventions (device batch layout of include/dcdg.h):

  fp32:  torch.complex64   H [S, C, U, Bc], y [S, C, Bc], s [S, U]
  fp16:  torch.float16     H [S, C, U, Bc, 2], y [S, C, Bc, 2], s [S, U, 2]
         binary16 — the paper's half-precision path.  s, x_local and x are
         interleaved (re, im); the channel tiles H and receive vectors y are
         ROW-PAIR PLANAR along the antenna axis ({re_2i, re_2i+1, im_2i,
         im_2i+1}, include/dcdg.h): build them with ``to_fp16_pairs``.

Each tile H[s, c] is the cluster's B_c x U uplink block stored column by
column (one user column of B_c antennas after the other), i.e. the memory
order of dcd::ComplexMatrix (include/dcd/numerics.hpp:35-40).  The downlink
uses the same tiles (reciprocity, src/precode.cpp:19-27).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import FP16, FP32, FUSION_OPTIMAL, FUSION_UNIFORM, check, lib


def _fmt_of(t: torch.Tensor) -> int:
    if t.dtype == torch.complex64:
        return FP32
    if t.dtype == torch.float16 and t.shape[-1] == 2:
        return FP16
    if t.dtype == torch.complex32:
        return FP16
    raise TypeError(f"unsupported dtype {t.dtype} (need complex64, or float16 [...,2] for fp16)")


def _shape(t: torch.Tensor, fmt: int):
    return tuple(t.shape[:-1]) if (fmt == FP16 and t.dtype == torch.float16) else tuple(t.shape)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _need(t: torch.Tensor, what: str):
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (the CD path has no CPU implementation)")
    if not t.is_contiguous():
        raise ValueError(f"{what} must be contiguous")
    if t.data_ptr() % 16:
        raise ValueError(f"{what} must be 16-byte aligned")


def _fusion(f) -> int:
    if isinstance(f, int):
        return f
    return {"optimal": FUSION_OPTIMAL, "uniform": FUSION_UNIFORM}[f]


def complex_empty(shape, fmt: int, device) -> torch.Tensor:
    if fmt == FP32:
        return torch.empty(shape, dtype=torch.complex64, device=device)
    return torch.empty((*shape, 2), dtype=torch.float16, device=device)


def to_fp16(t: torch.Tensor) -> torch.Tensor:
    """complex64 -> float16 [..., 2] (RNE), on the tensor's device."""
    return torch.view_as_real(t).to(torch.float16).contiguous()


def to_fp16_pairs(t: torch.Tensor) -> torch.Tensor:
    """complex64 [..., B] -> float16 [..., B, 2] in the row-pair planar layout
    of fp16 channel tiles / receive vectors (B even)."""
    r = torch.view_as_real(t)
    shp = r.shape
    if shp[-2] % 2:
        raise ValueError("fp16 row-pair planar layout needs an even antenna count")
    r = r.reshape(*shp[:-2], shp[-2] // 2, 2, 2).transpose(-1, -2)
    return r.reshape(shp).to(torch.float16).contiguous()


def from_fp16_pairs(t: torch.Tensor) -> torch.Tensor:
    """Inverse of ``to_fp16_pairs`` (returns complex64)."""
    shp = t.shape
    r = t.float().reshape(*shp[:-2], shp[-2] // 2, 2, 2).transpose(-1, -2).reshape(shp)
    return torch.view_as_complex(r.contiguous())


def to_complex64(t: torch.Tensor) -> torch.Tensor:
    if t.dtype == torch.complex64:
        return t
    if t.dtype == torch.float16:
        return torch.view_as_complex(t.float().contiguous())
    return t.to(torch.complex64)


@dataclass
class UplinkResult:
    x_local: torch.Tensor | None
    xhat: torch.Tensor | None
    sigma2: torch.Tensor | None
    wsum: torch.Tensor | None


@dataclass
class DownlinkResult:
    x: torch.Tensor
    gain_part: torch.Tensor | None
    gain: torch.Tensor | None


class Engine:
    """One dcdg context bound to a CUDA device."""

    def __init__(self, device: int | None = None):
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        self.device = device
        self._ctx = C.c_void_p()
        check(lib().dcdg_init(device, C.byref(self._ctx)))

    def close(self):
        if self._ctx:
            lib().dcdg_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return int(lib().dcdg_launch_count(self._ctx))

    def set_fp16_algorithm(self, alg: str) -> None:
        """fp16 uplink kernel: "gram" (tensor-core Gram + fp32 sweeps in the
        U-dimensional space, default) or "sweep" (half2 residual sweeps, the
        paper's half-precision arithmetic).  See include/dcdg.h."""
        codes = {"sweep": _lib.ALG_SWEEP, "gram": _lib.ALG_GRAM}
        if alg not in codes:
            raise ValueError(f"unknown fp16 algorithm {alg!r}")
        check(lib().dcdg_set_fp16_algorithm(self._ctx, codes[alg]))
        self._fp16_alg = alg

    @property
    def fp16_algorithm(self) -> str:
        return getattr(self, "_fp16_alg", "gram")

    def kernel_name(self, direction: int, bc: int, u: int, fmt: int) -> str:
        """Kernel this context dispatches a (direction, B_c, U, fmt) batch to."""
        buf = C.create_string_buffer(96)
        check(lib().dcdg_ctx_kernel_name(self._ctx, direction, bc, u, fmt, buf, 96))
        return buf.value.decode()

    def _stream(self, stream):
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        return C.c_void_p(stream.cuda_stream)

    def sync(self, stream=None):
        """Wait for the stream; raise the first recorded numerical error."""
        check(lib().dcdg_sync_status(self._ctx, self._stream(stream)))

    # ------------------------------------------------------------------ uplink
    def ul_detect(self, H, y, *, n0: float, ex: float = 1.0, K: int = 3, fusion="uniform", C_total=None,
                  want_local: bool = True, want_xhat: bool = True, x_local=None, sigma2=None, xhat=None,
                  stream=None) -> UplinkResult:
        fmt = _fmt_of(H)
        S, Cn, U, Bc = _shape(H, fmt)
        if _shape(y, fmt) != (S, Cn, Bc) or _fmt_of(y) != fmt:
            raise ValueError("detector: observation length must match antenna count")
        _need(H, "H")
        _need(y, "y")
        C_total = Cn if C_total is None else C_total
        fu = _fusion(fusion)
        dev = H.device
        if x_local is None and want_local:
            x_local = complex_empty((S, Cn, U), fmt, dev)
        if fu == FUSION_OPTIMAL and sigma2 is None:
            sigma2 = torch.empty((S, Cn), dtype=torch.float32, device=dev)
        if xhat is None and want_xhat:
            xhat = torch.empty((S, U), dtype=torch.complex64, device=dev)
        wsum = None
        if want_xhat and fu == FUSION_OPTIMAL and C_total > Cn:
            wsum = torch.empty((S,), dtype=torch.float32, device=dev)
        check(lib().dcdg_ul_detect(self._ctx, _ptr(H), _ptr(y), S, Cn, C_total, Bc, U, K, float(n0), float(ex), fmt,
                                   fu, _ptr(x_local), _ptr(sigma2), _ptr(xhat), _ptr(wsum), self._stream(stream)))
        return UplinkResult(x_local, xhat, sigma2, wsum)

    def ul_trace(self, H, y, *, n0: float, ex: float = 1.0, K: int = 3, stream=None):
        """Per-update iterates of ONE problem (the SweepObserver debug path,
        detect.hpp:28-36): H [U, Bc] / y [Bc] (or [1,1,...] batches of one) ->
        (x [K*U, U], r [K*U, Bc]) complex64, entry t*U + j after update (t, j)."""
        fmt = _fmt_of(H)
        U, Bc = _shape(H, fmt)[-2:]
        _need(H, "H")
        _need(y, "y")
        xt = torch.empty((K * U, U), dtype=torch.complex64, device=H.device)
        rt = torch.empty((K * U, Bc), dtype=torch.complex64, device=H.device)
        check(lib().dcdg_ul_trace(self._ctx, _ptr(H), _ptr(y), Bc, U, K, float(n0), float(ex), fmt, _ptr(xt),
                                  _ptr(rt), self._stream(stream)))
        return xt, rt

    def dl_trace(self, H, s, *, K: int = 3, stream=None):
        """Per-update beamformers of ONE problem (precode.cpp:95): H [U, Bc],
        s [U] -> x [K*U, Bc] complex64 (unscaled, as cd_precode)."""
        fmt = _fmt_of(H)
        U, Bc = _shape(H, fmt)[-2:]
        _need(H, "H")
        _need(s, "s")
        xt = torch.empty((K * U, Bc), dtype=torch.complex64, device=H.device)
        check(lib().dcdg_dl_trace(self._ctx, _ptr(H), _ptr(s), Bc, U, K, fmt, _ptr(xt), self._stream(stream)))
        return xt

    def post_eq_variance(self, H, *, n0: float, ex: float = 1.0, out=None, stream=None):
        fmt = _fmt_of(H)
        S, Cn, U, Bc = _shape(H, fmt)
        _need(H, "H")
        if out is None:
            out = torch.empty((S, Cn), dtype=torch.float32, device=H.device)
        check(lib().dcdg_post_eq_variance(self._ctx, _ptr(H), S * Cn, Bc, U, float(n0), float(ex), fmt, _ptr(out),
                                          self._stream(stream)))
        return out

    def fuse(self, x_local, sigma2=None, *, fusion="uniform", C_total=None, xhat=None, wsum=None, stream=None):
        fmt = _fmt_of(x_local)
        S, Cn, U = _shape(x_local, fmt)
        C_total = Cn if C_total is None else C_total
        if xhat is None:
            xhat = torch.empty((S, U), dtype=torch.complex64, device=x_local.device)
        check(lib().dcdg_fuse(self._ctx, _ptr(x_local), _ptr(sigma2), S, Cn, C_total, U, fmt, _fusion(fusion),
                              _ptr(xhat), _ptr(wsum), self._stream(stream)))
        return xhat

    def fuse_finalize(self, xhat, wsum, stream=None):
        S, U = xhat.shape
        check(lib().dcdg_fuse_finalize(self._ctx, _ptr(xhat), _ptr(wsum), S, U, self._stream(stream)))
        return xhat

    def fusion_weights(self, sigma2, stream=None):
        S, Cn = sigma2.shape
        w = torch.empty_like(sigma2)
        check(lib().dcdg_fusion_weights(self._ctx, _ptr(sigma2), S, Cn, _ptr(w), self._stream(stream)))
        return w

    # ---------------------------------------------------------------- downlink
    def dl_precode(self, H, s, *, rho: float, K: int = 3, C_total=None, want_gain: bool = True, x=None,
                   gain_part=None, gain=None, stream=None) -> DownlinkResult:
        fmt = _fmt_of(H)
        S, Cn, U, Bc = _shape(H, fmt)
        if _shape(s, fmt) != (S, U) or _fmt_of(s) != fmt:
            raise ValueError("precoder: symbol count must match user count")
        _need(H, "H")
        _need(s, "s")
        C_total = Cn if C_total is None else C_total
        dev = H.device
        if x is None:
            x = complex_empty((S, Cn, Bc), fmt, dev)
        if want_gain and gain_part is None:
            gain_part = torch.empty((S, Cn), dtype=torch.float32, device=dev)
        if want_gain and gain is None and Cn == C_total:
            gain = torch.empty((S,), dtype=torch.float32, device=dev)
        check(lib().dcdg_dl_precode(self._ctx, _ptr(H), _ptr(s), S, Cn, C_total, Bc, U, K, float(rho), fmt, _ptr(x),
                                    _ptr(gain_part), _ptr(gain), self._stream(stream)))
        return DownlinkResult(x, gain_part, gain)

    def power_scale(self, x, rho: float, stream=None):
        fmt = _fmt_of(x)
        shp = _shape(x, fmt)
        n = shp[-1]
        P = math.prod(shp[:-1]) if len(shp) > 1 else 1
        check(lib().dcdg_power_scale(self._ctx, _ptr(x), P, n, float(rho), fmt, self._stream(stream)))
        return x

    def gain_reduce(self, gain_part, s, stream=None):
        fmt = _fmt_of(s)
        S, U = _shape(s, fmt)
        Cn = gain_part.shape[1]
        g = torch.empty((S,), dtype=torch.float32, device=s.device)
        check(lib().dcdg_gain_reduce(self._ctx, _ptr(gain_part), _ptr(s), S, Cn, U, fmt, _ptr(g), self._stream(stream)))
        return g

    # ------------------------------------------------------- hard decisions
    def mmse_bias(self, H, *, n0: float, ex: float = 1.0, stream=None):
        """Full-H MMSE bias factors beta [S, U] (mmse_bias_factors) of subcarriers
        whose C cluster tiles H[s, :] are all on this GPU."""
        fmt = _fmt_of(H)
        S, Cn, U, Bc = _shape(H, fmt)
        _need(H, "H")
        beta = torch.empty((S, U), dtype=torch.float32, device=H.device)
        check(lib().dcdg_mmse_bias(self._ctx, _ptr(H), S, Cn, Bc, U, float(n0), float(ex), fmt, _ptr(beta),
                                   self._stream(stream)))
        return beta

    def slice(self, x, beta=None, *, qam: int = 16, ex: float = 1.0, stream=None):
        """Gray-QAM labels of x / beta (Constellation::slice), uint8, x's shape."""
        fmt = _fmt_of(x)
        shp = _shape(x, fmt)
        n = math.prod(shp)
        labels = torch.empty(shp, dtype=torch.uint8, device=x.device)
        if beta is not None and beta.numel() != n:
            raise ValueError("beta must have one factor per symbol")
        check(lib().dcdg_slice(self._ctx, _ptr(x), fmt, _ptr(beta), n, qam, float(ex), _ptr(labels),
                               self._stream(stream)))
        return labels

    def bit_errors(self, labels, bits, *, qam: int = 16, stream=None) -> torch.Tensor:
        """Device counter (int64 tensor of 1) of bit errors vs MSB-first bits."""
        n = labels.numel()
        errs = torch.zeros((1,), dtype=torch.int64, device=labels.device)
        check(lib().dcdg_bit_errors(self._ctx, _ptr(labels.contiguous()), _ptr(bits.contiguous()), n, qam,
                                    _ptr(errs), self._stream(stream)))
        return errs

    def dl_receive(self, H, x, s, noise=None, *, qam: int = 16, ex: float = 1.0, stream=None):
        """(labels [S, U] uint8 (0xff where flagged), beta [S], flagged [S] bool)."""
        fmt = _fmt_of(H)
        S, Cn, U, Bc = _shape(H, fmt)
        dev = H.device
        labels = torch.empty((S, U), dtype=torch.uint8, device=dev)
        beta = torch.empty((S,), dtype=torch.float32, device=dev)
        flagged = torch.empty((S,), dtype=torch.uint8, device=dev)
        check(lib().dcdg_dl_receive(self._ctx, _ptr(H), _ptr(x), _ptr(s), _ptr(noise), S, Cn, Bc, U, fmt, qam,
                                    float(ex), _ptr(labels), _ptr(beta), _ptr(flagged), self._stream(stream)))
        return labels, beta, flagged.bool()

    def uplink_round(self, H, y, bits, *, n0: float, ex: float = 1.0, K: int = 3, fusion="uniform", qam: int = 16,
                     stream=None):
        """A device-resident run_uplink_round for the decentralized method
        (src/cluster.cpp:160-206): detect + fuse, unbias with the full-H
        factors, slice, count bit errors.  Returns (xhat, labels, errors)."""
        r = self.ul_detect(H, y, n0=n0, ex=ex, K=K, fusion=fusion, want_local=False, stream=stream)
        beta = self.mmse_bias(H, n0=n0, ex=ex, stream=stream) if n0 > 0 else None
        labels = self.slice(r.xhat, beta, qam=qam, ex=ex, stream=stream)
        return r.xhat, labels, self.bit_errors(labels, bits, qam=qam, stream=stream)

    # ---- BER-sweep building blocks (fp32) ----------------------------------
    def synth(self, S: int, C: int, Bc: int, U: int, *, qam: int = 16, ex: float = 1.0, n0: float = 0.0,
              seed: int = 1, first_trial: int = 0, uplink: bool = True, downlink: bool = False, stream=None):
        """Device-side batch synthesis (dcdg_synth): returns a dict with
        H [S, C, U, Bc] complex64, bits [S, U*log2(qam)] uint8, and
        y [S, C, Bc] (uplink) / sym [S, U] + noise_dl [S, U] (downlink)."""
        dev = self.device
        bps = {4: 2, 16: 4, 64: 6}.get(qam, 0)
        out = {"H": torch.empty((S, C, U, Bc), dtype=torch.complex64, device=dev),
               "bits": torch.empty((S, U * max(bps, 1)), dtype=torch.uint8, device=dev)}
        out["y"] = torch.empty((S, C, Bc), dtype=torch.complex64, device=dev) if uplink else None
        out["sym"] = torch.empty((S, U), dtype=torch.complex64, device=dev) if downlink else None
        out["noise_dl"] = torch.empty((S, U), dtype=torch.complex64, device=dev) if downlink else None
        check(lib().dcdg_synth(self._ctx, S, C, Bc, U, qam, float(ex), float(n0), int(seed) & (2**64 - 1),
                               int(first_trial) & (2**64 - 1), _ptr(out["H"]), _ptr(out["y"]), _ptr(out["bits"]),
                               _ptr(out["sym"]), _ptr(out["noise_dl"]), self._stream(stream)))
        return out

    def mf_detect(self, H, y, stream=None):
        """Matched-filter estimates [S, U] complex64 (mf_detect, detect.cpp:191-218)."""
        _need(H, "H")
        S, Cn, U, Bc = H.shape
        x = torch.empty((S, U), dtype=torch.complex64, device=H.device)
        check(lib().dcdg_mf_detect(self._ctx, _ptr(H), _ptr(y), S, Cn, Bc, U, _ptr(x), self._stream(stream)))
        return x

    def mf_precode(self, H, s, *, rho: float, stream=None):
        """Matched-filter beamformer [S, C, Bc] (mf_precode, precode.cpp:171-202)."""
        _need(H, "H")
        S, Cn, U, Bc = H.shape
        x = torch.empty((S, Cn, Bc), dtype=torch.complex64, device=H.device)
        check(lib().dcdg_mf_precode(self._ctx, _ptr(H), _ptr(s), S, Cn, Bc, U, float(rho), _ptr(x),
                                    self._stream(stream)))
        return x

    def lmmse_exact(self, H, y, *, n0: float, ex: float = 1.0, stream=None):
        """Exact full-channel L-MMSE estimates [S, U] (lmmse_exact, detect.cpp:54-65)."""
        _need(H, "H")
        S, Cn, U, Bc = H.shape
        x = torch.empty((S, U), dtype=torch.complex64, device=H.device)
        check(lib().dcdg_lmmse_exact(self._ctx, _ptr(H), _ptr(y), S, Cn, Bc, U, float(n0), float(ex), _ptr(x),
                                     self._stream(stream)))
        return x

    def zf_exact(self, H, s, *, rho: float, stream=None):
        """Exact min-norm ZF beamformer scaled to rho (zf_exact + power_scale,
        precode.cpp:31-50,101-111; rho == 0: raw), [S, C, Bc]."""
        _need(H, "H")
        S, Cn, U, Bc = H.shape
        x = torch.empty((S, Cn, Bc), dtype=torch.complex64, device=H.device)
        check(lib().dcdg_zf_exact(self._ctx, _ptr(H), _ptr(s), S, Cn, Bc, U, float(rho), _ptr(x),
                                  self._stream(stream)))
        return x

    def round_fp16(self, t, stream=None):
        """In-place binary16 rounding of an fp32/complex64 tensor (wire format)."""
        n = t.numel() * (2 if t.is_complex() else 1)
        check(lib().dcdg_round_fp16(self._ctx, _ptr(t), n, self._stream(stream)))
        return t


class ExchangeWindow:
    """This rank's window of the fused cross-GPU uplink exchange (include/dcdg.h,
    dcdg_xwin_*): the CD kernel stores each cluster estimate straight into the
    window of the GPU that owns the subcarrier (peer memory, CUDA IPC) and the
    owner fuses in ascending cluster order once every rank has published the
    batch.  ``handle()`` bytes go to the peers (any transport); ``open(peer,
    handle)`` maps theirs."""

    def __init__(self, eng: Engine, world: int, rank: int, *, S: int, C_total: int, U: int, fmt: str = "fp32",
                 optimal: bool = True):
        self.eng, self.world, self.rank = eng, world, rank
        if S % world:
            raise ValueError(f"batch of {S} subcarriers must divide over {world} GPUs")
        esz = 8 if fmt == "fp32" else 4
        s_own = S // world
        ul = ((s_own * C_total * U * esz + 255) // 256) * 256 + (s_own * C_total * 4 if optimal else 0)
        dl = ((S * U * esz + 255) // 256) * 256 + S * C_total * 4
        nbytes = max(ul, dl)
        self._w = C.c_void_p()
        check(lib().dcdg_xwin_create(eng._ctx, world, rank, nbytes, C.byref(self._w)))

    def handle(self) -> bytes:
        buf = C.create_string_buffer(_lib.XWIN_HANDLE_BYTES)
        check(lib().dcdg_xwin_handle(self._w, buf))
        return buf.raw

    def open(self, peer: int, handle: bytes):
        if len(handle) != _lib.XWIN_HANDLE_BYTES:
            raise ValueError("exchange-window handle has the wrong size")
        check(lib().dcdg_xwin_open(self._w, peer, C.c_char_p(handle)))

    def set_timeout(self, seconds: float):
        check(lib().dcdg_xwin_set_timeout(self._w, int(seconds * 1e9)))

    def close(self):
        if self._w:
            lib().dcdg_xwin_destroy(self._w)
            self._w = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def ul_detect(self, H, y, *, c0: int, C_total: int, n0: float, ex: float = 1.0, K: int = 3, fusion="uniform",
                  xhat=None, stream=None) -> torch.Tensor:
        """This rank's clusters [c0, c0 + C) over all S subcarriers -> the fused
        estimates [S/world, U] of the subcarriers it owns."""
        fmt = _fmt_of(H)
        S, Cn, U, Bc = _shape(H, fmt)
        if _shape(y, fmt) != (S, Cn, Bc) or _fmt_of(y) != fmt:
            raise ValueError("detector: observation length must match antenna count")
        _need(H, "H")
        _need(y, "y")
        if xhat is None:
            xhat = torch.empty((S // self.world, U), dtype=torch.complex64, device=H.device)
        check(lib().dcdg_ul_detect_xchg(self.eng._ctx, self._w, _ptr(H), _ptr(y), S, Cn, c0, C_total, Bc, U, K,
                                        float(n0), float(ex), fmt, _fusion(fusion), _ptr(xhat),
                                        self.eng._stream(stream)))
        return xhat


    def dl_precode(self, H, s, *, root: int = 0, c0: int, C_total: int, rho: float, K: int = 3, want_gain=True,
                   x=None, stream=None):
        """This rank's clusters [c0, c0 + C) over all S subcarriers; `s` [S, U]
        is read on the root only (the centre's symbols).  Returns (x_dl
        [S, C, Bc], effective gain [S] or None) on every rank."""
        fmt = _fmt_of(H)
        S, Cn, U, Bc = _shape(H, fmt)
        _need(H, "H")
        if self.rank == root:
            if s is None or _shape(s, fmt) != (S, U) or _fmt_of(s) != fmt:
                raise ValueError("precoder: symbol vector length must match the users")
            _need(s, "s")
        if x is None:
            x = complex_empty((S, Cn, Bc), fmt, H.device)
        gain = torch.empty((S,), dtype=torch.float32, device=H.device) if want_gain else None
        check(lib().dcdg_dl_precode_xchg(self.eng._ctx, self._w, root, _ptr(H), _ptr(s if self.rank == root else None),
                                         S, Cn, c0, C_total, Bc, U, K, float(rho), fmt, _ptr(x), _ptr(gain),
                                         self.eng._stream(stream)))
        return x, gain


def kernel_name(direction: str, bc: int, u: int, fmt: str) -> str:
    return _lib.kernel_name(0 if direction == "ul" else 1, bc, u, FP16 if fmt == "fp16" else FP32)


class GraphedUplink:
    """One uplink batch (CD kernel + fusion) captured into a CUDA graph over
    fixed device buffers: per-batch host overhead becomes a single graph
    launch, which matters for small, latency-bound batches (one OFDM symbol's
    subcarriers).  Refill ``H`` / ``y`` in place, then ``replay()``."""

    def __init__(self, eng: Engine, H, y, *, n0: float, ex: float = 1.0, K: int = 3, fusion="uniform"):
        self.eng, self.H, self.y = eng, H, y
        kw = dict(n0=n0, ex=ex, K=K, fusion=fusion)
        fmt = _fmt_of(H)
        S, Cn, U, _ = _shape(H, fmt)
        dev = H.device
        # every buffer the launches touch is allocated up front (no allocation during capture)
        self.x_local = complex_empty((S, Cn, U), fmt, dev)
        self.sigma2 = torch.empty((S, Cn), dtype=torch.float32, device=dev) if fusion == "optimal" else None
        self.xhat = torch.empty((S, U), dtype=torch.complex64, device=dev)
        self.stream = torch.cuda.Stream(dev)
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(self.stream):  # warm-up: static launch configs, function attributes
            eng.ul_detect(H, y, x_local=self.x_local, sigma2=self.sigma2, xhat=self.xhat, **kw)
        self.stream.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            eng.ul_detect(H, y, x_local=self.x_local, sigma2=self.sigma2, xhat=self.xhat, **kw)

    def replay(self):
        self.graph.replay()
        return self.xhat
