"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the CPU checkers.

Two interchangeable back-ends with one numpy-facing API:

* ``Oracle("port")``      -> oracle/libdcdoracle.so, the plain-C restatement
  (oracle/dcd_oracle.c) of the reference path, scalar-backend semantics.
* ``Oracle("reference")`` -> oracle/_ref/libdcdref.so, the UNMODIFIED reference
  sources (/root/reference/proj/src) compiled by oracle/Makefile plus
  oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module.  The product path (paper_1902_08653_b200) never does.

Arrays: complex128 numpy arrays; matrices in Fortran (column-major) order as
dcd::ComplexMatrix stores them (include/dcd/numerics.hpp:35-40).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libdcdoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdcdref.so")

FP64, FP32, FP16 = 0, 1, 2
MESSAGES, FULL_STORAGE = 0, 1
OPTIMAL, UNIFORM = 0, 1

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_up = C.POINTER(C.c_uint)


class OracleError(Exception):
    """Raised with the reference exception text; ``kind`` is 'invalid_argument'
    or 'runtime_error' (mirrors std::invalid_argument / std::runtime_error)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


class InvalidArgument(OracleError, ValueError):
    pass


class RuntimeErr(OracleError, RuntimeError):
    pass


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _cin(a, shape=None) -> np.ndarray:
    """complex128, contiguous in memory in the column-major sense for 2-D."""
    a = np.asarray(a, dtype=np.complex128)
    if a.ndim == 2:
        a = np.asfortranarray(a)
    else:
        a = np.ascontiguousarray(a)
    if shape is not None:
        assert a.shape == shape, (a.shape, shape)
    return a


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle` / `make -C oracle ref`)")
        self.lib = C.CDLL(path)
        self.p = "dcdo_" if kind == "port" else "dcdref_"
        L = self.lib
        f = self._f
        f("last_error").restype = C.c_char_p
        f("norm2sq").restype = C.c_double
        f("derive_seed").restype = C.c_uint64
        f("derive_seed").argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        f("f64_to_f16_bits").restype = C.c_uint16
        f("f64_to_f16_bits").argtypes = [C.c_double]
        f("f16_bits_to_f64").restype = C.c_double
        f("f16_bits_to_f64").argtypes = [C.c_uint16]
        f("snr_to_n0").restype = C.c_double
        f("snr_to_n0").argtypes = [C.c_double, C.c_int, C.c_double]
        f("rng_draw").argtypes = [C.c_uint64, C.c_int, C.c_int, _dp]
        f("make_batch").argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint, C.c_int, C.c_uint64,
                                    C.c_uint64, _dp, _u8p]
        f("uplink_observe").argtypes = [_dp, C.c_int, C.c_int, _u8p, C.c_uint, C.c_double,
                                        C.c_uint64, C.c_uint64, _dp, _dp]
        if kind == "reference":
            for name in ("ul_batch_run", "dl_batch_run"):
                f(name).restype = C.c_double
            L.dcdref_ul_batch_create.restype = C.c_void_p
            L.dcdref_dl_batch_create.restype = C.c_void_p
            L.dcdref_ul_batch_create.argtypes = [C.c_int] * 4 + [_dp, _dp]
            L.dcdref_dl_batch_create.argtypes = [C.c_int] * 4 + [_dp, _dp]
            L.dcdref_ul_batch_destroy.argtypes = [C.c_void_p]
            L.dcdref_dl_batch_destroy.argtypes = [C.c_void_p]
            L.dcdref_set_concurrent.argtypes = [C.c_int]
            L.dcdref_ul_batch_run.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_uint, C.c_int,
                                              C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
            L.dcdref_dl_batch_run.argtypes = [C.c_void_p, C.c_double, C.c_uint, C.c_int, C.c_int,
                                              C.c_int, C.c_int, C.c_int, _dp, _dp]

    # -- plumbing -----------------------------------------------------------
    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc: int):
        if rc == 0:
            return
        msg = self._f("last_error")().decode()
        if rc == 1:
            raise InvalidArgument("invalid_argument", msg)
        raise RuntimeErr("runtime_error", msg)

    def set_backend(self, b: str):
        """Reference only: pin the SIMD table ('scalar' or 'avx2')."""
        if self.kind != "reference":
            return
        self._check(self.lib.dcdref_set_backend(1 if b == "avx2" else 0))

    def backend(self) -> str:
        if self.kind != "reference":
            return "scalar"
        return "avx2" if self.lib.dcdref_active_backend() else "scalar"

    # -- kernels ------------------------------------------------------------
    def cdotc(self, a, b) -> complex:
        a, b = _cin(a), _cin(b)
        out = np.zeros(2)
        self._f("cdotc")(_ptr(a), _ptr(b), C.c_int(a.size), _ptr(out))
        return complex(out[0], out[1])

    def caxpy(self, alpha: complex, x, y) -> np.ndarray:
        x, y = _cin(x), _cin(y).copy()
        self._f("caxpy")(C.c_double(alpha.real), C.c_double(alpha.imag), _ptr(x), _ptr(y), C.c_int(x.size))
        return y

    def norm2sq(self, a) -> float:
        a = _cin(a)
        return self._f("norm2sq")(_ptr(a), C.c_int(a.size))

    def f64_to_f16_bits(self, x: float) -> int:
        return int(self._f("f64_to_f16_bits")(float(x)))

    def f16_bits_to_f64(self, h: int) -> float:
        return float(self._f("f16_bits_to_f64")(int(h)))

    def round_precision(self, x, fmt: int):
        arr = np.array(x, dtype=np.float64 if not np.iscomplexobj(x) else np.complex128, copy=True)
        flat = arr.view(np.float64).reshape(-1) if np.iscomplexobj(arr) else arr.reshape(-1)
        if self.kind == "port":
            self.lib.dcdo_round_precision(_ptr(flat), C.c_int(flat.size), C.c_int(fmt))
        else:
            self._check(self.lib.dcdref_round_precision(_ptr(flat), C.c_int(flat.size), C.c_int(fmt)))
        return arr

    # -- uplink -------------------------------------------------------------
    def cd_detect(self, h, y, n0, ex, t_max, fmt=FP64, scope=MESSAGES) -> np.ndarray:
        h = _cin(h)
        y = _cin(y)
        b, u = h.shape
        if y.size != b:
            raise InvalidArgument("invalid_argument", "detector: observation length must match antenna count")
        x = np.zeros(u, np.complex128)
        self._check(self._f("cd_detect")(_ptr(h), C.c_int(b), C.c_int(u), _ptr(y), C.c_double(n0),
                                         C.c_double(ex), C.c_uint(t_max), C.c_int(fmt), C.c_int(scope), _ptr(x)))
        return x

    def lmmse_exact(self, h, y, n0, ex) -> np.ndarray:
        h, y = _cin(h), _cin(y)
        b, u = h.shape
        x = np.zeros(u, np.complex128)
        self._check(self._f("lmmse_exact")(_ptr(h), C.c_int(b), C.c_int(u), _ptr(y), C.c_double(n0),
                                           C.c_double(ex), _ptr(x)))
        return x

    def post_eq_variance(self, h, n0, ex) -> float:
        h = _cin(h)
        b, u = h.shape
        out = np.zeros(1)
        self._check(self._f("post_eq_variance")(_ptr(h), C.c_int(b), C.c_int(u), C.c_double(n0),
                                                C.c_double(ex), _ptr(out)))
        return float(out[0])

    def fusion_weights(self, s2) -> np.ndarray:
        s2 = np.ascontiguousarray(s2, dtype=np.float64)
        w = np.zeros(max(s2.size, 1))
        self._check(self._f("fusion_weights")(_ptr(s2), C.c_int(s2.size), _ptr(w)))
        return w[: s2.size]

    def mmse_bias_factors(self, h, n0, ex) -> np.ndarray:
        h = _cin(h)
        b, u = h.shape
        beta = np.zeros(u)
        self._check(self._f("mmse_bias_factors")(_ptr(h), C.c_int(b), C.c_int(u), C.c_double(n0),
                                                 C.c_double(ex), _ptr(beta)))
        return beta

    def decentralized_cd_detect(self, hs, ys, n0, ex, t_max, fusion=OPTIMAL, fmt=FP64, scope=MESSAGES):
        """hs: list of B_c x U blocks; ys: list of B_c vectors.
        Returns dict(xhat, local (C x U), sigma2 (C or empty), weights)."""
        nc = len(hs)
        u = hs[0].shape[1] if nc else 0
        bc = np.array([h.shape[0] for h in hs], dtype=np.int32)
        tiles = np.concatenate([_cin(h).ravel(order="F") for h in hs]) if nc else np.zeros(1, np.complex128)
        yy = np.concatenate([_cin(y) for y in ys]) if nc else np.zeros(1, np.complex128)
        xhat = np.zeros(max(u, 1), np.complex128)
        local = np.zeros((max(nc, 1), max(u, 1)), np.complex128)
        s2 = np.zeros(max(nc, 1))
        w = np.zeros(max(nc, 1))
        args = [C.c_int(nc), bc.ctypes.data_as(C.POINTER(C.c_int)), C.c_int(u), _ptr(tiles), _ptr(yy),
                C.c_double(n0), C.c_double(ex), C.c_uint(t_max), C.c_int(fusion), C.c_int(fmt),
                C.c_int(scope)]
        if self.kind == "reference":
            args.append(C.c_int(0))
        args += [_ptr(xhat), _ptr(local), _ptr(s2), _ptr(w)]
        self._check(self._f("decentralized_cd_detect")(*args))
        return {"xhat": xhat[:u], "local": local[:nc, :u], "sigma2": s2[:nc] if fusion == OPTIMAL else np.zeros(0),
                "weights": w[:nc]}

    # -- downlink -----------------------------------------------------------
    def cd_precode(self, h_dl, s, t_max, fmt=FP64, scope=MESSAGES) -> np.ndarray:
        h_dl, s = _cin(h_dl), _cin(s)
        u, b = h_dl.shape
        if s.size != u:
            raise InvalidArgument("invalid_argument", "precoder: symbol count must match user count")
        x = np.zeros(b, np.complex128)
        self._check(self._f("cd_precode")(_ptr(h_dl), C.c_int(u), C.c_int(b), _ptr(s), C.c_uint(t_max),
                                          C.c_int(fmt), C.c_int(scope), _ptr(x)))
        return x

    def zf_exact(self, h_dl, s) -> np.ndarray:
        h_dl, s = _cin(h_dl), _cin(s)
        u, b = h_dl.shape
        x = np.zeros(b, np.complex128)
        self._check(self._f("zf_exact")(_ptr(h_dl), C.c_int(u), C.c_int(b), _ptr(s), _ptr(x)))
        return x

    def mf_detect(self, hs, ys) -> np.ndarray:
        """mf_detect (detect.cpp:191-218) over cluster blocks hs (B_c x U) and ys."""
        nc = len(hs)
        u = hs[0].shape[1]
        bc = np.array([h.shape[0] for h in hs], dtype=np.int32)
        tiles = np.concatenate([_cin(h).ravel(order="F") for h in hs])
        yy = np.concatenate([_cin(y) for y in ys])
        x = np.zeros(u, np.complex128)
        self._check(self._f("mf_detect")(C.c_int(nc), bc.ctypes.data_as(C.POINTER(C.c_int)), C.c_int(u),
                                         _ptr(tiles), _ptr(yy), _ptr(x)))
        return x

    def mf_precode(self, h_dl_blocks, s, rho) -> np.ndarray:
        """mf_precode (precode.cpp:171-202): concatenated per-cluster beamformers."""
        nc = len(h_dl_blocks)
        s = _cin(s)
        bc = np.array([h.shape[1] for h in h_dl_blocks], dtype=np.int32)
        tiles = np.concatenate([_cin(h).ravel(order="F") for h in h_dl_blocks])
        x = np.zeros(int(bc.sum()), np.complex128)
        self._check(self._f("mf_precode")(C.c_int(nc), bc.ctypes.data_as(C.POINTER(C.c_int)), C.c_int(s.size),
                                          _ptr(tiles), _ptr(s), C.c_double(rho), _ptr(x)))
        return x

    def power_scale(self, x, rho) -> np.ndarray:
        x = _cin(x).copy()
        self._check(self._f("power_scale")(_ptr(x), C.c_int(x.size), C.c_double(rho)))
        return x

    def decentralized_cd_precode(self, h_dl_blocks, s, rho, t_max, fmt=FP64, scope=MESSAGES):
        nc = len(h_dl_blocks)
        s = _cin(s)
        u = s.size
        bc = np.array([h.shape[1] for h in h_dl_blocks], dtype=np.int32)
        tiles = np.concatenate([_cin(h).ravel(order="F") for h in h_dl_blocks]) if nc else np.zeros(1, np.complex128)
        x = np.zeros(max(int(bc.sum()), 1), np.complex128)
        g = np.zeros(1)
        args = [C.c_int(nc), bc.ctypes.data_as(C.POINTER(C.c_int)), C.c_int(u), _ptr(tiles), _ptr(s),
                C.c_double(rho), C.c_uint(t_max), C.c_int(fmt), C.c_int(scope)]
        if self.kind == "reference":
            args.append(C.c_int(0))
        args += [_ptr(x), _ptr(g)]
        self._check(self._f("decentralized_cd_precode")(*args))
        return {"x": x[: int(bc.sum())], "effective_gain": float(g[0])}

    # -- batched over the device layout -------------------------------------
    def ul_detect_batch(self, h_tiles, y, n0, ex, t_max, fusion=UNIFORM, fmt=FP64, scope=MESSAGES):
        """h_tiles: [S, C, U, B_c] complex (each tile column-major B_c x U);
        y: [S, C, B_c].  Returns (xhat [S,U], local [S,C,U], sigma2 [S,C])."""
        S, Cn, U, Bc = h_tiles.shape
        h_tiles = np.ascontiguousarray(h_tiles, np.complex128)
        y = np.ascontiguousarray(y, np.complex128)
        xhat = np.zeros((S, U), np.complex128)
        local = np.zeros((S, Cn, U), np.complex128)
        s2 = np.zeros((S, Cn))
        if self.kind == "port":
            self._check(self.lib.dcdo_ul_detect_batch(
                C.c_int(S), C.c_int(Cn), C.c_int(Bc), C.c_int(U), _ptr(h_tiles), _ptr(y), C.c_double(n0),
                C.c_double(ex), C.c_uint(t_max), C.c_int(fusion), C.c_int(fmt), C.c_int(scope), _ptr(xhat),
                _ptr(local), _ptr(s2)))
        else:
            for s in range(S):
                r = self.decentralized_cd_detect([h_tiles[s, c].T for c in range(Cn)], list(y[s]), n0, ex,
                                                 t_max, fusion, fmt, scope)
                xhat[s], local[s] = r["xhat"], r["local"]
                if fusion == OPTIMAL:
                    s2[s] = r["sigma2"]
        return xhat, local, s2

    def dl_precode_batch(self, h_tiles, sym, rho, t_max, fmt=FP64, scope=MESSAGES):
        """h_tiles: [S, C, U, B_c] uplink tiles; sym: [S, U].
        Returns (x [S, C, B_c], gain [S])."""
        S, Cn, U, Bc = h_tiles.shape
        h_tiles = np.ascontiguousarray(h_tiles, np.complex128)
        sym = np.ascontiguousarray(sym, np.complex128)
        x = np.zeros((S, Cn, Bc), np.complex128)
        g = np.zeros(S)
        if self.kind == "port":
            self._check(self.lib.dcdo_dl_precode_batch(
                C.c_int(S), C.c_int(Cn), C.c_int(Bc), C.c_int(U), _ptr(h_tiles), _ptr(sym), C.c_double(rho),
                C.c_uint(t_max), C.c_int(fmt), C.c_int(scope), _ptr(x), _ptr(g)))
        else:
            for s in range(S):
                blocks = [np.conj(h_tiles[s, c]) for c in range(Cn)]  # [U, B_c] = H_ul,c^H
                r = self.decentralized_cd_precode(blocks, sym[s], rho, t_max, fmt, scope)
                x[s] = r["x"].reshape(Cn, Bc)
                g[s] = r["effective_gain"]
        return x, g

    # -- system model -------------------------------------------------------
    def derive_seed(self, master, purpose, index) -> int:
        return int(self._f("derive_seed")(master, purpose, index))

    def rng_draw(self, seed, kind, n) -> np.ndarray:
        out = np.zeros(n)
        self._f("rng_draw")(seed, kind, n, _ptr(out))
        return out

    def qam_points(self, order, ex=1.0) -> np.ndarray:
        pts = np.zeros(order, np.complex128)
        self._check(self._f("qam_points")(C.c_uint(order), C.c_double(ex), _ptr(pts)))
        return pts

    def slice(self, order, y, ex=1.0) -> np.ndarray:
        y = _cin(y)
        lab = np.zeros(y.size, np.uint32)
        self._check(self._f("slice")(C.c_uint(order), C.c_double(ex), _ptr(y), C.c_int(y.size),
                                     lab.ctypes.data_as(_up)))
        return lab

    def make_batch(self, nc, bc, u, qam, count, seed, first_trial=0):
        """Returns (H [count, B, U] complex, bits [count, U*bps] uint8) exactly as
        dcd::make_batch (src/cluster.cpp:80-105)."""
        b = nc * bc
        bps = {4: 2, 16: 4, 64: 6}[qam]
        hf = np.zeros((count, u, b), np.complex128)  # per subcarrier: U columns of B (column-major)
        bits = np.zeros((count, u * bps), np.uint8)
        self._check(self._f("make_batch")(nc, bc, u, qam, count, seed, first_trial, _ptr(hf),
                                          bits.ctypes.data_as(_u8p)))
        return np.transpose(hf, (0, 2, 1)), bits

    def uplink_observe(self, h, bits, qam, n0, seed, trial):
        h = _cin(h)
        b, u = h.shape
        bits = np.ascontiguousarray(bits, np.uint8)
        y = np.zeros(b, np.complex128)
        x = np.zeros(u, np.complex128)
        self._check(self._f("uplink_observe")(_ptr(h), b, u, bits.ctypes.data_as(_u8p), qam, n0, seed, trial,
                                              _ptr(y), _ptr(x)))
        return y, x

    def snr_to_n0(self, snr_db, users, ex=1.0) -> float:
        return float(self._f("snr_to_n0")(snr_db, users, ex))


def tiles_from_full(h_full: np.ndarray, nc: int) -> np.ndarray:
    """[S, B, U] full channels -> [S, C, U, B_c] device tiles (row partition in
    antenna order, src/mimo.cpp:28-44)."""
    S, B, U = h_full.shape
    bc = B // nc
    return np.ascontiguousarray(np.transpose(h_full.reshape(S, nc, bc, U), (0, 1, 3, 2)))


def reference_batch(nc, bc, u, qam, count, seed, snr_db=10.0, first_trial=0, kind="port"):
    """The reference's own input synthesis for an uplink+downlink batch:
    make_batch + run_uplink_round's observation (src/cluster.cpp:142-145).
    Returns dict(h_tiles [S,C,U,B_c], y [S,C,B_c], x_true [S,U], bits, n0)."""
    o = Oracle(kind)
    h, bits = o.make_batch(nc, bc, u, qam, count, seed, first_trial)
    n0 = o.snr_to_n0(snr_db, u, 1.0)
    ys = np.zeros((count, nc * bc), np.complex128)
    xs = np.zeros((count, u), np.complex128)
    for s in range(count):
        ys[s], xs[s] = o.uplink_observe(h[s], bits[s], qam, n0, seed, first_trial + s)
    return {"h_tiles": tiles_from_full(h, nc), "y": ys.reshape(count, nc, bc), "x_true": xs, "bits": bits,
            "n0": n0, "h_full": h}
