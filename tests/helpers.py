"""Shared test helpers: reference-generated batches, device conversion,
per-problem relative errors (the parity metric of BASELINE.md §4)."""
from __future__ import annotations

import functools

import numpy as np

from oracle.oracle import FP16, FP64, FULL_STORAGE, MESSAGES, OPTIMAL, UNIFORM, Oracle, reference_batch  # noqa: F401

TOL_FP32 = 1e-5   # north_star: fp32 vectors within 1e-5 relative of the CPU oracle
TOL_FP16 = 2e-2   # north_star: fp16 (half2) within 2e-2


@functools.lru_cache(maxsize=32)
def batch(nc, bc, u, qam=16, S=64, seed=1, snr_db=10.0, first_trial=0):
    """Reference-generated (make_batch + uplink observation) batch, cached."""
    return reference_batch(nc, bc, u, qam, S, seed, snr_db, first_trial, kind="port")


def rel_err(got, want, axis=-1):
    """max over problems of ||got - want|| / ||want|| (vectors along `axis`)."""
    got = np.asarray(got, np.complex128)
    want = np.asarray(want, np.complex128)
    num = np.linalg.norm(got - want, axis=axis)
    den = np.linalg.norm(want, axis=axis)
    den = np.where(den == 0, 1.0, den)
    return float(np.max(num / den)) if num.size else 0.0


def to_dev(a, fmt="fp32", pairs=False):
    """numpy complex -> device tensor; fp16 channel tiles / receive vectors use
    the row-pair planar layout (pairs=True), symbol vectors stay interleaved."""
    import torch

    from paper_1902_08653_b200 import to_fp16_pairs
    t = torch.from_numpy(np.ascontiguousarray(a, np.complex128)).to(torch.complex64).cuda()
    if fmt == "fp16":
        if pairs:
            return to_fp16_pairs(t)
        return torch.view_as_real(t).to(torch.float16).contiguous()
    return t.contiguous()


def to_host(t):
    import torch
    if t.dtype == torch.float16:
        t = torch.view_as_complex(t.float().contiguous())
    return t.cpu().numpy().astype(np.complex128)


def qam_symbols(S, u, qam=16, seed=7):
    """Random QAM symbol vectors [S, U] on the reference constellation."""
    pts = Oracle("port").qam_points(qam)
    rng = np.random.default_rng(seed)
    return pts[rng.integers(0, qam, size=(S, u))]
