"""GPU-backed BER sweeps: the reference's run_ber_sweep
(src/harness.cpp:136-238, include/dcd/harness.hpp) on the device path.

Every chunk of trials is synthesised on the GPU (dcdg_synth, counter-based and
keyed by (seed, SNR index, trial) like harness.cpp:176), detected/precoded by
the CUDA kernels, sliced and error-counted on the device; the host only reads
one error counter per point.  Methods and their semantics follow
run_uplink_round / run_downlink_round (src/cluster.cpp:125-300):

  uplink   dcd    decentralized CD (Alg. 1) + fusion, unbiased by the full-H
                  MMSE factors before slicing (cluster.cpp:196-203)
           cd     centralized CD on the stacked channel (raw-sample forwarding)
           exact  exact full-channel L-MMSE (lmmse_exact)
           mf     matched filter, sliced raw
  downlink dcd    decentralized CD ZF (Alg. 2) with rho/sqrt(C) per cluster
           cd     centralized CD ZF + power_scale(rho)
           exact  min-norm ZF + power_scale(rho)
           mf     matched filter, rho/sqrt(C) per cluster
  receive  downlink_receive_and_ber: genie beta, AWGN, flagged trials count
           half their bits (precode.cpp:204-233)

Precision: "fp64" and "fp32" compute in fp32 on the GPU; fp16 "full" runs the
half2 kernels on binary16 tiles; fp16 "messages" runs fp32 kernels and rounds
the wire payloads to binary16 (detect.cpp:170-173, precode.cpp:159-160).  The
exact and MF baselines compute in fp32 in every mode.

The random streams are not the reference's mt19937_64 streams, so BER values
agree statistically, not bit for bit; the bit-exact parity of the detection
path itself is tested on the reference's own batches (tests/)."""
from __future__ import annotations

import contextlib
import math
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import torch

from .engine import Engine, to_complex64, to_fp16, to_fp16_pairs

METHODS = ("dcd", "cd", "exact", "mf")
_BPS = {4: 2, 16: 4, 64: 6}
_BYTES_PER_COMPLEX = {"fp64": 16, "fp32": 8, "fp16": 4}  # precision.cpp:8-15


@dataclass
class SweepSpec:
    """Mirror of dcd::SweepSpec (include/dcd/harness.hpp:35-60)."""
    direction: str = "uplink"
    methods: Sequence[str] = ("dcd",)
    users: int = 8
    cluster_size: int = 32
    clusters: int = 4
    qam_order: int = 16
    ex: float = 1.0
    snr_db: Sequence[float] = (0, 2, 4, 6, 8)
    t_max: Sequence[int] = (3,)
    precision: str = "fp64"      # fp64 | fp32 | fp16
    scope: str = "messages"      # messages | full (fp16 only)
    fusion: str = "optimal"
    min_bits: int = 1_000_000
    max_trials: int = 4_000_000_000
    seed: int = 1
    batch_subcarriers: int = 16384  # GPU chunk (the reference's engine chunk is 256)

    @property
    def antennas(self) -> int:
        return self.cluster_size * self.clusters

    def validate(self) -> None:
        """SweepSpec::validate (harness.cpp:41-62), same order and texts."""
        if self.users <= 0 or self.cluster_size <= 0 or self.clusters <= 0:
            raise ValueError("sweep: users, cluster size and cluster count must be positive")
        if not self.methods:
            raise ValueError("sweep: no methods selected")
        if not self.snr_db:
            raise ValueError("sweep: empty SNR grid")
        if not self.t_max:
            raise ValueError("sweep: empty T_max list")
        if any(t <= 0 for t in self.t_max):
            raise ValueError("sweep: T_max entries must be >= 1")
        if not self.ex > 0.0:
            raise ValueError("sweep: symbol energy must be positive")
        if self.min_bits < 10_000:
            raise ValueError("sweep: min_bits must be at least 10000")
        if self.max_trials <= 0 or self.max_trials > 0xFFFFFFFF:
            raise ValueError("sweep: max_trials must be in [1, 2^32-1]")
        if self.batch_subcarriers <= 0:
            raise ValueError("sweep: batch size must be positive")
        if self.antennas < self.users:
            raise ValueError("sweep: need at least as many antennas as users")
        if self.direction == "downlink" and self.cluster_size < self.users:
            raise ValueError("sweep: downlink clusters need at least as many antennas as users (B_c >= U)")
        if self.qam_order not in _BPS:
            raise ValueError("Constellation::qam: order must be 4, 16 or 64")
        if self.direction not in ("uplink", "downlink"):
            raise ValueError(f"unknown direction: {self.direction}")
        for m in self.methods:
            if m not in METHODS:
                raise ValueError(f"unknown method: {m}")
        if self.precision not in _BYTES_PER_COMPLEX or self.scope not in ("messages", "full"):
            raise ValueError("unknown precision mode")


@dataclass
class BerPoint:
    """Mirror of dcd::BerPoint (harness.hpp:64-74)."""
    method: str
    t_max: int
    snr_db: float
    bits: int = 0
    errors: int = 0
    ber: float = 0.0
    ci_halfwidth: float = 0.0
    message_bytes: int = 0
    flagged_trials: int = 0
    seconds: float = 0.0  # device time of the point (not in the reference)


def snr_to_n0(snr_db: float, users: int, ex: float) -> float:
    """mimo.cpp:159-163."""
    if users <= 0 or not ex > 0.0:
        raise ValueError("snr_to_n0: need users >= 1 and positive symbol energy")
    return users * ex / 10.0 ** (snr_db / 10.0)


def message_bytes_per_trial(spec: SweepSpec, method: str) -> int:
    """Interconnect bytes per subcarrier as run_uplink_round / run_downlink_round
    log them (cluster.cpp:9-22,158-190,253-280): CD and MF exchange U-vectors
    (plus sigma^2 for optimal fusion, plus U energies for the uplink MF);
    centralized methods forward B_c samples per cluster."""
    bpc = _BYTES_PER_COMPLEX[spec.precision]
    u, bc, nc = spec.users, spec.cluster_size, spec.clusters
    if method in ("cd", "exact"):
        elems, aux = bc, 0
    elif spec.direction == "uplink" and method == "mf":
        elems, aux = u, u
    else:
        elems = u
        aux = 1 if (spec.direction == "uplink" and spec.fusion == "optimal") else 0
    return nc * (elems * bpc + aux * (bpc // 2))


def analytic_qam_ber(order: int, es_over_n0: float) -> float:
    """harness.cpp:388-422: exact Gray-QAM BER over AWGN at symbol SNR."""
    if order not in _BPS:
        raise ValueError("analytic_qam_ber: order must be 4, 16 or 64")
    if not es_over_n0 > 0.0:
        raise ValueError("analytic_qam_ber: SNR must be positive")
    levels = 2
    while levels * levels < order:
        levels <<= 1
    axis_bits = round(math.log2(levels))
    scale = math.sqrt(3.0 / (2.0 * (levels * levels - 1.0)))
    sigma = math.sqrt(1.0 / es_over_n0 / 2.0)

    def phi(x):
        return 0.5 * math.erfc(-x / math.sqrt(2.0))

    level = [scale * (2.0 * p - (levels - 1.0)) for p in range(levels)]
    label = [p ^ (p >> 1) for p in range(levels)]
    bad = 0.0
    for sent in range(levels):
        for dec in range(levels):
            lo = -math.inf if dec == 0 else 0.5 * (level[dec - 1] + level[dec])
            hi = math.inf if dec + 1 == levels else 0.5 * (level[dec] + level[dec + 1])
            p = phi((hi - level[sent]) / sigma) - phi((lo - level[sent]) / sigma)
            bad += p * bin(label[sent] ^ label[dec]).count("1")
    return bad / (levels * axis_bits)


def snr_at_ber(curve: Sequence[Tuple[float, float]], target: float) -> float:
    """harness.cpp:424-438: log-linear interpolation of the first bracketing pair."""
    if not target > 0.0:
        return math.nan
    for (s0, b0), (s1, b1) in zip(curve, curve[1:]):
        if b0 <= 0.0 or b1 <= 0.0:
            continue
        if b0 >= target >= b1 and b0 > b1:
            f = (math.log10(target) - math.log10(b0)) / (math.log10(b1) - math.log10(b0))
            return s0 + f * (s1 - s0)
    return math.nan


def curve_of(points: Sequence[BerPoint], method: str, t: int) -> List[Tuple[float, float]]:
    return [(p.snr_db, p.ber) for p in points if p.method == method and p.t_max == t]


# ---------------------------------------------------------------------------
# one point
# ---------------------------------------------------------------------------
@contextlib.contextmanager
def _fp16_arithmetic(eng: Engine, full: bool):
    """fp16 'full' scope measures the loss of fp16 ARITHMETIC (precision.cpp,
    full_storage), so it runs the half2 sweep kernels, not the default
    tensor-core Gram kernels (fp32 arithmetic on fp16 storage); the engine's
    previous choice is restored afterwards."""
    if not full:
        yield
        return
    prev = eng.fp16_algorithm
    eng.set_fp16_algorithm("sweep")
    try:
        yield
    finally:
        eng.set_fp16_algorithm(prev)


def _uplink_chunk(eng: Engine, spec: SweepSpec, method: str, t: int, n0: float, S: int, first_trial: int):
    U, C, Bc = spec.users, spec.clusters, spec.cluster_size
    central = method == "cd"
    b = eng.synth(S, 1 if central else C, spec.antennas if central else Bc, U, qam=spec.qam_order, ex=spec.ex,
                  n0=n0, seed=spec.seed, first_trial=first_trial, uplink=True)
    H, y = b["H"], b["y"]
    fp16 = spec.precision == "fp16"
    full = fp16 and spec.scope == "full"
    unbias = method != "mf"
    if method in ("dcd", "cd"):
        Hd, yd = (to_fp16_pairs(H), to_fp16_pairs(y)) if full else (H, y)
        if central and fp16 and not full:
            eng.round_fp16(yd)  # raw-sample forwarding in binary16 (cluster.cpp:176-178)
        if method == "dcd" and fp16 and not full:
            r = eng.ul_detect(Hd, yd, n0=n0, ex=spec.ex, K=t, fusion=spec.fusion, want_xhat=False)
            eng.round_fp16(r.x_local)
            s2 = r.sigma2
            if s2 is not None:
                eng.round_fp16(s2)
            xhat = eng.fuse(r.x_local, s2, fusion=spec.fusion)
        else:
            with _fp16_arithmetic(eng, full):
                xhat = eng.ul_detect(Hd, yd, n0=n0, ex=spec.ex, K=t, fusion=spec.fusion, want_local=False).xhat
    elif method == "exact":
        if fp16:
            eng.round_fp16(y)
        xhat = eng.lmmse_exact(H, y, n0=n0, ex=spec.ex)
    else:
        xhat = eng.mf_detect(H, y)
    beta = eng.mmse_bias(H, n0=n0, ex=spec.ex) if (unbias and n0 > 0) else None
    labels = eng.slice(xhat, beta, qam=spec.qam_order, ex=spec.ex)
    return eng.bit_errors(labels, b["bits"], qam=spec.qam_order), None


def _downlink_chunk(eng: Engine, spec: SweepSpec, method: str, t: int, n0: float, S: int, first_trial: int):
    U, C, Bc = spec.users, spec.clusters, spec.cluster_size
    rho = math.sqrt(U * spec.ex)  # harness.cpp:159
    central = method == "cd"
    b = eng.synth(S, 1 if central else C, spec.antennas if central else Bc, U, qam=spec.qam_order, ex=spec.ex,
                  n0=n0, seed=spec.seed, first_trial=first_trial, uplink=False, downlink=True)
    H, sym = b["H"], b["sym"]
    fp16 = spec.precision == "fp16"
    full = fp16 and spec.scope == "full"
    if method in ("dcd", "cd"):
        if full:
            with _fp16_arithmetic(eng, full):
                x = to_complex64(eng.dl_precode(to_fp16_pairs(H), to_fp16(sym), rho=rho, K=t, want_gain=False).x)
        else:
            s_in = sym.clone() if fp16 else sym
            if fp16:
                eng.round_fp16(s_in)  # binary16 symbol broadcast (precode.cpp:159-160)
            x = eng.dl_precode(H, s_in, rho=rho, K=t, want_gain=False).x
            if fp16 and central:
                eng.round_fp16(x)  # beamformer forwarding in binary16 (cluster.cpp:268)
    elif method == "exact":
        x = eng.zf_exact(H, sym, rho=rho)
        if fp16:
            eng.round_fp16(x)
    else:
        x = eng.mf_precode(H, sym, rho=rho)
    labels, _, flagged = eng.dl_receive(H, x, sym, b["noise_dl"], qam=spec.qam_order, ex=spec.ex)
    return eng.bit_errors(labels, b["bits"], qam=spec.qam_order), flagged.sum()


def measure_point(eng: Engine, spec: SweepSpec, method: str, t: int, snr_idx: int, snr: float) -> BerPoint:
    """harness.cpp:136-184 with the chunks on the device."""
    n0 = snr_to_n0(snr, spec.users, spec.ex)
    bits_per_trial = spec.users * _BPS[spec.qam_order]
    trials = min((spec.min_bits + bits_per_trial - 1) // bits_per_trial, spec.max_trials) or 1
    dev = eng.device
    errors = torch.zeros((), dtype=torch.int64, device=dev)
    flagged = torch.zeros((), dtype=torch.int64, device=dev)
    fn = _uplink_chunk if spec.direction == "uplink" else _downlink_chunk
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    done = 0
    while done < trials:
        chunk = min(spec.batch_subcarriers, trials - done)
        first_trial = (snr_idx << 32) + done
        e, f = fn(eng, spec, method, t, n0, chunk, first_trial)
        errors += e.reshape(())
        if f is not None:
            flagged += f
        done += chunk
    e1.record(st)
    eng.sync()
    p = BerPoint(method, t if method in ("dcd", "cd") else 0, float(snr))
    p.bits = trials * bits_per_trial
    p.errors = int(errors.item())
    p.flagged_trials = int(flagged.item())
    p.ber = p.errors / p.bits if p.bits else 0.0
    p.ci_halfwidth = 1.96 * math.sqrt(max(p.ber * (1.0 - p.ber), 0.0) / p.bits) if p.bits else 0.0
    p.message_bytes = trials * message_bytes_per_trial(spec, method)
    p.seconds = e0.elapsed_time(e1) / 1e3
    return p


@dataclass
class ConvergencePoint:
    """Mirror of dcd::ConvergencePoint (harness.hpp:81-85)."""
    t: int
    median: float
    p95: float


def run_convergence_study(spec: SweepSpec, engine: Optional[Engine] = None, instances: int = 200,
                          csv_path: str = "") -> List[ConvergencePoint]:
    """run_convergence_study (harness.cpp:240-307): median and 95th-percentile
    relative distance between the T-sweep centralized CD solution (cd_detect /
    raw cd_precode on the full channel) and the direction's exact solution
    (lmmse_exact / raw zf_exact) over `instances` systems at the first SNR
    point, for T = 1 .. max(t_max).  Both sides run in fp32 on the GPU, so the
    distance floors near 1e-6 instead of the reference's fp64 1e-15."""
    spec.validate()
    if instances <= 0:
        raise ValueError("convergence study: need at least one instance")
    eng = engine or Engine(0)
    t_top = max(spec.t_max)
    n0 = snr_to_n0(spec.snr_db[0], spec.users, spec.ex)
    B, U = spec.antennas, spec.users
    up = spec.direction == "uplink"
    b = eng.synth(instances, 1, B, U, qam=spec.qam_order, ex=spec.ex, n0=n0, seed=spec.seed, uplink=up,
                  downlink=not up)
    H = b["H"]
    if up:
        oracle = eng.lmmse_exact(H, b["y"], n0=n0, ex=spec.ex)
    else:
        oracle = eng.zf_exact(H, b["sym"], rho=0.0).reshape(instances, B)
    onorm = torch.linalg.vector_norm(oracle, dim=1)
    out: List[ConvergencePoint] = []
    for t in range(1, t_top + 1):
        if up:
            xt = eng.ul_detect(H, b["y"], n0=n0, ex=spec.ex, K=t, fusion="uniform", want_xhat=False).x_local
            xt = xt.reshape(instances, U)
        else:
            xt = eng.dl_precode(H, b["sym"], rho=0.0, K=t, want_gain=False).x.reshape(instances, B)
        d = torch.linalg.vector_norm(xt - oracle, dim=1)
        d = torch.where(onorm > 0, d / torch.where(onorm > 0, onorm, torch.ones_like(onorm)), d)
        v = torch.sort(d.double()).values.cpu()
        n = v.numel()
        out.append(ConvergencePoint(t, float(v[n // 2]), float(v[min(n - 1, int(0.95 * (n - 1) + 0.5))])))
    eng.sync()
    if csv_path:
        with open(csv_path, "w") as f:
            f.write("# dcdg-converge-v1 (GPU, fp32)\nt,median_rel_distance,p95_rel_distance\n")
            for p in out:
                f.write(f"{p.t},{p.median:.9e},{p.p95:.9e}\n")
    return out


def run_ber_sweep(spec: SweepSpec, engine: Optional[Engine] = None, csv_path: str = "") -> List[BerPoint]:
    """run_ber_sweep (harness.cpp:188-238): methods x T_max x SNR points."""
    spec.validate()
    eng = engine or Engine(0)
    points: List[BerPoint] = []
    for m in spec.methods:
        ts = list(spec.t_max) if m in ("dcd", "cd") else [0]
        for t in ts:
            for i, snr in enumerate(spec.snr_db):
                points.append(measure_point(eng, spec, m, t, i, snr))
    if csv_path:
        with open(csv_path, "w") as f:
            f.write("# dcdg-ber-v1 (GPU, counter-based synthesis)\n")
            f.write("direction,method,t_max,precision,scope,fusion,snr_db,bits,errors,ber,ci_halfwidth,"
                    "message_bytes,flagged_trials\n")
            for p in points:
                f.write(f"{spec.direction},{p.method},{p.t_max},{spec.precision},{spec.scope},{spec.fusion},"
                        f"{p.snr_db:.6g},{p.bits},{p.errors},{p.ber:.9e},{p.ci_halfwidth:.9e},{p.message_bytes},"
                        f"{p.flagged_trials}\n")
    return points
