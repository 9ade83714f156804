#!/usr/bin/env python
"""Benchmark of the decentralized CD hot path on B200 (BASELINE.json metric:
"CD detect/precode throughput (Gbps) & batch latency, B=256 U=16 C=8").

Workload (configs[1]): uplink CD L-MMSE detection, B=256 antennas in C=8
clusters of B_c=32, U=16 users, 16-QAM, K=3 sweeps, fp32, uniform fusion;
one batch = 1200 subcarriers x 14 OFDM symbols = 16,800 subcarrier-symbol
problems per GPU-cluster-set.  Gbps = S * U * log2(Q) / t_batch (the paper's
definition).

N GPUs (torchrun, one process per GPU): the 8 clusters are partitioned over
the ranks (C/N per rank) and every rank processes S = 16,800*N subcarriers of
its clusters (weak scaling: per-GPU work fixed); the partial fused estimates
are reduce-scattered over the subcarrier axis (NCCL), so each rank ends with
the fused estimates of S/N subcarriers.

  value  device-resident throughput (inputs in HBM, CUDA events, max over
         ranks); the batch (602 MB/GPU) is larger than L2 (126 MB).
  e2e    same metric through Engine.ul_detect with pinned HOST buffers: H2D of
         the batch's H and y + detection + D2H of the fused estimates.
  --impl reference   the reference's CPU implementation (oracle/_ref, built
         from /root/reference sources) on this host's cores, same config.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B, C, U, QAM, K_SWEEPS = 256, 8, 16, 16, 3
BC = B // C
S_PER_GPU = 1200 * 14
SNR_DB = 10.0
BITS = int(math.log2(QAM))
METRIC = "CD detect/precode throughput (Gbps) & batch latency, B=256 U=16 C=8, 1-8 GPUs"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def alg_bytes_per_problem(bc, u, esz):
    """(B_c*U + B_c + U) * bytes-per-complex per cluster-problem."""
    return (bc * u + bc + u) * esz


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML polled
    from a thread every ~0.5 ms (no process fork next to the launching thread),
    nvidia-smi when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.source = "nvml"
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            try:  # CUDA ordinal -> NVML handle by PCI location (CUDA_VISIBLE_DEVICES may reorder)
                import torch
                pr = torch.cuda.get_device_properties(index)
                loc = (int(pr.pci_domain_id), int(pr.pci_bus_id), int(pr.pci_device_id))
                for i in range(pynvml.nvmlDeviceGetCount()):
                    hi = pynvml.nvmlDeviceGetHandleByIndex(i)
                    pi = pynvml.nvmlDeviceGetPciInfo(hi)
                    if (int(pi.domain), int(pi.bus), int(pi.device)) == loc:
                        h = hi
                        break
            except Exception:
                pass
            self._nvml = (pynvml, h)
        except Exception:
            self.source = "nvidia-smi"

    def _sample_nvml(self):
        nv, h = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        return [str(sm), str(mx)] + ["Active" if r & b else "Not Active" for b in bits]

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self.samples.append(self._sample_nvml())
                    self._stop.wait(0.0005)
                    continue
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                f = [x.strip() for x in out.stdout.strip().split(",")]
                if len(f) >= 6:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "source": self.source}


# ---------------------------------------------------------------------------
# synthetic inputs (device-side, torch RNG; same distribution as the
# reference's make_batch: H ~ CN(0,1), Gray 16-QAM at unit energy, AWGN N0)
# ---------------------------------------------------------------------------
def make_inputs(S, c_local, device, seed, u=U, bc=BC):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    n0 = u * 1.0 / 10 ** (SNR_DB / 10)
    H = torch.randn((S, c_local, u, bc), dtype=torch.complex64, device=device, generator=g)  # CN(0,1)
    lv = torch.tensor([-3.0, -1.0, 1.0, 3.0], device=device) / math.sqrt(10.0)
    idx = torch.randint(0, 4, (S, u, 2), device=device, generator=g)
    x = torch.complex(lv[idx[..., 0]], lv[idx[..., 1]])
    noise = torch.randn((S, c_local, bc), dtype=torch.complex64, device=device, generator=g) * math.sqrt(n0)
    y = torch.einsum("scub,su->scb", H, x) + noise
    return H.contiguous(), y.contiguous(), x.contiguous(), n0


def _ev():
    import torch
    return torch.cuda.Event(enable_timing=True)


def _time_stream(fn, stream, reps):
    """Average ms of `fn` over `reps` calls, CUDA events on `stream`."""
    import torch
    torch.cuda.synchronize()
    a, b = _ev(), _ev()
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def secondary_lines(eng, dev, S, reps, hbm):
    """Kernel-level numbers for the other north-star workloads (configs[2],
    configs[3] and optimal fusion) at the same batch size, N=1."""
    import torch

    from paper_1902_08653_b200 import to_fp16, to_fp16_pairs
    out = {}
    H, y, x, n0 = make_inputs(S, C, dev, 4321)
    st = torch.cuda.current_stream(dev)
    P = S * C
    rho = math.sqrt(U)
    # fp16: the default kernels are the tensor-core Gram kernels; "fp16sweep"
    # are the half2 residual-sweep kernels (the paper's half-precision arithmetic)
    for fmt in ("fp32", "fp16", "fp16sweep"):
        esz = 8 if fmt == "fp32" else 4
        Hh, yh, xh = (H, y, x) if fmt == "fp32" else (to_fp16_pairs(H), to_fp16_pairs(y), to_fp16(x))
        eng.set_fp16_algorithm("sweep" if fmt == "fp16sweep" else "gram")
        for d in ("ul", "dl"):
            if d == "ul":
                fn = lambda: eng.ul_detect(Hh, yh, n0=n0, K=K_SWEEPS, fusion="uniform")  # noqa: E731
                kfn = lambda: eng.ul_detect(Hh, yh, n0=n0, K=K_SWEEPS, want_xhat=False)  # noqa: E731
            else:
                fn = lambda: eng.dl_precode(Hh, xh, rho=rho, K=K_SWEEPS, want_gain=True)  # noqa: E731
                kfn = lambda: eng.dl_precode(Hh, xh, rho=rho, K=K_SWEEPS, want_gain=False)  # noqa: E731
            for _ in range(3):
                fn()
                kfn()  # both kernel instantiations warmed (first launch sets attributes)
            ms = _time_stream(fn, st, reps)
            kms = _time_stream(kfn, st, reps)
            ach = P * alg_bytes_per_problem(BC, U, esz) / (kms * 1e-3) / 1e9
            fcode = 0 if fmt == "fp32" else 1
            out[f"{d}_{fmt}"] = {"value": round(S * U * BITS / (ms * 1e-3) / 1e9, 4), "unit": "Gbps",
                                 "ms_per_batch": round(ms, 5), "kernel_ms": round(kms, 5),
                                 "roofline_frac": round(ach / hbm, 4), "achieved_GBps": round(ach, 1),
                                 "kernel": eng.kernel_name(0 if d == "ul" else 1, BC, U, fcode)}
    eng.set_fp16_algorithm("gram")
    # latency of one OFDM symbol's batch (1200 subcarriers x 8 clusters): eager vs CUDA graph
    from paper_1902_08653_b200 import GraphedUplink
    Hs, ys = H[:1200].contiguous(), y[:1200].contiguous()
    ef = lambda: eng.ul_detect(Hs, ys, n0=n0, K=K_SWEEPS, fusion="uniform")  # noqa: E731
    for _ in range(3):
        ef()
    eager_ms = _time_stream(ef, st, 50)
    g = GraphedUplink(eng, Hs, ys, n0=n0, K=K_SWEEPS)
    for _ in range(3):
        g.replay()
    graph_ms = _time_stream(g.replay, st, 50)
    out["ul_fp32_symbol_batch_latency"] = {"subcarriers": 1200, "eager_ms": round(eager_ms, 5),
                                           "cuda_graph_ms": round(graph_ms, 5),
                                           "value": round(1200 * U * BITS / (graph_ms * 1e-3) / 1e9, 4),
                                           "unit": "Gbps"}
    fn = lambda: eng.ul_detect(H, y, n0=n0, K=K_SWEEPS, fusion="optimal")  # noqa: E731
    fn()
    ms = _time_stream(fn, st, reps)
    out["ul_fp32_optimal_fusion"] = {"value": round(S * U * BITS / (ms * 1e-3) / 1e9, 4), "unit": "Gbps",
                                     "ms_per_batch": round(ms, 5),
                                     "note": "CD kernel + post-equalization variance (Gram+Cholesky) + fusion"}
    H16, y16 = to_fp16_pairs(H), to_fp16_pairs(y)
    fn = lambda: eng.ul_detect(H16, y16, n0=n0, K=K_SWEEPS, fusion="optimal")  # noqa: E731
    fn()
    ms = _time_stream(fn, st, reps)
    out["ul_fp16_optimal_fusion"] = {"value": round(S * U * BITS / (ms * 1e-3) / 1e9, 4), "unit": "Gbps",
                                     "ms_per_batch": round(ms, 5),
                                     "kernel": eng.kernel_name(0, BC, U, 1),
                                     "note": "Gram kernel with the variance fused (sweep operator on its Gram) + fusion"}
    eng.sync()
    return out


def measure_e2e(eng, dcd, part, H, y, n0, fusion, world, dev, n_e2e, barrier):
    """The metric end to end through the public API (Engine.ul_detect -> C ABI
    dcdg_ul_detect, or DistributedCD.uplink at N>1): every step copies its own
    pinned host H, y to the device (in chunks on a copy stream, overlapped with
    detection on a compute stream) and reads its fused estimates back to pinned
    host memory, and the host waits for each step's estimates.  Device inputs
    are double-buffered, so step i+1's copies are queued before the host
    consumes step i (a streaming receiver); plus the copy-only time of the same
    bytes (the PCIe bound of the step)."""
    import torch
    import torch.distributed as dist
    Hh = H.cpu().pin_memory()
    yh = y.cpu().pin_memory()
    Hd = [torch.empty_like(H), torch.empty_like(H)]
    yd = [torch.empty_like(y), torch.empty_like(y)]
    n_chunks = 8 if (world == 1 and part.S_local % 8 == 0) else 1
    cs = part.S_local // n_chunks
    copy_st, comp_st = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    own = part.own_hi - part.own_lo
    xh_host = [torch.empty((own, U), dtype=torch.complex64).pin_memory() for _ in range(2)]

    def copies(b, after=None):
        evs = []
        with torch.cuda.stream(copy_st):
            if after is not None:  # buffer b is free once the step that last read it is done
                copy_st.wait_event(after)
            for i in range(n_chunks):
                Hd[b][i * cs:(i + 1) * cs].copy_(Hh[i * cs:(i + 1) * cs], non_blocking=True)
                yd[b][i * cs:(i + 1) * cs].copy_(yh[i * cs:(i + 1) * cs], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy_st)
                evs.append(ev)
        return evs

    def e2e_step(b, after=None):
        evs = copies(b, after)
        with torch.cuda.stream(comp_st):
            if world == 1:
                for i in range(n_chunks):
                    comp_st.wait_event(evs[i])
                    r = eng.ul_detect(Hd[b][i * cs:(i + 1) * cs], yd[b][i * cs:(i + 1) * cs], n0=n0, K=K_SWEEPS,
                                      fusion=fusion, want_local=False, stream=comp_st)
                    xh_host[b][i * cs:(i + 1) * cs].copy_(r.xhat, non_blocking=True)
            else:
                comp_st.wait_event(evs[-1])
                out = dcd.uplink(Hd[b], yd[b], n0=n0, K=K_SWEEPS, fusion=fusion)
                xh_host[b].copy_(out, non_blocking=True)
            done = torch.cuda.Event()
            done.record(comp_st)
        return done

    e2e_step(0).synchronize()
    e2e_step(1).synchronize()
    barrier()
    t0, t1 = _ev(), _ev()
    torch.cuda.synchronize(dev)
    t0.record(copy_st)
    done = [None, None]
    done[0] = e2e_step(0)
    for i in range(n_e2e):
        if i + 1 < n_e2e:
            b = (i + 1) & 1
            done[b] = e2e_step(b, after=done[b])
        done[i & 1].synchronize()  # the host consumes step i's estimates
    t1.record(comp_st)
    barrier()
    e_ms = t0.elapsed_time(t1) / n_e2e
    if world > 1:
        t = torch.tensor([e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    h2d = H.numel() * H.element_size() + y.numel() * y.element_size()
    copies(0)
    torch.cuda.synchronize(dev)
    c0, c1 = _ev(), _ev()
    c0.record(copy_st)
    for i in range(n_e2e):
        copies(i & 1)
    c1.record(copy_st)
    torch.cuda.synchronize(dev)
    c_ms = c0.elapsed_time(c1) / n_e2e
    S_total = part.S
    return {"value": round(S_total * U * BITS / (e_ms * 1e-3) / 1e9, 5), "unit": "Gbps", "ms_per_step": round(e_ms, 4),
            "steps": n_e2e, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(own * U * 8),
            "h2d_copy_only_ms": round(c_ms, 4), "h2d_GBps": round(h2d / (c_ms * 1e-3) / 1e9, 2),
            "frac_of_copy_bound": round(c_ms / e_ms, 4),
            "path": "Engine.ul_detect (C ABI dcdg_ul_detect): pinned host H,y -> device in %d chunks on a copy "
                    "stream overlapped with detection -> pinned host fused estimates, host waits for every "
                    "step; device inputs double-buffered (step i+1's copies queued before the host consumes "
                    "step i)" % n_chunks}


PARITY_S = 96  # subcarriers of the bench batch re-checked against the reference after timing


def parity_check(eng, H, y, n0, fusion):
    """Outside every timed region: the fused estimates of the first PARITY_S
    subcarriers of the bench's own batch against the reference's
    decentralized_cd_detect (oracle/_ref, fp64) on the same values — the
    checker, never the measured path.  north_star tolerance 1e-5 (fp32)."""
    S = min(PARITY_S, H.shape[0])
    if _ref_lib() is None:
        return {"checked_subcarriers": 0, "note": "oracle/_ref/libdcdref.so missing"}
    r = eng.ul_detect(H[:S].contiguous(), y[:S].contiguous(), n0=n0, K=K_SWEEPS, fusion=fusion, want_local=False)
    got = r.xhat.cpu().numpy().astype(np.complex128)
    Hn = H[:S].cpu().numpy().astype(np.complex128)
    yn = y[:S].cpu().numpy().astype(np.complex128)
    c, u, bc = Hn.shape[1], Hn.shape[2], Hn.shape[3]
    ref = RefCPU(S, arrays=(Hn, yn, n0), c=c, u=u, bc=bc)
    want = np.zeros((S, u), np.complex128)
    try:
        ref.run(S, os.cpu_count() or 1, fusion=fusion, out=want)
    finally:
        ref.close()
    err = np.linalg.norm(got - want, axis=1) / np.maximum(np.linalg.norm(want, axis=1), 1e-300)
    worst = float(err.max())
    return {"checked_subcarriers": S, "max_rel_err": worst, "tol": 1e-5, "ok": bool(worst <= 1e-5),
            "against": "the reference's decentralized_cd_detect (oracle/_ref, fp64) on the bench's own first "
                       f"{S} subcarriers ({fusion} fusion), run after the timed regions"}


def configs0_line(eng, dev, hbm, reps):
    """BASELINE.json configs[0] (the reference's CPU-runnable case): uplink
    B=64, U=8, C=2 (B_c=32), 16-QAM, K=3, 1200x14 subcarrier-symbols; the GPU
    kernels next to the reference's decentralized_cd_detect on this host."""
    import torch
    u0, c0, bc0, S = 8, 2, 32, S_PER_GPU
    H, y, _, n0 = make_inputs(S, c0, dev, 77, u=u0, bc=bc0)
    st = torch.cuda.current_stream(dev)
    fn = lambda: eng.ul_detect(H, y, n0=n0, K=K_SWEEPS, fusion="uniform")  # noqa: E731
    kfn = lambda: eng.ul_detect(H, y, n0=n0, K=K_SWEEPS, want_xhat=False)  # noqa: E731
    for _ in range(3):
        fn()
        kfn()
    ms = _time_stream(fn, st, reps)
    kms = _time_stream(kfn, st, reps)
    ach = S * c0 * alg_bytes_per_problem(bc0, u0, 8) / (kms * 1e-3) / 1e9
    out = {"workload": "configs[0]: uplink CD B=64 U=8 C=2 (B_c=32), 16-QAM, K=3, 16,800 subcarrier-symbols, fp32, "
                       "uniform fusion", "value": round(S * u0 * BITS / (ms * 1e-3) / 1e9, 4), "unit": "Gbps",
           "ms_per_batch": round(ms, 5), "kernel_ms": round(kms, 5), "roofline_frac": round(ach / hbm, 4),
           "kernel": eng.kernel_name(0, bc0, u0, 0)}
    if _ref_lib() is not None:
        threads = os.cpu_count() or 1
        ref = RefCPU(2400, c=c0, u=u0, bc=bc0)
        try:
            out["reference_cpu"] = dict(_timed_mode(ref, threads, 2.0), kind="reference", cpu_model=cpu_model())
        finally:
            ref.close()
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1902_08653_b200 import Engine, kernel_name, to_fp16_pairs
    from paper_1902_08653_b200.distributed import CudaCompute, DistributedCD, partition

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_ONE_GPU=1 (harness self-test only): every rank on cuda:0 with the gloo
    # control plane, so the multi-rank p2p path runs on a one-GPU box
    one_gpu = os.environ.get("BENCH_ONE_GPU") == "1"
    if one_gpu:
        local_rank = 0
    elif world > torch.cuda.device_count():
        raise SystemExit(f"bench.py: {world} ranks but {torch.cuda.device_count()} visible GPU(s); one rank per GPU "
                         f"(BENCH_ONE_GPU=1 runs every rank on cuda:0 as a harness self-test only)")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    S_total = args.S * world  # weak scaling: per-GPU work fixed at args.S * C problems
    part = partition(C, world, rank, S_total)
    fmt = args.fmt
    esz = 8 if fmt == "fp32" else 4
    eng = Engine(local_rank)
    dcd = DistributedCD(part, CudaCompute(eng), mode=args.mode)

    H, y, _, n0 = make_inputs(part.S_local, part.C_local, dev, 1234 + rank)
    if fmt == "fp16":
        H, y = to_fp16_pairs(H), to_fp16_pairs(y)
    P = part.S_local * part.C_local
    stream = torch.cuda.current_stream(dev)

    # Multi-GPU: with the NCCL modes the fusion collective of batch i is left in
    # flight while batch i+1's detection kernel runs (NCCL stream vs compute
    # stream) and is waited on only when the next batch has been launched.  The
    # p2p mode has no collective: the CD kernel stores into the owners' windows.
    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def timed(d, steps, warmup, sample_clocks=False):
        pending = []

        def step():
            h = d.uplink(H, y, n0=n0, K=K_SWEEPS, fusion=args.fusion, async_op=world > 1)
            if world > 1:
                if pending:
                    pending.pop().wait()
                pending.append(h)

        def drain():
            while pending:
                pending.pop().wait()

        for _ in range(warmup):
            step()
        drain()
        eng.sync()
        barrier()
        l_a = eng.launches
        tr_a = (d.traffic.uplink_payload_bytes, d.traffic.uplink_bus_bytes, d.traffic.messages)
        # The K steps are captured once into a CUDA graph and the timed region
        # is its replay, so host launch overhead (and the clock sampler thread)
        # cannot starve the GPU between steps: at N=1, and at N>1 with the
        # peer-memory exchange (its batch epochs advance on the device, so the
        # replay publishes fresh epochs).  The NCCL modes run eagerly.
        graph = None
        if (world == 1 or getattr(d, "mode", None) == "p2p") and not args.eager:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                for _ in range(steps):
                    step()
            graph.replay()  # one untimed replay
            torch.cuda.synchronize(dev)
        n_launch = (eng.launches - l_a) // max(steps, 1) if graph is not None else None
        e0, e1 = _ev(), _ev()
        clk = ClockSampler(local_rank) if sample_clocks else None
        if clk:
            clk.__enter__()
        try:
            barrier()
            e0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                for _ in range(steps):
                    step()
                drain()
            e1.record(stream)
            barrier()
        finally:
            if clk:
                clk.__exit__(None, None, None)
        if n_launch is None:
            n_launch = (eng.launches - l_a) // max(steps, 1)
        tr = tuple((b - a) // max(steps, 1) for a, b in zip(
            tr_a, (d.traffic.uplink_payload_bytes, d.traffic.uplink_bus_bytes, d.traffic.messages)))
        t = e0.elapsed_time(e1) / steps
        if world > 1:
            tt = torch.tensor([t], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t, clk, n_launch, tr

    # (p2p: the first warm-up step maps the exchange windows, a one-time IPC handshake)
    mode_used, p2p_error = args.mode, None
    try:
        ms, clk, launches, (pay, bus, msgs) = timed(dcd, args.steps, args.warmup, sample_clocks=True)
    except Exception as e:
        # a box without CUDA-IPC peer mappings between its GPUs: every rank's
        # exchange fails (the waiting ranks by the kernel's own timeout), and the
        # line is measured with the NCCL reduce-scatter exchange instead,
        # recorded as such in config.parallelism and p2p_error
        if world == 1 or args.mode != "p2p":
            raise
        mode_used, p2p_error = "reduce", f"{type(e).__name__}: {e}"[:200]
        dcd = DistributedCD(part, CudaCompute(eng), mode=mode_used)
        ms, clk, launches, (pay, bus, msgs) = timed(dcd, args.steps, args.warmup, sample_clocks=True)
    compare = None
    if world > 1 and p2p_error is None:
        # the same step with the NCCL exchange of the other mode, for comparison
        other = "reduce" if args.mode == "p2p" else "p2p"
        try:
            d2 = DistributedCD(part, CudaCompute(eng), mode=other)
            ms2 = timed(d2, args.steps, args.warmup)[0]
            compare = {"mode": other, "ms_per_step": round(ms2, 5),
                       "value": round(S_total * U * BITS / (ms2 * 1e-3) / 1e9, 4), "unit": "Gbps"}
        except Exception as e:  # reported, never silently substituted for the main line
            compare = {"mode": other, "error": str(e)[:200]}
    # configs[2] across the GPUs: the distributed downlink step (symbol broadcast
    # from rank 0, local precoding, effective-gain exchange), same protocol
    downlink = None
    if world > 1 and fmt == "fp32":
        try:
            g_s = torch.Generator(device=dev)
            g_s.manual_seed(99)
            lv = torch.tensor([-3.0, -1.0, 1.0, 3.0], device=dev) / math.sqrt(10.0)
            idx = torch.randint(0, 4, (S_total, U, 2), device=dev, generator=g_s)
            s_sym = torch.complex(lv[idx[..., 0]], lv[idx[..., 1]]).contiguous()
            rho = math.sqrt(U)

            def dl_step():
                dcd.downlink(H, dcd.broadcast_symbols(s_sym), rho=rho, K=K_SWEEPS)

            for _ in range(args.warmup):
                dl_step()
            barrier()
            d0, d1 = _ev(), _ev()
            barrier()
            d0.record(stream)
            for _ in range(args.steps):
                dl_step()
            d1.record(stream)
            barrier()
            dms = d0.elapsed_time(d1) / args.steps
            tt = torch.tensor([dms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dms = float(tt.item())
            downlink = {"workload": "downlink CD ZF precoding + power split + effective gain (configs[2])",
                        "mode": mode_used, "ms_per_step": round(dms, 5),
                        "value": round(S_total * U * BITS / (dms * 1e-3) / 1e9, 4), "unit": "Gbps"}
        except Exception as e:  # reported, never silently substituted
            downlink = {"mode": mode_used, "error": str(e)[:200]}
    interconnect = {
        "payload_bytes_per_step_per_gpu": int(pay), "bus_bytes_per_step_per_gpu": int(bus),
        "messages_per_step_per_gpu": int(msgs),
        "model_total_bytes_per_step": int(pay * world),
        "raw_sample_forwarding_bytes_per_step": int(S_total * B * esz),
        "reduction_ratio": round(pay * world / (S_total * B * esz), 4),
        "note": "payload = the reference's MessageLog model for this GPU's clusters (U complex per cluster and "
                "subcarrier); bus = bytes this GPU sends to its peers per step (p2p: the estimates its CD kernel "
                "stores into other GPUs' exchange windows; NCCL modes: the collective's bus factor); 0 at N=1"}
    value = S_total * U * BITS / (ms * 1e-3) / 1e9  # whole-job Gbps: S_total subcarrier-symbols detected per step

    # dominant kernel alone (the CD kernel, same stream) for the roofline
    kfn = lambda: eng.ul_detect(H, y, n0=n0, K=K_SWEEPS, want_xhat=False)  # noqa: E731
    for _ in range(3):
        kfn()
    k_ms = _time_stream(kfn, stream, max(args.steps, 5))
    hbm, hbm_src = peaks()
    alg = P * alg_bytes_per_problem(BC, U, esz)
    achieved = alg / (k_ms * 1e-3) / 1e9

    n_e2e = max(3, min(args.steps, 10))
    e2e = measure_e2e(eng, dcd, part, H, y, n0, args.fusion, world, dev, n_e2e, barrier)
    h2d = e2e["h2d_bytes_per_step"]

    extra = None
    if rank == 0 and world == 1 and not args.fast:
        extra = secondary_lines(eng, dev, args.S, max(5, args.steps // 2), hbm)
        if fmt == "fp32":
            # the same e2e step with binary16 host buffers (half the PCIe bytes),
            # through the default fp16 kernel
            eng.set_fp16_algorithm("gram")
            e16 = measure_e2e(eng, None, part, to_fp16_pairs(H), to_fp16_pairs(y), n0, args.fusion, world, dev,
                              n_e2e, barrier)
            e16["kernel"] = kernel_name("ul", BC, U, "fp16")
            extra["e2e_fp16"] = e16
        extra["configs0"] = configs0_line(eng, dev, hbm, max(5, args.steps // 2))
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            key = f"ul_{fmt}_{BC}_{U}"
            if key in tj:
                traffic = int(tj[key]["dram_bytes_per_problem"] * P)
        except Exception:
            traffic = None
    line = {
        "metric": METRIC,
        "value": round(value, 4),
        "unit": "Gbps",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if fmt == "fp32" else "f16",
        "data": "synthetic: CN(0,1) Rayleigh H, Gray 16-QAM, AWGN at 10 dB, generated on device (torch RNG)",
        "config": {"workload": f"uplink CD L-MMSE detection + {args.fusion} fusion (configs[1])",
                   "B": B, "U": U, "C": C, "B_c": BC, "K": K_SWEEPS, "qam": QAM, "fmt": fmt,
                   "subcarrier_symbols_per_step": S_total, "problems_per_gpu": P, "clusters_per_gpu": part.C_local,
                   "parallelism": (f"clusters/{world}, fusion exchange {mode_used}" if world > 1
                                   else "single GPU, all clusters"),
                   "l2": f"inputs {alg / 1e6:.0f} MB/GPU > 126 MB L2, no flush needed",
                   "launch": ("one CUDA-graph replay of the K steps"
                              if (world == 1 or mode_used == "p2p") and not args.eager
                              else "eager, one host call per step"),
                   "kernel": kernel_name("ul", BC, U, fmt)},
        "batch_latency_ms": round(ms, 5),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "traffic": traffic, "peak_source": hbm_src,
                     "kernel_ms": round(k_ms, 5), "alg_bytes_per_launch": alg,
                     "alg_bytes_per_problem": alg_bytes_per_problem(BC, U, esz)},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "interconnect": interconnect,
    }
    if world > 1:
        # False: the fused peer-memory exchange could not run and the line was
        # measured with the NCCL reduce-scatter exchange instead
        line["p2p_ok"] = p2p_error is None and mode_used == "p2p"
        if one_gpu:
            line["harness_self_test"] = "BENCH_ONE_GPU=1: all ranks share cuda:0; not scaling data"
    if p2p_error:
        line["p2p_error"] = p2p_error
    if compare:
        line["exchange_comparison"] = compare
    if downlink:
        line["downlink_distributed"] = downlink
    if extra:
        line["extra"] = extra
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args.cpu_seconds)
    if rank == 0 and fmt == "fp32":
        line["parity"] = parity_check(eng, H, y, n0, args.fusion)
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# CPU reference (the unmodified reference library, oracle/_ref)
# ---------------------------------------------------------------------------
def _ref_lib():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        return None
    return Oracle("reference")


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_inputs(S, seed=5, c=C, u=U, bc=BC):
    """Host batch of the bench workload (configs[1]): H [S][C][U][B_c], y, and
    downlink symbols [S][U] (numpy, fp64 as the reference computes)."""
    rng = np.random.default_rng(seed)
    n0 = u * 1.0 / 10 ** (SNR_DB / 10)
    H = np.empty((S, c, u, bc), np.complex128)
    H.real = rng.standard_normal(H.shape)
    H.imag = rng.standard_normal(H.shape)
    H *= 1 / math.sqrt(2)
    lv = np.array([-3.0, -1.0, 1.0, 3.0]) / math.sqrt(10.0)
    x = lv[rng.integers(0, 4, (S, u))] + 1j * lv[rng.integers(0, 4, (S, u))]
    y = np.einsum("scub,su->scb", H, x) + math.sqrt(n0 / 2) * (
        rng.standard_normal((S, c, bc)) + 1j * rng.standard_normal((S, c, bc)))
    sym = lv[rng.integers(0, 4, (S, u))] + 1j * lv[rng.integers(0, 4, (S, u))]
    return np.ascontiguousarray(H), np.ascontiguousarray(y), np.ascontiguousarray(sym), n0


class RefCPU:
    """The reference's own decentralized_cd_detect / decentralized_cd_precode
    (oracle/_ref, compiled from the reference sources) over a host batch of S
    subcarriers, timed by the shim with contiguous subcarrier slices on
    `threads` std::threads (oracle/ref_shim.cpp dcdref_*_batch_run)."""

    def __init__(self, S, *, downlink=False, seed=5, c=C, u=U, bc=BC, arrays=None):
        import ctypes as Ct
        self.o = _ref_lib()
        self.L = self.o.lib
        if arrays is None:
            H, y, sym, self.n0 = cpu_inputs(S, seed, c, u, bc)
        else:  # (H [S][c][u][bc], y [S][c][bc], n0) from the caller
            H, y, self.n0 = (np.ascontiguousarray(arrays[0], np.complex128), np.ascontiguousarray(arrays[1], np.complex128),
                             arrays[2])
            sym = np.zeros((S, u), np.complex128)
        dp = Ct.POINTER(Ct.c_double)
        self.S, self.u = S, u
        self.ul = self.L.dcdref_ul_batch_create(S, c, bc, u, H.ctypes.data_as(dp), y.ctypes.data_as(dp))
        self.dl = (self.L.dcdref_dl_batch_create(S, c, bc, u, H.ctypes.data_as(dp), sym.ctypes.data_as(dp))
                   if downlink else None)
        self.backend = self.o.backend()

    def run(self, count, threads, *, direction="ul", fusion="uniform", concurrent=False, reps=1, first=0, out=None):
        import ctypes as Ct
        L = self.L
        L.dcdref_set_concurrent(1 if concurrent else 0)
        ts = []
        optr = out.ctypes.data_as(Ct.POINTER(Ct.c_double)) if out is not None else None
        try:
            for _ in range(reps):
                if direction == "ul":
                    t = L.dcdref_ul_batch_run(self.ul, self.n0, 1.0, K_SWEEPS, 1 if fusion == "uniform" else 0, 0, 0,
                                              threads, first, count, optr)
                else:
                    t = L.dcdref_dl_batch_run(self.dl, math.sqrt(self.u), K_SWEEPS, 0, 0, threads, first, count, None,
                                              None)
                if t < 0:
                    raise RuntimeError(L.dcdref_last_error().decode())
                ts.append(t)
        finally:
            L.dcdref_set_concurrent(0)
        return ts

    def close(self):
        self.L.dcdref_ul_batch_destroy(self.ul)
        if self.dl:
            self.L.dcdref_dl_batch_destroy(self.dl)


CPU_SAMPLE_S = 2400  # subcarrier-symbols of the CPU sample (x C = 19,200 cluster-problems, ~150 MB fp64)


def _timed_mode(ref, threads, target_s, **kw):
    """Gbps of one reference mode on a sample sized to ~target_s seconds."""
    u = ref.u
    probe = min(ref.S, max(threads * 2, 16))
    t0 = ref.run(probe, threads, **kw)[0]
    per_sc = max(t0 / probe, 1e-7)
    count = int(min(ref.S, max(probe, target_s / per_sc)))
    reps = max(1, int(target_s / (per_sc * count)))
    sec = sum(ref.run(count, threads, reps=reps, **kw))
    return {"value": round(count * reps * u * BITS / sec / 1e9, 6), "unit": "Gbps", "threads": threads,
            "subcarriers": count * reps, "seconds": round(sec, 3),
            "us_per_subcarrier_per_thread": round(sec * threads / (count * reps) * 1e6, 2)}


def cpu_baseline(target_s=10.0):
    """The reference's CPU path on this host: the headline (uplink, uniform
    fusion, all host threads, like the GPU arm) plus the SURVEY §8(d) matrix:
    1 thread, the reference's own concurrent=true mode, optimal fusion and the
    downlink decentralized_cd_precode."""
    threads = os.cpu_count() or 1
    if _ref_lib() is None:
        return {"value": None, "unit": "Gbps", "cores": threads, "kind": "reference",
                "sample": "oracle/_ref/libdcdref.so missing"}
    ref = RefCPU(CPU_SAMPLE_S, downlink=True)
    try:
        head = _timed_mode(ref, threads, target_s)
        side = max(1.0, target_s / 6)
        modes = {
            "ul_uniform_1thread": _timed_mode(ref, 1, side),
            "ul_uniform_concurrent_true": dict(_timed_mode(ref, 1, side, concurrent=True),
                                               note="one caller thread, the reference's concurrent=true "
                                                    "(a std::thread per cluster per call, detect.cpp:32-52)"),
            "ul_optimal_all_threads": _timed_mode(ref, threads, side, fusion="optimal"),
            "ul_optimal_1thread": _timed_mode(ref, 1, side, fusion="optimal"),
            "dl_all_threads": _timed_mode(ref, threads, side, direction="dl"),
            "dl_1thread": _timed_mode(ref, 1, side, direction="dl"),
        }
    finally:
        ref.close()
    return {"value": head["value"], "unit": "Gbps", "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": f"{head['subcarriers']} subcarrier-symbols (C={C} clusters each) through the reference's "
                      f"decentralized_cd_detect (uniform fusion, K=3, fp64) on {threads} std::threads, "
                      f"{head['seconds']:.2f} s, reference kernels backend={ref.backend}",
            "seconds": head["seconds"], "modes": modes}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if _ref_lib() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdcdref.so not built"}))
        return
    # the GPU arm's exact workload: S = 16,800 subcarrier-symbols per GPU (x N
    # GPUs, weak scaling), each through the reference's own
    # decentralized_cd_detect on all host threads
    S = args.S * world
    ref = RefCPU(S)
    try:
        ts = ref.run(S, threads, reps=args.warmup + args.steps)
    finally:
        ref.close()
    timed = ts[args.warmup:]
    sec = sum(timed) / len(timed)
    value = S * U * BITS / sec / 1e9
    line = {
        "metric": METRIC, "value": round(value, 6), "unit": "Gbps", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic CN(0,1) H / 16-QAM / AWGN (numpy), host-resident",
        "config": {"workload": "uplink CD L-MMSE detection + uniform fusion (configs[1])", "B": B, "U": U, "C": C,
                   "B_c": BC, "K": K_SWEEPS, "qam": QAM, "fmt": "fp64", "subcarrier_symbols_per_step": S},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 6), "unit": "Gbps", "cores": threads, "kind": "reference",
                         "cpu_model": cpu_model(),
                         "sample": f"the full step: {S} subcarrier-symbols (the GPU arm's per-step batch) through "
                                   f"decentralized_cd_detect on {threads} std::threads, backend={ref.backend}"},
        "e2e": {"value": round(value, 6), "unit": "Gbps", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _relaunch_torchrun(n: int) -> int:
    """`python bench.py --gpus N` without a torchrun environment: start N ranks
    (one per GPU) on this node with the same arguments; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--fmt", choices=["fp32", "fp16"], default="fp32")
    ap.add_argument("--fusion", choices=["uniform", "optimal"], default="uniform")
    ap.add_argument("--S", type=int, default=S_PER_GPU, help="subcarrier-symbols per GPU per step")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--eager", action="store_true", help="N=1: launch the K timed steps eagerly instead of one "
                                                         "CUDA-graph replay")
    ap.add_argument("--fast", action="store_true", help="skip the secondary (DL, fp16, optimal) lines")
    ap.add_argument("--mode", choices=["p2p", "reduce", "gather"], default="p2p",
                    help="multi-GPU fusion exchange: p2p = fused into the CD kernel over peer memory (NVLink), "
                         "reduce/gather = NCCL reduce-scatter / all-to-all after the CD kernel")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus < 1:
        raise SystemExit(f"bench.py: --gpus must be >= 1 (got {args.gpus})")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun
        sys.exit(_relaunch_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
                         f"(torchrun --nproc-per-node {args.gpus}) or drop WORLD_SIZE from the environment")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
