"""Multi-GPU decentralized CD: antenna clusters mapped onto the GPUs of one
node, one process per GPU, NCCL (torch.distributed) for the only data that
crosses GPUs — the U-vector fusion payloads (uplink) and the symbol broadcast
plus the effective-gain scalars (downlink).  Channel tiles and receive samples
never leave their GPU (the isolation invariant of SPEC.md:440).

Reference behaviour this distributes (paths relative to /root/reference/proj):
  per-cluster workers          run_cluster_workers   src/detect.cpp:32-52
  uplink fusion (ascending c)  decentralized_cd_detect src/detect.cpp:178-187
  downlink broadcast + power   decentralized_cd_precode src/precode.cpp:153-168
  effective gain               assemble_blocks        src/precode.cpp:115-132

Partitioning (ClusterPartition):
  world <= C_total: rank r owns clusters [r*C/W, (r+1)*C/W) for all S
      subcarriers of the batch; fused outputs are owned by subcarrier chunks
      [r*S/W, (r+1)*S/W).
  world >  C_total: each cluster is served by R = W/C ranks (rank = c*R + i),
      rank (c, i) computes subcarriers [i*S/R, (i+1)*S/R) of cluster c.

Uplink fusion modes:
  "reduce"  each rank forms its partial fused sum in the fusion kernel
            (uniform: sum_c x_c / C; optimal: sum_c x_c/sigma_c^2 and
            sum_c 1/sigma_c^2) and the partials are reduce-scattered over
            the subcarrier axis.  One collective, fp32 sum order = NCCL's.
  "gather"  the per-cluster estimates are exchanged all-to-all so the owner of
            each subcarrier chunk holds all C estimates in ascending cluster
            order and runs the ordinary fusion kernel: the reference's exact
            ascending-c summation order, independent of the GPU count.
  "p2p"     the gather exchange fused into the CD kernel over peer memory
            (NVLink P2P, CUDA IPC windows; include/dcdg.h dcdg_ul_detect_xchg):
            the kernel's epilogue stores each x_c into the owner's window, its
            last CTA publishes the batch epoch, the owner fuses once every rank
            has published.  No NCCL call on the data path; bitwise the
            single-GPU result.  Needs world <= C_total and CudaCompute.

The per-rank compute is pluggable (`compute` objects below): CudaCompute runs
the CD kernels (libdcdg.so); tests substitute a CPU checker to exercise the
partitioning and collectives on the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class ClusterPartition:
    C_total: int
    world: int
    rank: int
    S: int
    c_lo: int
    c_hi: int
    s_lo: int   # subcarrier range this rank computes
    s_hi: int
    own_lo: int  # fused-output subcarriers this rank owns (uplink)
    own_hi: int

    @property
    def clusters(self):
        return range(self.c_lo, self.c_hi)

    @property
    def C_local(self):
        return self.c_hi - self.c_lo

    @property
    def S_local(self):
        return self.s_hi - self.s_lo

    @property
    def replicas(self):
        return max(1, self.world // self.C_total)


def partition(C_total: int, world: int, rank: int, S: int) -> ClusterPartition:
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    if world <= C_total:
        if C_total % world:
            raise ValueError(f"{C_total} clusters cannot be split evenly over {world} GPUs")
        if S % world:
            raise ValueError(f"batch of {S} subcarriers must divide over {world} GPUs")
        per = C_total // world
        chunk = S // world
        return ClusterPartition(C_total, world, rank, S, rank * per, (rank + 1) * per, 0, S, rank * chunk,
                                (rank + 1) * chunk)
    if world % C_total:
        raise ValueError(f"{world} GPUs cannot serve {C_total} clusters evenly")
    R = world // C_total
    if S % world:
        raise ValueError(f"batch of {S} subcarriers must divide over {world} GPUs")
    c, i = divmod(rank, R)
    sl = S // R
    # the C ranks sharing slice i reduce-scatter it further into S/world chunks
    chunk = S // world
    own_lo = i * sl + c * chunk
    return ClusterPartition(C_total, world, rank, S, c, c + 1, i * sl, (i + 1) * sl, own_lo, own_lo + chunk)


class _Groups:
    """Process groups of the ranks that share a subcarrier slice (world > C)."""

    def __init__(self, part: ClusterPartition):
        self.group = None
        if part.world > part.C_total:
            R = part.replicas
            for i in range(R):
                ranks = [c * R + i for c in range(part.C_total)]
                g = dist.new_group(ranks)
                if part.rank in ranks:
                    self.group = g


# ---------------------------------------------------------------------------
# interconnect accounting
# ---------------------------------------------------------------------------
def bytes_per_complex(t: torch.Tensor) -> int:
    """Wire size of one complex element of a payload tensor (precision.cpp:8-15):
    complex128 16, complex64 8, binary16 pair 4."""
    if t.dtype == torch.complex128:
        return 16
    if t.dtype == torch.complex64:
        return 8
    if t.dtype == torch.float16:
        return 4
    raise ValueError(f"no complex wire format for {t.dtype}")


@dataclass
class Traffic:
    """What this rank's exchanges moved.

    payload: the reference's MessageLog model (make_message, cluster.cpp:9-22)
      for this rank's clusters: uplink U complex (+1 real for optimal fusion)
      per cluster and subcarrier, downlink U complex per cluster and
      subcarrier (the symbol broadcast).
    bus: bytes per rank on the interconnect for the collectives actually issued,
      with the NCCL-tests bus-bandwidth factors: reduce-scatter / all-to-all /
      all-gather (W-1)/W of the buffer, broadcast the buffer, all-reduce
      2(W-1)/W (the p2p exchanges are accounted as the collective they replace)."""
    uplink_payload_bytes: int = 0
    downlink_payload_bytes: int = 0
    uplink_bus_bytes: int = 0
    downlink_bus_bytes: int = 0
    messages: int = 0
    collectives: list = field(default_factory=list)

    def add_bus(self, kind: str, nbytes: int, world: int, uplink: bool):
        f = {"reduce_scatter": (world - 1) / world, "all_to_all": (world - 1) / world, "broadcast": 1.0,
             "all_gather": (world - 1) / world, "all_reduce": 2 * (world - 1) / world}[kind] if world > 1 else 0.0
        b = int(round(f * nbytes))
        if uplink:
            self.uplink_bus_bytes += b
        else:
            self.downlink_bus_bytes += b
        self.collectives.append((kind, nbytes))


def interconnect_summary(traffic, total_antennas: int, subcarriers: int, bpc: int) -> dict:
    """interconnect_summary (cluster.cpp:42-68) over one or more ranks' Traffic:
    totals of the message model and the reduction ratio against forwarding every
    antenna sample (B * S complex); plus the bus bytes actually moved."""
    ts = traffic if isinstance(traffic, (list, tuple)) else [traffic]
    up = sum(t.uplink_payload_bytes for t in ts)
    down = sum(t.downlink_payload_bytes for t in ts)
    base = total_antennas * subcarriers * bpc
    return {"messages": sum(t.messages for t in ts), "uplink_bytes": up, "downlink_bytes": down,
            "total_bytes": up + down, "baseline_bytes": base,
            "reduction_ratio": (up + down) / base if base else 0.0,
            "uplink_bus_bytes": sum(t.uplink_bus_bytes for t in ts),
            "downlink_bus_bytes": sum(t.downlink_bus_bytes for t in ts)}


# ---------------------------------------------------------------------------
# per-rank compute back-ends
# ---------------------------------------------------------------------------
class CudaCompute:
    """The CD kernels through the C ABI (libdcdg.so) on this rank's GPU."""

    def __init__(self, engine):
        self.eng = engine

    def ul_partial(self, H, y, *, n0, ex, K, fusion, C_total, want_local):
        """-> (partial [S,U] complex64, wsum [S] or None, x_local, sigma2)."""
        r = self.eng.ul_detect(H, y, n0=n0, ex=ex, K=K, fusion=fusion, C_total=C_total, want_local=True)
        return r.xhat, r.wsum, r.x_local, r.sigma2

    def ul_local(self, H, y, *, n0, ex, K, fusion):
        r = self.eng.ul_detect(H, y, n0=n0, ex=ex, K=K, fusion=fusion, want_xhat=False)
        if fusion == "optimal" and r.sigma2 is None:
            raise RuntimeError("optimal fusion needs sigma2")
        return r.x_local, r.sigma2

    def fuse(self, x_local, sigma2, *, fusion, C_total):
        return self.eng.fuse(x_local, sigma2, fusion=fusion, C_total=C_total)

    def dl(self, H, s, *, rho, K, C_total):
        r = self.eng.dl_precode(H, s, rho=rho, K=K, C_total=C_total, want_gain=True)
        return r.x, r.gain_part


# ---------------------------------------------------------------------------
# the distributed path
# ---------------------------------------------------------------------------
class DistributedCD:
    def __init__(self, part: ClusterPartition, compute, *, mode: str = "reduce"):
        if mode not in ("reduce", "gather", "p2p"):
            raise ValueError("mode must be 'reduce', 'gather' or 'p2p'")
        if mode == "p2p" and part.world > part.C_total:
            raise ValueError("the p2p exchange needs at most one GPU per cluster (world <= C_total)")
        self.part = part
        self.compute = compute
        self.mode = mode
        self._groups = _Groups(part)
        self.traffic = Traffic()
        self._xwin = None
        self._xkey = None

    def _log_uplink(self, S_local: int, U: int, bpc: int, optimal: bool):
        p = self.part
        self.traffic.uplink_payload_bytes += S_local * p.C_local * (U * bpc + (bpc // 2 if optimal else 0))
        self.traffic.messages += S_local * p.C_local

    # ---- uplink -----------------------------------------------------------
    def uplink(self, H, y, *, n0, ex=1.0, K=3, fusion="uniform", async_op=False):
        """H: [S_local, C_local, U, Bc], y: [S_local, C_local, Bc] for this rank's
        clusters and subcarriers.  Returns the fused estimates of the subcarriers
        this rank owns, [own_hi-own_lo, U] complex64 (plus the Work handle when
        async_op)."""
        p = self.part
        if p.world == 1:
            # one call: the CD kernel and the ascending-cluster fusion (launched as
            # its programmatic dependent inside dcdg_ul_detect)
            out, wsum, xl, _ = self.compute.ul_partial(H, y, n0=n0, ex=ex, K=K, fusion=fusion, C_total=p.C_total,
                                                       want_local=True)
            if wsum is not None:  # a compute that leaves the optimal weights' sum to the caller
                out = out / wsum.reshape(-1, 1)
            self._log_uplink(xl.shape[0], xl.shape[-1] if xl.dtype != torch.float16 else xl.shape[-2],
                             bytes_per_complex(xl), fusion == "optimal")
            return _Deferred(None, lambda: out) if async_op else out
        if self.mode == "p2p":
            return self._uplink_p2p(H, y, n0=n0, ex=ex, K=K, fusion=fusion, async_op=async_op)
        if self.mode == "gather" and p.world <= p.C_total:
            return self._uplink_gather(H, y, n0=n0, ex=ex, K=K, fusion=fusion, async_op=async_op)
        part_sum, wsum, _, _ = self.compute.ul_partial(H, y, n0=n0, ex=ex, K=K, fusion=fusion, C_total=p.C_total,
                                                       want_local=False)
        U = part_sum.shape[-1]
        self._log_uplink(part_sum.shape[0], U, bytes_per_complex(part_sum), fusion == "optimal")
        flat = torch.view_as_real(part_sum).reshape(part_sum.shape[0], 2 * U)
        if fusion == "optimal":
            flat = torch.cat([flat, wsum.reshape(-1, 1), torch.zeros_like(wsum).reshape(-1, 1)], dim=1)
        W = p.world if p.world <= p.C_total else p.C_total
        rows = flat.shape[0] // W
        out = torch.empty((rows, flat.shape[1]), dtype=flat.dtype, device=flat.device)
        work = dist.reduce_scatter_tensor(out.reshape(-1), flat.contiguous().reshape(-1), op=dist.ReduceOp.SUM,
                                          group=self._groups.group, async_op=async_op)
        self.traffic.add_bus("reduce_scatter", flat.numel() * flat.element_size(), W, True)

        def finish():
            if fusion == "optimal":
                num = torch.view_as_complex(out[:, : 2 * U].reshape(rows, U, 2).contiguous())
                return num / out[:, 2 * U].reshape(rows, 1)
            return torch.view_as_complex(out.reshape(rows, U, 2).contiguous())

        if async_op:
            return _Deferred(work, finish)
        return finish()

    def _window(self, U: int, fmt: str):
        """Create this rank's exchange window and map every peer's (one
        all_gather of the 64-byte IPC handles; collective, all ranks call)."""
        from .engine import ExchangeWindow
        p = self.part
        key = (p.S, U, fmt)
        if self._xwin is None or self._xkey != key:
            if self._xwin is not None:
                self._xwin.close()
            self._xwin = ExchangeWindow(self.compute.eng, p.world, p.rank, S=p.S, C_total=p.C_total, U=U, fmt=fmt)
            handles = [None] * p.world
            dist.all_gather_object(handles, self._xwin.handle())
            for q, h in enumerate(handles):
                self._xwin.open(q, h)
            dist.barrier()
            self._xkey = key
        return self._xwin

    def _uplink_p2p(self, H, y, *, n0, ex, K, fusion, async_op):
        p = self.part
        if not hasattr(self.compute, "eng"):
            raise ValueError("the p2p exchange runs the CUDA kernels (CudaCompute)")
        fp16 = H.dtype == torch.float16
        U = H.shape[2]
        esz = 4 if fp16 else 8
        w = self._window(U, "fp16" if fp16 else "fp32")
        out = w.ul_detect(H, y, c0=p.c_lo, C_total=p.C_total, n0=n0, ex=ex, K=K, fusion=fusion)
        S_local = H.shape[0]
        self._log_uplink(S_local, U, esz, fusion == "optimal")
        nbytes = S_local * p.C_local * (U * esz + (4 if fusion == "optimal" else 0))
        self.traffic.add_bus("all_to_all", nbytes, p.world, True)
        return _Deferred(None, lambda: out) if async_op else out

    def _uplink_gather(self, H, y, *, n0, ex, K, fusion, async_op):
        p = self.part
        xl, s2 = self.compute.ul_local(H, y, n0=n0, ex=ex, K=K, fusion=fusion)
        self._log_uplink(xl.shape[0], xl.shape[2], bytes_per_complex(xl), fusion == "optimal")
        # x_local [S, C_loc, U] (complex64 or f16 pairs) -> chunk r of the subcarriers to rank r
        send = xl.contiguous()
        self.traffic.add_bus("all_to_all", send.numel() * send.element_size(), p.world, True)
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv.reshape(-1) if recv.dtype != torch.complex64 else torch.view_as_real(recv).reshape(-1),
                               send.reshape(-1) if send.dtype != torch.complex64 else torch.view_as_real(send).reshape(-1))
        chunk = p.S // p.world
        # recv holds, for each source rank q, its C_loc clusters of MY subcarrier chunk, in rank order
        recv = recv.reshape(p.world, chunk, p.C_local, *xl.shape[2:]).transpose(0, 1).reshape(
            chunk, p.C_total, *xl.shape[2:]).contiguous()
        sig = None
        if fusion == "optimal":
            ssend = s2.contiguous()
            self.traffic.add_bus("all_to_all", ssend.numel() * ssend.element_size(), p.world, True)
            srecv = torch.empty_like(ssend)
            dist.all_to_all_single(srecv.reshape(-1), ssend.reshape(-1))
            sig = srecv.reshape(p.world, chunk, p.C_local).transpose(0, 1).reshape(chunk, p.C_total).contiguous()
        out = self.compute.fuse(recv, sig, fusion=fusion, C_total=p.C_total)
        return _Deferred(None, lambda: out) if async_op else out

    # ---- downlink ---------------------------------------------------------
    def broadcast_symbols(self, s_root, *, src=0):
        """Root's [S, U] symbol batch to every rank (the centre -> cluster
        broadcast, src/cluster.cpp:256-259).  In p2p mode the broadcast is part
        of downlink() (NVLink stores into every window), so this is a no-op."""
        if self.mode == "p2p":
            return s_root
        buf = s_root if not s_root.is_complex() else torch.view_as_real(s_root)
        dist.broadcast(buf, src)
        self.traffic.add_bus("broadcast", buf.numel() * buf.element_size(), self.part.world, False)
        return s_root

    def downlink(self, H, s, *, rho, K=3):
        """H: [S_local, C_local, U, Bc]; s: the broadcast [S, U] batch.  Returns
        (x_local [S_local, C_local, Bc], effective gain [S] on every rank)."""
        p = self.part
        if self.mode == "p2p":
            return self._downlink_p2p(H, s, rho=rho, K=K)
        s_mine = s[p.s_lo:p.s_hi].contiguous()
        U = s.shape[1]
        self.traffic.downlink_payload_bytes += s_mine.shape[0] * p.C_local * U * bytes_per_complex(s)
        self.traffic.messages += s_mine.shape[0] * p.C_local
        x, gpart = self.compute.dl(H, s_mine, rho=rho, K=K, C_total=p.C_total)
        num = torch.zeros((p.S,), dtype=torch.float32, device=gpart.device)
        num[p.s_lo:p.s_hi] = gpart.sum(dim=1)
        if p.world > 1:
            dist.all_reduce(num)
            self.traffic.add_bus("all_reduce", num.numel() * num.element_size(), p.world, False)
        sf = s.float() if s.dtype == torch.float16 else torch.view_as_real(s)
        se = (sf.reshape(p.S, -1) ** 2).sum(dim=1)
        gain = torch.where(se > 0, num / torch.where(se > 0, se, torch.ones_like(se)), torch.zeros_like(se))
        return x, gain


    def _downlink_p2p(self, H, s, *, rho, K):
        """decentralized_cd_precode's exchanges over peer memory
        (dcdg_dl_precode_xchg): rank 0 (the centre) stores its symbols into
        every window, every rank precodes its clusters from its own window and
        gathers all C_total gain shares; no NCCL call."""
        p = self.part
        if not hasattr(self.compute, "eng"):
            raise ValueError("the p2p exchange runs the CUDA kernels (CudaCompute)")
        fp16 = H.dtype == torch.float16
        U = H.shape[2]
        esz = 4 if fp16 else 8
        w = self._window(U, "fp16" if fp16 else "fp32")
        x, gain = w.dl_precode(H, s if p.rank == 0 else None, root=0, c0=p.c_lo, C_total=p.C_total, rho=rho, K=K)
        self.traffic.downlink_payload_bytes += p.S * p.C_local * U * esz
        self.traffic.messages += p.S * p.C_local
        self.traffic.add_bus("broadcast", p.S * U * esz, p.world, False)
        self.traffic.add_bus("all_gather", p.S * p.C_total * 4, p.world, False)
        return x, gain


class _Deferred:
    """Async collective + the epilogue that turns its output into estimates."""

    def __init__(self, work, finish):
        self.work, self._finish = work, finish

    def wait(self):
        if self.work is not None:
            self.work.wait()
        return self._finish()
