"""CPU, world_size > 1 on the gloo backend: the multi-GPU partitioner and the
fusion / broadcast / gain exchanges of paper_1902_08653_b200.distributed.

The per-rank CD compute is replaced by the CPU oracle (test infrastructure;
the product path runs CudaCompute = the CUDA kernels).  Every rank builds the
same reference batch, keeps only its clusters and subcarriers (the isolation
invariant: no H or y crosses ranks), and the exchanged results must equal the
single-process reference fusion (src/detect.cpp:180-187) and effective gain
(src/precode.cpp:123-131)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleCompute:
    """CPU stand-in for CudaCompute (tests only)."""

    def __init__(self, port):
        self.o = port

    def ul_local(self, H, y, *, n0, ex, K, fusion):
        Hn, yn = H.numpy().astype(np.complex128), y.numpy().astype(np.complex128)
        S, Cl, U, Bc = Hn.shape
        xl = np.zeros((S, Cl, U), np.complex128)
        s2 = np.zeros((S, Cl))
        for s in range(S):
            for c in range(Cl):
                xl[s, c] = self.o.cd_detect(Hn[s, c].T, yn[s, c], n0, ex, K)
                if fusion == "optimal":
                    s2[s, c] = self.o.post_eq_variance(Hn[s, c].T, n0, ex)
        return torch.from_numpy(xl), torch.from_numpy(s2)

    def ul_partial(self, H, y, *, n0, ex, K, fusion, C_total, want_local):
        xl, s2 = self.ul_local(H, y, n0=n0, ex=ex, K=K, fusion=fusion)
        if fusion == "optimal":
            w = 1.0 / s2
            return (w[..., None] * xl).sum(1), w.sum(1), xl, s2
        return xl.sum(1) / C_total, None, xl, s2

    def fuse(self, x_local, sigma2, *, fusion, C_total):
        if fusion == "optimal":
            w = (1.0 / sigma2) / (1.0 / sigma2).sum(1, keepdim=True)
        else:
            w = torch.full(x_local.shape[:2], 1.0 / C_total, dtype=torch.float64)
        acc = w[:, 0, None] * x_local[:, 0]
        for c in range(1, x_local.shape[1]):
            acc = acc + w[:, c, None] * x_local[:, c]
        return acc

    def dl(self, H, s, *, rho, K, C_total):
        Hn, sn = H.numpy().astype(np.complex128), s.numpy().astype(np.complex128)
        S, Cl, U, Bc = Hn.shape
        x = np.zeros((S, Cl, Bc), np.complex128)
        gp = np.zeros((S, Cl))
        for i in range(S):
            for c in range(Cl):
                xc = self.o.cd_precode(Hn[i, c].conj(), sn[i], K)
                xc = self.o.power_scale(xc, rho / np.sqrt(C_total))
                x[i, c] = xc
                gp[i, c] = np.real(np.vdot(Hn[i, c].T @ sn[i], xc))  # Re(s^H H_dl x) = Re((H s)^H x)
        return torch.from_numpy(x), torch.from_numpy(gp).float()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, C, Bc, U, S, mode, fusion, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from helpers import batch
        from oracle.oracle import Oracle
        from paper_1902_08653_b200.distributed import DistributedCD, partition

        b = batch(C, Bc, U, S=S, seed=3)
        part = partition(C, world, rank, S)
        H = torch.from_numpy(b["h_tiles"][part.s_lo:part.s_hi, part.c_lo:part.c_hi].copy())
        y = torch.from_numpy(b["y"][part.s_lo:part.s_hi, part.c_lo:part.c_hi].copy())
        eng = DistributedCD(part, OracleCompute(Oracle("port")), mode=mode)
        xh = eng.uplink(H, y, n0=b["n0"], K=3, fusion=fusion)
        s_root = torch.from_numpy(b["x_true"].copy()) if rank == 0 else torch.zeros(b["x_true"].shape,
                                                                                     dtype=torch.complex128)
        s = eng.broadcast_symbols(s_root)
        x, gain = eng.downlink(H, s, rho=float(np.sqrt(U)), K=3)
        t = eng.traffic
        q.put((rank, part.own_lo, part.own_hi, xh.numpy(), part.s_lo, part.s_hi, part.c_lo, part.c_hi, x.numpy(),
               gain.numpy(), {k: v for k, v in vars(t).items() if k != "collectives"}))
    finally:
        dist.destroy_process_group()


def _run(world, C, Bc, U, S, mode, fusion):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, C, Bc, U, S, mode, fusion, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,C,mode,fusion", [
    (2, 8, "reduce", "uniform"),
    (2, 8, "reduce", "optimal"),
    (4, 8, "gather", "uniform"),
    (2, 4, "gather", "optimal"),
    (4, 2, "reduce", "uniform"),   # more GPUs than clusters: subcarrier replicas
])
def test_distributed_matches_single_process_reference(world, C, mode, fusion, port):
    Bc, U, S = 16, 4, 8
    from helpers import batch
    from oracle.oracle import OPTIMAL, UNIFORM
    b = batch(C, Bc, U, S=S, seed=3)
    xhat_ref, _, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, OPTIMAL if fusion == "optimal" else UNIFORM)
    x_ref, g_ref = port.dl_precode_batch(b["h_tiles"], b["x_true"], float(np.sqrt(U)), 3)
    res = _run(world, C, Bc, U, S, mode, fusion)
    covered = np.zeros(S, bool)
    for (rank, lo, hi, xh, s_lo, s_hi, c_lo, c_hi, x, gain, _) in res:
        assert np.allclose(xh, xhat_ref[lo:hi], rtol=0, atol=1e-12), (rank, np.abs(xh - xhat_ref[lo:hi]).max())
        covered[lo:hi] = True
        assert np.allclose(x, x_ref[s_lo:s_hi, c_lo:c_hi], rtol=0, atol=1e-12)
        assert np.allclose(gain, g_ref, rtol=1e-6, atol=0)  # fp32 gain accumulator
    assert covered.all()  # every subcarrier's fused estimate is owned by exactly one rank


def test_partition_layouts():
    from paper_1902_08653_b200.distributed import partition
    ps = [partition(8, 2, r, 16) for r in range(2)]
    assert [list(p.clusters) for p in ps] == [[0, 1, 2, 3], [4, 5, 6, 7]]
    assert [(p.own_lo, p.own_hi) for p in ps] == [(0, 8), (8, 16)]
    ps = [partition(2, 4, r, 16) for r in range(4)]
    assert [(p.c_lo, p.s_lo, p.s_hi) for p in ps] == [(0, 0, 8), (0, 8, 16), (1, 0, 8), (1, 8, 16)]
    assert sorted((p.own_lo, p.own_hi) for p in ps) == [(0, 4), (4, 8), (8, 12), (12, 16)]
    with pytest.raises(ValueError):
        partition(8, 3, 0, 16)
    with pytest.raises(ValueError):
        partition(8, 2, 0, 15)


def test_interconnect_accounting_matches_the_message_model():
    """the payload each rank's clusters put on the
    interconnect equals the reference's MessageLog model (test_cluster.cpp:201-230
    KAT: B=128, C=4, U=8, 1200 subcarriers -> 307200 bytes in fp32; the CPU
    stand-in exchanges complex128, i.e. the fp64 model, twice that), and the
    bus bytes follow the collectives actually issued."""
    from paper_1902_08653_b200.distributed import Traffic, interconnect_summary
    S, C, Bc, U, W = 1200, 4, 32, 8, 2
    res = _run(W, C, Bc, U, S, "gather", "uniform")
    tr = []
    for r in res:
        t = Traffic(**r[-1])
        tr.append(t)
        assert t.uplink_bus_bytes == (S // W) * W * (C // W) * U * 16 // 2  # all-to-all of x_local, half stays local
        assert t.downlink_bus_bytes == S * U * 16 + 2 * (W - 1) * S * 4 // W  # symbol broadcast + gain all-reduce
    summ = interconnect_summary(tr, total_antennas=C * Bc, subcarriers=S, bpc=16)
    assert summ["uplink_bytes"] == 2 * 307200
    assert summ["downlink_bytes"] == S * C * U * 16
    assert summ["messages"] == 2 * S * C
    assert summ["reduction_ratio"] == pytest.approx(2 * U / Bc / 1)  # (U up + U down) per cluster vs B_c samples


def test_p2p_mode_needs_one_gpu_per_cluster_at_most():
    """The fused peer-memory exchange owns whole clusters per rank (world <= C)."""
    from paper_1902_08653_b200.distributed import DistributedCD, partition
    with pytest.raises(ValueError, match="at most one GPU per cluster"):
        DistributedCD(partition(2, 4, 0, 16), None, mode="p2p")
    with pytest.raises(ValueError, match="mode must be"):
        DistributedCD(partition(2, 2, 0, 16), None, mode="nccl")
