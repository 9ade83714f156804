"""Fused cross-GPU exchange (include/dcdg.h dcdg_ul_detect_xchg): the uplink
CD kernel stores each cluster estimate straight into the exchange window of
the rank owning the subcarrier (peer memory, CUDA IPC) and the owner fuses in
ascending cluster order (detect.cpp:180-187).

The result must be BITWISE the single-GPU dcdg_ul_detect result (same
per-problem arithmetic, same fusion order), and within the fp32/fp16
tolerance of the CPU oracle.  The gpurun box has one GPU, so the multi-rank
case runs two processes on cuda:0: the windows are mapped by CUDA IPC and the
stores/flags go through the same code as over NVLink.
"""
import os
import socket

import numpy as np
import pytest
import torch

from helpers import OPTIMAL, TOL_FP32, UNIFORM, batch, rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


def _single(engine, H, y, *, fusion, n0):
    r = engine.ul_detect(H, y, n0=n0, K=3, fusion=fusion, want_local=False)
    engine.sync()
    return r.xhat


@pytest.mark.parametrize("shape,fmt,fusion", [
    ((8, 32, 16), "fp32", "uniform"),   # fused epilogue (ul_reg_f32)
    ((8, 32, 16), "fp16", "uniform"),   # fused epilogue (ul_reg_f16)
    ((8, 32, 16), "fp32", "optimal"),   # CD + variances, then xchg_put_kernel
    ((8, 32, 16), "fp16", "optimal"),   # Gram kernel with fused variances, then xchg_put_kernel
    ((2, 256, 16), "fp32", "uniform"),  # multi-warp kernel: xchg_put_kernel path
    ((3, 24, 6), "fp32", "uniform"),    # generic kernel
])
def test_single_rank_window_is_bitwise_single_gpu(engine, port, shape, fmt, fusion):
    from paper_1902_08653_b200 import ExchangeWindow
    C, BC, U = shape
    S = 96
    b = batch(C, BC, U, 16, S, seed=11)
    H, y = to_dev(b["h_tiles"], fmt, pairs=True), to_dev(b["y"], fmt, pairs=True)
    want = _single(engine, H, y, fusion=fusion, n0=b["n0"])
    w = ExchangeWindow(engine, 1, 0, S=S, C_total=C, U=U, fmt=fmt)
    w.open(0, w.handle())  # own window: a no-op, like the peers' loop in DistributedCD
    for _ in range(3):  # both parities and the epoch counter
        got = w.ul_detect(H, y, c0=0, C_total=C, n0=b["n0"], K=3, fusion=fusion)
        engine.sync()
        assert torch.equal(torch.view_as_real(got), torch.view_as_real(want))
    if fmt == "fp32":
        xhat, _, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3,
                                          OPTIMAL if fusion == "optimal" else UNIFORM)
        assert rel_err(to_host(got), xhat) <= TOL_FP32
    w.close()


@pytest.mark.parametrize("fusion", ["uniform", "optimal"])
def test_exchange_calls_replay_from_a_cuda_graph(engine, fusion):
    """The batch epochs advance on the device, so exchange calls captured once
    into a CUDA graph (uplink, downlink, uplink: both parities, both
    directions) replay with fresh epochs: every replay bitwise the eager
    single-GPU results."""
    from helpers import qam_symbols
    from paper_1902_08653_b200 import ExchangeWindow
    C, BC, U, S = 8, 32, 16, 64
    b = batch(C, BC, U, 16, S, seed=13)
    H, y = to_dev(b["h_tiles"]), to_dev(b["y"])
    sym = to_dev(qam_symbols(S, U))
    want_ul = _single(engine, H, y, fusion=fusion, n0=b["n0"])
    want_dl = engine.dl_precode(H, sym, rho=4.0, K=3, want_gain=True)
    engine.sync()
    w = ExchangeWindow(engine, 1, 0, S=S, C_total=C, U=U, fmt="fp32")
    # warm up eagerly (scratch allocation, kernel attributes), then capture
    w.ul_detect(H, y, c0=0, C_total=C, n0=b["n0"], K=3, fusion=fusion)
    w.dl_precode(H, sym, root=0, c0=0, C_total=C, rho=4.0, K=3)
    engine.sync()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        u1 = w.ul_detect(H, y, c0=0, C_total=C, n0=b["n0"], K=3, fusion=fusion)
        x, gain = w.dl_precode(H, sym, root=0, c0=0, C_total=C, rho=4.0, K=3)
        u2 = w.ul_detect(H, y, c0=0, C_total=C, n0=b["n0"], K=3, fusion=fusion)
    for _ in range(3):
        for t in (u1, u2, x, gain):
            t.zero_()
        g.replay()
        engine.sync()
        assert torch.equal(torch.view_as_real(u1), torch.view_as_real(want_ul))
        assert torch.equal(torch.view_as_real(u2), torch.view_as_real(want_ul))
        assert torch.equal(x.view(torch.float32), want_dl.x.view(torch.float32))
        assert torch.equal(gain, want_dl.gain)
    w.close()


@pytest.mark.parametrize("shape,fmt", [((8, 32, 16), "fp32"), ((8, 32, 16), "fp16"), ((2, 64, 8), "fp32"),
                                       ((3, 24, 6), "fp32")])
def test_single_rank_downlink_window_is_bitwise_single_gpu(engine, port, shape, fmt):
    from helpers import qam_symbols
    from paper_1902_08653_b200 import ExchangeWindow
    C, BC, U = shape
    S = 64
    b = batch(C, BC, U, 16, S, seed=12)
    H = to_dev(b["h_tiles"], fmt, pairs=True)
    sym = to_dev(qam_symbols(S, U), fmt)
    rho = float(np.sqrt(U))
    want = engine.dl_precode(H, sym, rho=rho, K=3, want_gain=True)
    engine.sync()
    w = ExchangeWindow(engine, 1, 0, S=S, C_total=C, U=U, fmt=fmt)
    for _ in range(3):
        x, gain = w.dl_precode(H, sym, root=0, c0=0, C_total=C, rho=rho, K=3)
        engine.sync()
        assert torch.equal(x.view(torch.float32) if x.dtype != torch.float16 else x,
                           want.x.view(torch.float32) if want.x.dtype != torch.float16 else want.x)
        assert torch.equal(gain, want.gain)
    w.close()


def test_window_argument_errors(engine):
    from paper_1902_08653_b200 import ExchangeWindow, InvalidArgument
    with pytest.raises(InvalidArgument):
        ExchangeWindow(engine, 9, 0, S=72, C_total=8, U=16)
    w = ExchangeWindow(engine, 2, 0, S=16, C_total=8, U=16)
    H = torch.zeros((16, 4, 16, 32), dtype=torch.complex64, device="cuda")
    y = torch.zeros((16, 4, 32), dtype=torch.complex64, device="cuda")
    with pytest.raises(InvalidArgument, match="peer window 1 not open"):
        w.ul_detect(H, y, c0=0, C_total=8, n0=1.0)
    with pytest.raises(InvalidArgument, match="outside C_total"):
        w.ul_detect(H, y, c0=6, C_total=8, n0=1.0)
    w.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port_, fmt, fusion, out_dir):
    import torch.distributed as dist

    from paper_1902_08653_b200 import Engine
    from paper_1902_08653_b200.distributed import CudaCompute, DistributedCD, partition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    C, BC, U, S = 8, 32, 16, 64
    g = torch.Generator().manual_seed(5)
    H = (torch.randn((S, C, U, BC), dtype=torch.complex64, generator=g))
    y = (torch.randn((S, C, BC), dtype=torch.complex64, generator=g)) * 2.0
    part = partition(C, world, rank, S)
    eng = Engine(0)
    from paper_1902_08653_b200 import to_fp16_pairs
    Hl = H[:, part.c_lo:part.c_hi].contiguous().cuda()
    yl = y[:, part.c_lo:part.c_hi].contiguous().cuda()
    if fmt == "fp16":
        Hl, yl = to_fp16_pairs(Hl), to_fp16_pairs(yl)
    dcd = DistributedCD(part, CudaCompute(eng), mode="p2p")
    outs = []
    for _ in range(3):
        outs.append(dcd.uplink(Hl, yl, n0=1.6, K=3, fusion=fusion).cpu())
    eng.sync()
    np.save(os.path.join(out_dir, f"r{rank}.npy"), torch.stack(outs).numpy())
    traffic = dcd.traffic.uplink_bus_bytes
    np.save(os.path.join(out_dir, f"t{rank}.npy"), np.array([traffic]))
    # downlink: rank 0 (the centre) pushes its symbols, every rank precodes its clusters
    if fusion == "uniform":
        sy = torch.randn((S, U), dtype=torch.complex64, generator=g)
        syd = sy.cuda() if fmt == "fp32" else torch.view_as_real(sy).to(torch.float16).cuda().contiguous()
        dres = []
        for _ in range(3):
            xd, gain = dcd.downlink(Hl, dcd.broadcast_symbols(syd), rho=4.0, K=3)
            dres.append((xd.cpu(), gain.cpu()))
        eng.sync()
        torch.save(dres, os.path.join(out_dir, f"d{rank}.pt"))
    # a rank whose peer never publishes: DCDG_ECUDA after the window timeout, no hang
    dist.barrier()
    if rank == 0:
        dcd._xwin.set_timeout(0.5)
        dcd._xwin.ul_detect(Hl, yl, c0=part.c_lo, C_total=C, n0=1.6, K=3, fusion=fusion)
        try:
            eng.sync()
            msg = "no error"
        except Exception as e:  # CudaError with the exchange text
            msg = f"{type(e).__name__}: {e}"
        with open(os.path.join(out_dir, "timeout.txt"), "w") as f:
            f.write(msg)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,fmt,fusion", [(2, "fp32", "uniform"), (2, "fp16", "uniform"), (2, "fp32", "optimal"),
                                              (4, "fp32", "uniform"), (4, "fp32", "optimal")])
def test_ranks_on_one_gpu_bitwise(engine, tmp_path, world, fmt, fusion):
    """world 2 / 4 (processes sharing cuda:0, windows mapped by CUDA IPC):
    each rank's owned subcarriers equal the single-process fusion bitwise."""
    import torch.multiprocessing as mp

    from paper_1902_08653_b200 import to_fp16_pairs
    mp.spawn(_rank_main, args=(world, _free_port(), fmt, fusion, str(tmp_path)), nprocs=world, join=True)
    C, BC, U, S = 8, 32, 16, 64
    g = torch.Generator().manual_seed(5)
    H = torch.randn((S, C, U, BC), dtype=torch.complex64, generator=g).cuda()
    y = (torch.randn((S, C, BC), dtype=torch.complex64, generator=g) * 2.0).cuda()
    if fmt == "fp16":
        H, y = to_fp16_pairs(H), to_fp16_pairs(y)
    want = _single(engine, H, y, fusion=fusion, n0=1.6).cpu()
    cl = C // world
    for r in range(world):
        got = torch.from_numpy(np.load(tmp_path / f"r{r}.npy"))
        for step in range(got.shape[0]):
            assert torch.equal(torch.view_as_real(got[step]),
                               torch.view_as_real(want[r * S // world:(r + 1) * S // world]))
        # bus bytes: (W-1)/W of this rank's x_local (C_local clusters x U x esz per subcarrier) crosses
        esz = 8 if fmt == "fp32" else 4
        per = S * cl * U * esz + (S * cl * 4 if fusion == "optimal" else 0)
        assert int(np.load(tmp_path / f"t{r}.npy")[0]) == 3 * round(per * (world - 1) / world)
    if fusion == "uniform":
        g = torch.Generator().manual_seed(5)
        torch.randn((S, C, U, BC), dtype=torch.complex64, generator=g)
        torch.randn((S, C, BC), dtype=torch.complex64, generator=g)
        sy = torch.randn((S, U), dtype=torch.complex64, generator=g)
        syd = sy.cuda() if fmt == "fp32" else torch.view_as_real(sy).to(torch.float16).cuda().contiguous()
        want_dl = engine.dl_precode(H, syd, rho=4.0, K=3, want_gain=True)
        engine.sync()
        for r in range(world):
            for xd, gain in torch.load(tmp_path / f"d{r}.pt"):
                wx = want_dl.x[:, cl * r:cl * (r + 1)].cpu()
                assert torch.equal(torch.view_as_real(xd) if xd.is_complex() else xd,
                                   torch.view_as_real(wx) if wx.is_complex() else wx)
                assert torch.equal(gain, want_dl.gain.cpu())
    msg = (tmp_path / "timeout.txt").read_text()
    assert "CudaError" in msg and "never published" in msg, msg


def _alternate_main(rank, world, port_, out_dir):
    """Uplink and downlink calls alternating on ONE window with no host sync in
    between: both directions share the window's epoch/parity sequence, so a
    call never overwrites a parity buffer a peer may still be reading."""
    import torch.distributed as dist

    from paper_1902_08653_b200 import Engine
    from paper_1902_08653_b200.distributed import CudaCompute, DistributedCD, partition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    C, BC, U, S = 8, 32, 16, 64
    g = torch.Generator().manual_seed(5)
    H = torch.randn((S, C, U, BC), dtype=torch.complex64, generator=g)
    y = torch.randn((S, C, BC), dtype=torch.complex64, generator=g) * 2.0
    sy = torch.randn((S, U), dtype=torch.complex64, generator=g)
    part = partition(C, world, rank, S)
    eng = Engine(0)
    Hl = H[:, part.c_lo:part.c_hi].contiguous().cuda()
    yl = y[:, part.c_lo:part.c_hi].contiguous().cuda()
    syd = sy.cuda()
    dcd = DistributedCD(part, CudaCompute(eng), mode="p2p")
    ul, dl = [], []
    for i in range(8):  # UL, DL, UL, DL, ... all enqueued, read back only at the end
        ul.append(dcd.uplink(Hl, yl, n0=1.6, K=3, fusion="uniform" if i % 4 else "optimal").clone())
        x, gain = dcd.downlink(Hl, dcd.broadcast_symbols(syd), rho=4.0, K=3)
        dl.append((x.clone(), gain.clone()))
    eng.sync()
    torch.save({"ul": [u.cpu() for u in ul], "dl": [(x.cpu(), gn.cpu()) for x, gn in dl]},
               os.path.join(out_dir, f"alt{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_alternating_directions_share_one_window(engine, tmp_path, world):
    import torch.multiprocessing as mp
    mp.spawn(_alternate_main, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    C, BC, U, S = 8, 32, 16, 64
    g = torch.Generator().manual_seed(5)
    H = torch.randn((S, C, U, BC), dtype=torch.complex64, generator=g).cuda()
    y = (torch.randn((S, C, BC), dtype=torch.complex64, generator=g) * 2.0).cuda()
    sy = torch.randn((S, U), dtype=torch.complex64, generator=g).cuda()
    want_u = _single(engine, H, y, fusion="uniform", n0=1.6).cpu()
    want_o = _single(engine, H, y, fusion="optimal", n0=1.6).cpu()
    want_dl = engine.dl_precode(H, sy, rho=4.0, K=3, want_gain=True)
    engine.sync()
    cl, so = C // world, S // world
    for r in range(world):
        got = torch.load(tmp_path / f"alt{r}.pt")
        for i, u in enumerate(got["ul"]):
            want = (want_u if i % 4 else want_o)[r * so:(r + 1) * so]
            assert torch.equal(torch.view_as_real(u), torch.view_as_real(want)), (r, i)
        for x, gain in got["dl"]:
            assert torch.equal(torch.view_as_real(x), torch.view_as_real(want_dl.x[:, cl * r:cl * (r + 1)].cpu()))
            assert torch.equal(gain, want_dl.gain.cpu())
