"""GPU: the device paths around the CD kernels — partial (cross-GPU) fusion,
fusion weights, post-equalization variances, power scaling, numerical-error
reporting with the reference's texts, format conversion, and the distributed
driver on one GPU — against the CPU oracle."""
import numpy as np
import pytest
import torch

from helpers import OPTIMAL, TOL_FP32, UNIFORM, batch, qam_symbols, rel_err, to_dev, to_host

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fusion", ["uniform", "optimal"])
def test_partial_fusion_over_cluster_halves_equals_full_fusion(engine, port, fusion):
    """What two GPUs holding 4 clusters each compute before the NCCL reduce."""
    b = batch(8, 32, 16, S=40, seed=21)
    fu = UNIFORM if fusion == "uniform" else OPTIMAL
    xhat, _, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, fu)
    H, y = to_dev(b["h_tiles"]), to_dev(b["y"])
    parts = [engine.ul_detect(H[:, h * 4:(h + 1) * 4].contiguous(), y[:, h * 4:(h + 1) * 4].contiguous(), n0=b["n0"],
                              K=3, fusion=fusion, C_total=8) for h in range(2)]
    engine.sync()
    if fusion == "uniform":
        got = parts[0].xhat + parts[1].xhat
    else:
        num = parts[0].xhat + parts[1].xhat
        den = parts[0].wsum + parts[1].wsum
        got = engine.fuse_finalize(num.contiguous(), den.contiguous())
        engine.sync()
    assert rel_err(to_host(got), xhat) <= TOL_FP32


def test_fusion_weights_and_variances(engine, port):
    b = batch(4, 32, 8, S=16, seed=5)
    s2 = engine.post_eq_variance(to_dev(b["h_tiles"]), n0=b["n0"])
    engine.sync()
    ref = np.array([[port.post_eq_variance(b["h_tiles"][s, c].T, b["n0"], 1.0) for c in range(4)] for s in range(16)])
    assert np.max(np.abs(s2.cpu().numpy() - ref) / ref) <= TOL_FP32
    w = engine.fusion_weights(s2)
    engine.sync()
    wref = np.stack([port.fusion_weights(ref[s]) for s in range(16)])
    assert np.max(np.abs(w.cpu().numpy() - wref)) <= 1e-6


def test_power_scale_kat(engine):
    # test_precode.cpp:286-302: (3, 4i) scaled to rho=2 is (1.2, 1.6i)
    x = torch.tensor([[3.0 + 0j, 4.0j]], dtype=torch.complex64, device="cuda")
    engine.power_scale(x, 2.0)
    engine.sync()
    v = x.cpu().numpy()[0]
    assert abs(v[0] - 1.2) < 1e-6 and abs(v[1] - 1.6j) < 1e-6


def test_zero_channel_row_raises_reference_error(engine):
    from paper_1902_08653_b200 import NumericError
    b = batch(2, 32, 8, S=4, seed=9)
    h = b["h_tiles"].copy()
    h[2, 1, 5, :] = 0  # subcarrier 2, cluster 1, user 5: all-zero downlink row
    r = engine.dl_precode(to_dev(h), to_dev(qam_symbols(4, 8)), rho=1.0, K=3)
    with pytest.raises(NumericError, match="cd_precode: user 5 has an all-zero channel row") as ei:
        engine.sync()
    assert ei.value.problem == 2 * 2 + 1
    del r
    engine.sync()  # the status word is cleared after being reported


def test_zero_beamformer_raises(engine):
    from paper_1902_08653_b200 import NumericError
    x = torch.zeros((3, 8), dtype=torch.complex64, device="cuda")
    engine.power_scale(x, 1.0)
    with pytest.raises(NumericError, match="power_scale: zero beamformer cannot be scaled"):
        engine.sync()


def test_fp16_pair_conversion_roundtrip(engine):
    from paper_1902_08653_b200 import from_fp16_pairs, to_fp16_pairs
    t = (torch.randn(6, 32, dtype=torch.complex64, device="cuda"))
    back = from_fp16_pairs(to_fp16_pairs(t))
    assert torch.max(torch.abs(back - t)).item() < 2e-3 * torch.max(torch.abs(t)).item()


def test_distributed_driver_single_gpu(engine, port):
    from paper_1902_08653_b200.distributed import CudaCompute, DistributedCD, partition
    b = batch(8, 32, 16, S=32, seed=13)
    xhat, _, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
    dcd = DistributedCD(partition(8, 1, 0, 32), CudaCompute(engine))
    got = dcd.uplink(to_dev(b["h_tiles"]), to_dev(b["y"]), n0=b["n0"], K=3)
    engine.sync()
    assert rel_err(to_host(got), xhat) <= TOL_FP32


def test_graphed_uplink_replays_with_new_inputs(engine, port):
    from paper_1902_08653_b200 import GraphedUplink
    b1 = batch(8, 32, 16, S=24, seed=31)
    b2 = batch(8, 32, 16, S=24, seed=32)
    H, y = to_dev(b1["h_tiles"]), to_dev(b1["y"])
    g = GraphedUplink(engine, H, y, n0=b1["n0"], K=3)
    x1 = to_host(g.replay().clone())
    H.copy_(to_dev(b2["h_tiles"]))
    y.copy_(to_dev(b2["y"]))
    torch.cuda.synchronize()
    x2 = to_host(g.replay().clone())
    engine.sync()
    for b, x in ((b1, x1), (b2, x2)):
        ref, _, _ = port.ul_detect_batch(b["h_tiles"], b["y"], b["n0"], 1.0, 3, UNIFORM)
        assert rel_err(x, ref) <= TOL_FP32


@pytest.mark.parametrize("bc,u,fmt", [(32, 16, "fp32"), (32, 8, "fp32"), (64, 16, "fp32"), (32, 16, "fp16")])
def test_nonfinite_channel_optimal_fusion_raises_singular(engine, bc, u, fmt):
    """A NaN channel entry makes the variance's pivot non-positive: the
    reference's hermitian_solve throws (numerics.cpp:51-54) before any fusion,
    from whichever factorisation runs the shape (the fused fp32 CD kernel, the
    tensor-core variance kernel, the fp16 Gram kernel)."""
    from paper_1902_08653_b200 import NumericError, to_fp16_pairs
    b = batch(4, bc, u, S=6, seed=13)
    h = b["h_tiles"].copy()
    h[3, 2, 1, 4] = np.nan  # subcarrier 3, cluster 2
    H, y = to_dev(h), to_dev(b["y"])
    if fmt == "fp16":
        H, y = to_fp16_pairs(H), to_fp16_pairs(y)
    r = engine.ul_detect(H, y, n0=b["n0"], K=3, fusion="optimal")
    with pytest.raises(NumericError, match="hermitian_solve: matrix is numerically singular") as ei:
        engine.sync()
    assert ei.value.problem == 3 * 4 + 2
    del r
    engine.sync()  # the status word is cleared after being reported
