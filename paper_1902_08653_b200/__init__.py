"""B200-native decentralized coordinate-descent baseband (arXiv 1902.08653):
per-cluster CD L-MMSE uplink detection with feed-forward fusion and
per-cluster CD ZF downlink precoding, as hand-written sm_100a CUDA kernels
behind the C ABI in include/dcdg.h.

Python is plumbing here (device memory, streams, torch.distributed); the
compute path is libdcdg.so.  There is no CPU fallback.
"""
from ._lib import (FP16, FP32, FUSION_OPTIMAL, FUSION_UNIFORM, CudaError, DcdgError, InvalidArgument,  # noqa: F401
                   NumericError)
from .engine import (DownlinkResult, Engine, ExchangeWindow, GraphedUplink, UplinkResult, complex_empty, from_fp16_pairs,  # noqa: F401
                     kernel_name, to_complex64, to_fp16, to_fp16_pairs)

__all__ = ["Engine", "ExchangeWindow", "GraphedUplink", "UplinkResult", "DownlinkResult", "FP32", "FP16", "FUSION_OPTIMAL", "FUSION_UNIFORM",
           "DcdgError", "InvalidArgument", "NumericError", "CudaError", "kernel_name", "to_fp16", "to_fp16_pairs", "from_fp16_pairs", "to_complex64",
           "complex_empty"]
